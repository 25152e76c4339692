// dvc_halo.cuh -- the multi-GPU halo of dvc_unet_decode_gop (row e of SURVEY 8; "passes the
// partial channels of the last sample ... to the subsequent batch (Inter-batch Shift)").
//
// A chain's frames are split into contiguous chunks, one per rank.  Before ResBlock k, rank r's
// block input X_k holds the slice X_k[T_local-1][..., 0:C_in/P] that rank r+1 needs as the carry of
// its first frame.  The exchange is a one-directional halo r -> r+1 per block (22 per decode call),
// lock-step: every rank works at the same depth.
//
// Two transports, one interface:
//   P2P (default): every rank owns a receive region (two epoch slots of the packed 22-slice carry,
//     22 arrival flags, 22 acknowledgement words).  The sender copies the slice straight from X_k into
//     its successor's slot with a copy-engine peer copy over NVLink (no SM, no staging), on the comm
//     stream, and raises the successor's arrival flag with a stream memory write; the receiver's
//     compute stream waits on its local flag with a stream memory wait (the front end blocks, no SM
//     spins, no NCCL kernel).  Peers are mapped with CUDA IPC (other processes) or directly (ranks of
//     one process: the single-GPU loopback used by the tests).
//   NCCL: the slice is staged into a contiguous buffer and moved by ncclSend/ncclRecv in one group on
//     the comm stream; the compute stream waits on an event.
// In both, the send of block k overlaps block k's own compute (only the receive is on the critical
// path), and the compute stream waits for the send to finish before block k+1 can overwrite X_k.
#pragma once
#include "dvc_common.cuh"

struct dvc_comm;

namespace dvc {

struct HaloSlice {
    const void *src;    // &X_k[T_local-1][0][0][0]
    size_t src_pitch;   // bytes between pixels of X_k (C_a * element size)
    size_t row_bytes;   // slice bytes per pixel (C_in/P * element size)
    size_t rows;        // pixels per frame (h * w)
    size_t off;         // byte offset of block k's slice in the packed carry
};

int comm_world(const dvc_comm *c);
int comm_rank(const dvc_comm *c);
// Start of one decode call: checks the comm against the call (carry bytes, device), advances the epoch.
// nccl_scratch: 2 x carry_bytes (256-aligned) of the caller's workspace (NCCL transport only).
dvc_status halo_call_begin(dvc_comm *c, size_t carry_bytes, void *nccl_scratch, cudaStream_t s);
// Block k: send my slice onward (rank < world-1), and (rank > 0) make s wait for the predecessor's
// slice; *carry receives the device pointer of that slice (unchanged on rank 0).
dvc_status halo_exchange(dvc_comm *c, int k, const HaloSlice &sl, cudaStream_t s, const void **carry);
// After block k is enqueued on s: the received slot may be reused (acknowledge to the sender), and s
// waits until my own send of block k has left X_k.
dvc_status halo_block_done(dvc_comm *c, int k, cudaStream_t s);
// End of the call: surfaces asynchronous transport errors.
dvc_status halo_call_end(dvc_comm *c, cudaStream_t s);

}  // namespace dvc
