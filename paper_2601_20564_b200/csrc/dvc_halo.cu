// dvc_halo.cu -- the multi-GPU halo transports of dvc_unet_decode_gop (see dvc_halo.cuh; SURVEY 8e;
// P:151 Inter-batch Shift across ranks).
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cstring>
#include <mutex>
#include "dvc_halo.cuh"

using namespace dvc;

namespace {
constexpr int kMaxBlocks = 32;                  // the U-Net has 22 ResBlocks
constexpr size_t kHdr = 256;                    // flags u32[32] | acks u32[32]
enum Transport { kP2P = 0, kNccl = 1 };

// ----------------------------------------------------------------- NCCL (dlopen'd from the process)
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // prefer the copy already loaded in the process (torch's), then the system one
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
        api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
        api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
        api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
                 api.GroupEnd;
    });
    return api;
}

#define DVC_NCCL(call)                                                                                   \
    do {                                                                                                 \
        ncclResult_t r_ = (call);                                                                        \
        if (r_ != ncclSuccess) {                                                                         \
            set_error("%s: NCCL error %d (%s)", #call, (int)r_,                                         \
                      nccl().GetErrorString ? nccl().GetErrorString(r_) : "?");                          \
            return DVC_ERR_NCCL;                                                                         \
        }                                                                                                \
    } while (0)

// ----------------------------------------------------------------- stream memory operations (driver API)
typedef CUresult (*PFN_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
    PFN_value32 wait = nullptr, write = nullptr;
};
const MemOps &memops() {
    static MemOps m;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            m.wait = reinterpret_cast<PFN_value32>(p);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            m.write = reinterpret_cast<PFN_value32>(p);
    });
    return m;
}

#define DVC_CU(call)                                                                                     \
    do {                                                                                                 \
        CUresult r_ = (call);                                                                            \
        if (r_ != CUDA_SUCCESS) {                                                                        \
            set_error("%s:%d %s: CUresult %d", __FILE__, __LINE__, #call, (int)r_);                      \
            return DVC_ERR_CUDA;                                                                         \
        }                                                                                                \
    } while (0)

inline CUdeviceptr dptr(const void *p) { return reinterpret_cast<CUdeviceptr>(p); }
}  // namespace

struct dvc_comm {
    int rank = 0, world = 1, transport = kP2P, device = 0;
    uint32_t epoch = 0;                 // decode calls so far (flag values; epoch parity = slot)
    cudaStream_t cs = nullptr;          // comm stream (sends, NCCL groups)
    cudaEvent_t ev_start = nullptr;     // start of the call on the compute stream
    cudaEvent_t ev_ready[kMaxBlocks] = {}, ev_sent[kMaxBlocks] = {};
    // P2P
    size_t carry_bytes = 0, slot_bytes = 0;
    uint8_t *region = nullptr;          // own: flags | acks | slot 0 | slot 1
    uint8_t *next = nullptr, *prev = nullptr;   // peers' regions (rank+1 / rank-1), mapped
    bool next_ipc = false, prev_ipc = false;
    // NCCL
    ncclComm_t nc = nullptr;
    uint8_t *scratch = nullptr;         // per call: received carries | staged slices (caller's workspace)
    size_t call_carry_bytes = 0;

    uint32_t *flags(uint8_t *r) const { return reinterpret_cast<uint32_t *>(r); }
    uint32_t *acks(uint8_t *r) const { return reinterpret_cast<uint32_t *>(r + 128); }
    uint8_t *slot(uint8_t *r, uint32_t e) const { return r + kHdr + (e & 1) * slot_bytes; }
};

static dvc_status comm_init_common(dvc_comm *c) {
    DVC_CUDA(cudaGetDevice(&c->device));
    int lo = 0, hi = 0;
    DVC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DVC_CUDA(cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi));   // highest priority
    DVC_CUDA(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    for (int k = 0; k < kMaxBlocks; ++k) {
        DVC_CUDA(cudaEventCreateWithFlags(&c->ev_ready[k], cudaEventDisableTiming));
        DVC_CUDA(cudaEventCreateWithFlags(&c->ev_sent[k], cudaEventDisableTiming));
    }
    return DVC_OK;
}

static void comm_free(dvc_comm *c) {
    if (!c) return;
    if (c->cs) cudaStreamSynchronize(c->cs);
    if (c->next_ipc && c->next) cudaIpcCloseMemHandle(c->next);
    if (c->prev_ipc && c->prev) cudaIpcCloseMemHandle(c->prev);
    if (c->region) cudaFree(c->region);
    if (c->nc && nccl().ok) nccl().CommDestroy(c->nc);
    for (int k = 0; k < kMaxBlocks; ++k) {
        if (c->ev_ready[k]) cudaEventDestroy(c->ev_ready[k]);
        if (c->ev_sent[k]) cudaEventDestroy(c->ev_sent[k]);
    }
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
}

namespace dvc {

int comm_world(const dvc_comm *c) { return c ? c->world : 1; }
int comm_rank(const dvc_comm *c) { return c ? c->rank : 0; }

dvc_status halo_call_begin(dvc_comm *c, size_t carry_bytes, void *nccl_scratch, cudaStream_t s) {
    int dev = -1;
    DVC_CUDA(cudaGetDevice(&dev));
    DVC_CHECK_ARG(dev == c->device, DVC_ERR_ARG, "comm was created on device %d, decode runs on %d", c->device, dev);
    if (c->transport == kP2P) {
        DVC_CHECK_ARG(carry_bytes <= c->carry_bytes, DVC_ERR_SHAPE,
                      "comm receive slots hold %zu bytes, the network's carry needs %zu", c->carry_bytes, carry_bytes);
        DVC_CHECK_ARG((c->rank == c->world - 1 || c->next) && (c->rank == 0 || c->prev), DVC_ERR_ARG,
                      "P2P comm not connected (dvc_comm_connect_ipc / dvc_comm_connect_local)");
        DVC_CHECK_ARG(memops().wait && memops().write, DVC_ERR_UNSUPPORTED, "stream memory operations unavailable");
    } else {
        DVC_CHECK_ARG(nccl().ok, DVC_ERR_NCCL, "NCCL unavailable");
        DVC_CHECK_ARG(nccl_scratch != nullptr, DVC_ERR_WORKSPACE, "NCCL halo needs workspace scratch");
        c->scratch = reinterpret_cast<uint8_t *>(nccl_scratch);
        c->call_carry_bytes = carry_bytes;
    }
    ++c->epoch;
    // the comm stream starts after everything the caller enqueued before this call (buffer reuse)
    DVC_CUDA(cudaEventRecord(c->ev_start, s));
    DVC_CUDA(cudaStreamWaitEvent(c->cs, c->ev_start, 0));
    return DVC_OK;
}

dvc_status halo_exchange(dvc_comm *c, int k, const HaloSlice &sl, cudaStream_t s, const void **carry) {
    DVC_CHECK_ARG(k >= 0 && k < kMaxBlocks, DVC_ERR_ARG, "halo block index %d", k);
    const uint32_t e = c->epoch;
    const bool sends = c->rank < c->world - 1, recvs = c->rank > 0;
    if (sends) {   // X_k is complete on s: the comm stream takes it from here
        DVC_CUDA(cudaEventRecord(c->ev_ready[k], s));
        DVC_CUDA(cudaStreamWaitEvent(c->cs, c->ev_ready[k], 0));
    }
    if (c->transport == kP2P) {
        if (sends) {
            // the successor consumed this slot two calls ago (double-buffered by epoch parity)
            if (e >= 3) DVC_CU(memops().wait(c->cs, dptr(c->acks(c->region) + k), e - 2, CU_STREAM_WAIT_VALUE_GEQ));
            DVC_CUDA(cudaMemcpy2DAsync(c->slot(c->next, e) + sl.off, sl.row_bytes, sl.src, sl.src_pitch, sl.row_bytes,
                                       sl.rows, cudaMemcpyDefault, c->cs));
            // default flags: the write is ordered after the copy's data (memory barrier before the write)
            DVC_CU(memops().write(c->cs, dptr(c->flags(c->next) + k), e, CU_STREAM_WRITE_VALUE_DEFAULT));
            DVC_CUDA(cudaEventRecord(c->ev_sent[k], c->cs));
        }
        if (recvs) {
            DVC_CU(memops().wait(s, dptr(c->flags(c->region) + k), e, CU_STREAM_WAIT_VALUE_GEQ));
            *carry = c->slot(c->region, e) + sl.off;
        }
        return DVC_OK;
    }
    // NCCL: stage the strided slice, then one send/recv group on the comm stream
    uint8_t *recvb = c->scratch, *stage = c->scratch + ((c->call_carry_bytes + 255) & ~size_t(255));
    const size_t count = sl.rows * sl.row_bytes / 2;   // 16-bit elements (the decode is 16-bit or fp32)
    if (sends)
        DVC_CUDA(cudaMemcpy2DAsync(stage + sl.off, sl.row_bytes, sl.src, sl.src_pitch, sl.row_bytes, sl.rows,
                                   cudaMemcpyDeviceToDevice, c->cs));
    DVC_NCCL(nccl().GroupStart());
    if (sends) DVC_NCCL(nccl().Send(stage + sl.off, count, ncclFloat16, c->rank + 1, c->nc, c->cs));
    if (recvs) DVC_NCCL(nccl().Recv(recvb + sl.off, count, ncclFloat16, c->rank - 1, c->nc, c->cs));
    DVC_NCCL(nccl().GroupEnd());
    DVC_CUDA(cudaEventRecord(c->ev_sent[k], c->cs));
    if (recvs) {
        DVC_CUDA(cudaStreamWaitEvent(s, c->ev_sent[k], 0));
        *carry = recvb + sl.off;
    }
    return DVC_OK;
}

dvc_status halo_block_done(dvc_comm *c, int k, cudaStream_t s) {
    const bool sends = c->rank < c->world - 1, recvs = c->rank > 0;
    if (c->transport == kP2P && recvs)   // block k has read its carry slot: the predecessor may reuse it
        DVC_CU(memops().write(s, dptr(c->acks(c->prev) + k), c->epoch, CU_STREAM_WRITE_VALUE_DEFAULT));
    if (sends) DVC_CUDA(cudaStreamWaitEvent(s, c->ev_sent[k], 0));   // X_k may be overwritten from here on
    return DVC_OK;
}

dvc_status halo_call_end(dvc_comm *c, cudaStream_t s) {
    (void)s;
    if (c->transport == kNccl && nccl().CommGetAsyncError) {
        ncclResult_t ar = ncclSuccess;
        nccl().CommGetAsyncError(c->nc, &ar);
        DVC_CHECK_ARG(ar == ncclSuccess || ar == ncclInProgress, DVC_ERR_NCCL, "NCCL async error %d", (int)ar);
    }
    return DVC_OK;
}

}  // namespace dvc

extern "C" {

dvc_status dvc_comm_unique_id(void *id128) {
    DVC_CHECK_ARG(id128, DVC_ERR_ARG, "null id");
    DVC_CHECK_ARG(nccl().ok, DVC_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    DVC_NCCL(nccl().GetUniqueId(&id));
    memcpy(id128, &id, sizeof(id));
    return DVC_OK;
}

dvc_status dvc_comm_create(int rank, int world, const void *id128, dvc_comm **out) {
    DVC_CHECK_ARG(out && id128 && world >= 1 && rank >= 0 && rank < world, DVC_ERR_ARG, "bad comm arguments");
    DVC_CHECK_ARG(nccl().ok, DVC_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    dvc_comm *c = new dvc_comm();
    c->rank = rank, c->world = world, c->transport = kNccl;
    dvc_status st = comm_init_common(c);
    if (st != DVC_OK) {
        comm_free(c);
        return st;
    }
    ncclResult_t r = nccl().CommInitRank(&c->nc, world, id, rank);
    if (r != ncclSuccess) {
        c->nc = nullptr;
        comm_free(c);
        set_error("ncclCommInitRank failed: %d", (int)r);
        return DVC_ERR_NCCL;
    }
    *out = c;
    return DVC_OK;
}

dvc_status dvc_comm_create_p2p(int rank, int world, size_t carry_bytes, dvc_comm **out) {
    DVC_CHECK_ARG(out && world >= 1 && rank >= 0 && rank < world && carry_bytes > 0, DVC_ERR_ARG,
                  "bad comm arguments");
    DVC_CHECK_ARG(memops().wait && memops().write, DVC_ERR_UNSUPPORTED, "stream memory operations unavailable");
    dvc_comm *c = new dvc_comm();
    c->rank = rank, c->world = world, c->transport = kP2P;
    c->carry_bytes = carry_bytes;
    c->slot_bytes = (carry_bytes + 255) & ~size_t(255);
    dvc_status st = comm_init_common(c);
    if (st == DVC_OK) {
        const size_t bytes = kHdr + 2 * c->slot_bytes;
        cudaError_t e = cudaMalloc(&c->region, bytes);
        if (e == cudaSuccess) e = cudaMemset(c->region, 0, kHdr);   // flags and acks start at epoch 0
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            set_error("P2P comm region (%zu bytes): %s", bytes, cudaGetErrorString(e));
            st = DVC_ERR_CUDA;
        }
    }
    if (st != DVC_OK) {
        comm_free(c);
        return st;
    }
    *out = c;
    return DVC_OK;
}

dvc_status dvc_comm_ipc_handle(const dvc_comm *c, void *handle64) {
    DVC_CHECK_ARG(c && handle64 && c->transport == kP2P, DVC_ERR_ARG, "need a P2P comm and a 64-byte buffer");
    cudaIpcMemHandle_t h;
    DVC_CUDA(cudaIpcGetMemHandle(&h, c->region));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle64, &h, sizeof(h));
    return DVC_OK;
}

dvc_status dvc_comm_connect_ipc(dvc_comm *c, const void *next64, const void *prev64) {
    DVC_CHECK_ARG(c && c->transport == kP2P, DVC_ERR_ARG, "need a P2P comm");
    DVC_CHECK_ARG((next64 != nullptr) == (c->rank < c->world - 1) && (prev64 != nullptr) == (c->rank > 0),
                  DVC_ERR_ARG, "rank %d of %d needs next=%s prev=%s", c->rank, c->world,
                  c->rank < c->world - 1 ? "handle" : "NULL", c->rank > 0 ? "handle" : "NULL");
    DVC_CHECK_ARG(!c->next && !c->prev, DVC_ERR_ARG, "comm already connected");
    cudaIpcMemHandle_t h;
    void *p = nullptr;
    if (next64) {
        memcpy(&h, next64, sizeof(h));
        DVC_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->next = reinterpret_cast<uint8_t *>(p), c->next_ipc = true;
    }
    if (prev64) {
        memcpy(&h, prev64, sizeof(h));
        DVC_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->prev = reinterpret_cast<uint8_t *>(p), c->prev_ipc = true;
    }
    return DVC_OK;
}

dvc_status dvc_comm_connect_local(dvc_comm *c, const dvc_comm *next, const dvc_comm *prev) {
    DVC_CHECK_ARG(c && c->transport == kP2P, DVC_ERR_ARG, "need a P2P comm");
    DVC_CHECK_ARG((next != nullptr) == (c->rank < c->world - 1) && (prev != nullptr) == (c->rank > 0), DVC_ERR_ARG,
                  "rank %d of %d: wrong neighbours", c->rank, c->world);
    DVC_CHECK_ARG(!next || (next->transport == kP2P && next->rank == c->rank + 1 && next->world == c->world &&
                            next->slot_bytes == c->slot_bytes),
                  DVC_ERR_ARG, "next is not rank+1 of the same P2P group");
    DVC_CHECK_ARG(!prev || (prev->transport == kP2P && prev->rank == c->rank - 1 && prev->world == c->world &&
                            prev->slot_bytes == c->slot_bytes),
                  DVC_ERR_ARG, "prev is not rank-1 of the same P2P group");
    DVC_CHECK_ARG(!c->next && !c->prev, DVC_ERR_ARG, "comm already connected");
    c->next = next ? next->region : nullptr;
    c->prev = prev ? prev->region : nullptr;
    return DVC_OK;
}

dvc_status dvc_comm_destroy(dvc_comm *c) {
    comm_free(c);
    return DVC_OK;
}

}  // extern "C"
