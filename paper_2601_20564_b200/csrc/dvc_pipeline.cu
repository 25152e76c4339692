// dvc_pipeline.cu -- f3: the Asynchronous and Parallel Decoding Pipeline.
//
// The paper's decoder has two branches: the Latent Compressor runs in the prediction loop
// (frame t needs Lbar_{t-1}) and the Frame Reconstructor (U-Net, then optionally the VAE
// decoder -> frames) runs out of the loop.  They
// are decoupled through buffers and the reconstructor takes N frames at a time on the batch
// dimension, the Batch-dimension OTSM carrying the shifted slices from batch to batch.
//
// B200 mapping: the in-loop producer is whatever the caller runs on its stream; push() copies
// each frame's (Lbar_t, C^m_t) into a FIFO slot on that stream (stream-ordered device copies,
// no host synchronisation), and a full slot is handed to the reconstructor stream through a CUDA
// event.  The reconstructor decodes slot after slot with the inter-batch carry ping-ponging
// between two device buffers (the decodes are serialised on one stream, so two suffice).
// pop() enqueues the copy-out of the oldest decoded slot on the caller's stream behind the
// decode's event and records the slot's release, which the next push into that slot waits for.
// All device work is the library's own kernels; the host only does bookkeeping.
#include <cstring>
#include <vector>
#include "dvc_common.cuh"

struct dvc_pipeline {
    dvc_unet *net = nullptr;
    dvc_vae *vae = nullptr;      // optional: the Frame Reconstructor's VAE decoder (frames out)
    void *vws = nullptr;
    size_t vws_bytes = 0, out_elems = 0;   // per frame: h*w*c_lat latents or 8h*8w*out_ch pixels
    dvc_unet_config cfg{};
    int N = 0, K = 0;
    size_t lat_elems = 0, ctx_elems = 0, es = 0;   // per frame
    struct Slot {
        void *lat = nullptr, *ctx = nullptr, *out = nullptr, *pix = nullptr;   // pix: VAE frames
        int frames = 0;
        long long first = 0;
        bool launched = false;   // decode enqueued, not yet popped
        bool freed_valid = false;
        cudaEvent_t filled = nullptr, decoded = nullptr, freed = nullptr;
    };
    std::vector<Slot> slots;
    int fill = 0, oldest = 0, in_flight = 0;
    void *carry[2] = {nullptr, nullptr};
    int cur = 0;
    bool chain_start = true;
    void *ws = nullptr;
    size_t ws_bytes = 0;
    cudaStream_t fr = nullptr;
    cudaStream_t last_stream = nullptr;
    long long frame_counter = 0;
};

using namespace dvc;

static void pipeline_free(dvc_pipeline *p) {
    if (!p) return;
    if (p->fr) cudaStreamSynchronize(p->fr);
    for (auto &s : p->slots) {
        cudaFree(s.lat);
        cudaFree(s.ctx);
        cudaFree(s.out);
        cudaFree(s.pix);
        if (s.filled) cudaEventDestroy(s.filled);
        if (s.decoded) cudaEventDestroy(s.decoded);
        if (s.freed) cudaEventDestroy(s.freed);
    }
    cudaFree(p->carry[0]);
    cudaFree(p->carry[1]);
    cudaFree(p->ws);
    cudaFree(p->vws);
    if (p->fr) cudaStreamDestroy(p->fr);
    delete p;
}

static dvc_status launch_slot(dvc_pipeline *p, cudaStream_t producer) {
    dvc_pipeline::Slot &s = p->slots[p->fill];
    DVC_CUDA(cudaEventRecord(s.filled, producer));
    DVC_CUDA(cudaStreamWaitEvent(p->fr, s.filled, 0));
    const void *cin = p->chain_start ? nullptr : p->carry[p->cur];
    void *cout = p->carry[p->cur ^ 1];
    dvc_status st = dvc_unet_decode_gop(p->net, nullptr, s.lat, s.ctx, s.frames, cin, cout, s.out, p->ws, p->ws_bytes,
                                        p->fr);
    if (st != DVC_OK) return st;
    if (p->vae) {   // Lhat -> frames through the VAE decoder on the same stream
        st = dvc_vae_decode(p->vae, s.out, s.frames, s.pix, p->vws, p->vws_bytes, p->fr);
        if (st != DVC_OK) return st;
    }
    DVC_CUDA(cudaEventRecord(s.decoded, p->fr));
    p->cur ^= 1;
    p->chain_start = false;
    s.launched = true;
    ++p->in_flight;
    p->fill = (p->fill + 1) % p->K;
    return DVC_OK;
}

extern "C" {

dvc_status dvc_pipeline_create(dvc_unet *net, dvc_vae *vae, int batch_n, int fifo_batches, dvc_pipeline **out) {
    DVC_CHECK_ARG(net && out, DVC_ERR_ARG, "null argument");
    const dvc_unet_config *c = dvc_unet_get_config(net);
    DVC_CHECK_ARG(batch_n >= 1 && batch_n <= c->max_T, DVC_ERR_ARG, "batch_n=%d outside [1, max_T=%d]", batch_n,
                  c->max_T);
    DVC_CHECK_ARG(fifo_batches >= 1 && fifo_batches <= 64, DVC_ERR_ARG, "fifo_batches outside [1, 64]");
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    dvc_pipeline *p = new dvc_pipeline();
    p->net = net;
    p->cfg = *c;
    p->N = batch_n;
    p->K = fifo_batches;
    p->es = dt_size(c->dt);
    p->lat_elems = (size_t)c->h * c->w * c->c_lat;
    p->ctx_elems = (size_t)c->h * c->w * c->c_ctx;
    p->out_elems = p->lat_elems;
    if (vae) {
        const dvc_vae_config *vc = dvc_vae_get_config(vae);
        if (vc->h != c->h || vc->w != c->w || vc->c_lat != c->c_lat || vc->dt != c->dt || vc->max_T < batch_n) {
            delete p;
            set_error("pipeline: VAE config does not match the U-Net (h, w, c_lat, dtype, max_T >= N)");
            return DVC_ERR_SHAPE;
        }
        p->vae = vae;
        p->out_elems = (size_t)64 * c->h * c->w * vc->out_ch;
        dvc_vae_workspace_size(vae, batch_n, &p->vws_bytes);
    }
    size_t carry = 0;
    dvc_unet_carry_size(net, &carry);
    dvc_unet_workspace_size(net, batch_n, &p->ws_bytes);
    bool ok = cudaStreamCreateWithFlags(&p->fr, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMalloc(&p->ws, p->ws_bytes) == cudaSuccess &&
              cudaMalloc(&p->carry[0], carry * p->es + 16) == cudaSuccess &&
              cudaMalloc(&p->carry[1], carry * p->es + 16) == cudaSuccess &&
              (!vae || cudaMalloc(&p->vws, p->vws_bytes) == cudaSuccess);
    p->slots.resize(fifo_batches);
    for (auto &s : p->slots) {
        ok = ok && cudaMalloc(&s.lat, p->lat_elems * p->es * batch_n) == cudaSuccess &&
             cudaMalloc(&s.ctx, p->ctx_elems * p->es * batch_n) == cudaSuccess &&
             cudaMalloc(&s.out, p->lat_elems * p->es * batch_n) == cudaSuccess &&
             (!vae || cudaMalloc(&s.pix, p->out_elems * p->es * batch_n) == cudaSuccess) &&
             cudaEventCreateWithFlags(&s.filled, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&s.decoded, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) {
        pipeline_free(p);
        set_error("pipeline: device allocation failed");
        return DVC_ERR_CUDA;
    }
    *out = p;
    return DVC_OK;
}

dvc_status dvc_pipeline_destroy(dvc_pipeline *p) {
    pipeline_free(p);
    return DVC_OK;
}

dvc_status dvc_pipeline_push(dvc_pipeline *p, const void *lat, const void *ctx, void *stream) {
    DVC_CHECK_ARG(p && lat && ctx, DVC_ERR_ARG, "null argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!p->slots[p->fill].launched && p->slots[p->fill].frames >= p->N) {
        // a full slot whose launch failed earlier (e.g. a pending CUDA error): launch it first, never
        // copy past the slot's N-frame allocation
        dvc_status st = launch_slot(p, p->last_stream);
        if (st != DVC_OK) return st;
    }
    dvc_pipeline::Slot &sl = p->slots[p->fill];
    DVC_CHECK_ARG(!sl.launched, DVC_ERR_ARG, "pipeline FIFO full: %d decoded batches not popped", p->in_flight);
    if (sl.frames == 0) {
        if (sl.freed_valid) DVC_CUDA(cudaStreamWaitEvent(s, sl.freed, 0));   // previous pop's copy-out
        sl.first = p->frame_counter;
    }
    const size_t lb = p->lat_elems * p->es, cb = p->ctx_elems * p->es;
    DVC_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t *>(sl.lat) + sl.frames * lb, lat, lb, cudaMemcpyDeviceToDevice, s));
    DVC_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t *>(sl.ctx) + sl.frames * cb, ctx, cb, cudaMemcpyDeviceToDevice, s));
    ++sl.frames;
    ++p->frame_counter;
    p->last_stream = s;
    if (sl.frames == p->N) return launch_slot(p, s);
    return DVC_OK;
}

dvc_status dvc_pipeline_pop(dvc_pipeline *p, void *out, void *stream, int *frames, long long *first_frame) {
    DVC_CHECK_ARG(p && out && frames, DVC_ERR_ARG, "null argument");
    *frames = 0;
    if (p->in_flight == 0) return DVC_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    dvc_pipeline::Slot &sl = p->slots[p->oldest];
    DVC_CUDA(cudaStreamWaitEvent(s, sl.decoded, 0));
    DVC_CUDA(cudaMemcpyAsync(out, p->vae ? sl.pix : sl.out, (size_t)sl.frames * p->out_elems * p->es,
                             cudaMemcpyDeviceToDevice, s));
    DVC_CUDA(cudaEventRecord(sl.freed, s));
    sl.freed_valid = true;
    *frames = sl.frames;
    if (first_frame) *first_frame = sl.first;
    sl.frames = 0;
    sl.launched = false;
    --p->in_flight;
    p->oldest = (p->oldest + 1) % p->K;
    return DVC_OK;
}

dvc_status dvc_pipeline_flush(dvc_pipeline *p) {
    DVC_CHECK_ARG(p, DVC_ERR_ARG, "null argument");
    dvc_pipeline::Slot &sl = p->slots[p->fill];
    if (sl.frames == 0 || sl.launched) return DVC_OK;
    return launch_slot(p, p->last_stream);
}

dvc_status dvc_pipeline_reset(dvc_pipeline *p) {
    DVC_CHECK_ARG(p, DVC_ERR_ARG, "null argument");
    dvc_status st = dvc_pipeline_flush(p);
    if (st != DVC_OK) return st;
    p->chain_start = true;
    p->frame_counter = 0;
    return DVC_OK;
}

}  // extern "C"
