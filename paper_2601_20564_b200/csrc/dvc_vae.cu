// dvc_vae.cu -- f2: the Pruned VAE Decoder ("reduces intermediate channels by 50%",
// P:108 256-channel latent interface, Table 8; readings R29-R31).
//
// Topology (SD-2.1 AutoencoderKL decoder, block widths x0.5 = (64, 128, 256, 256)):
//   x = conv_in(Lhat)                         3x3, c_lat -> 256, latent resolution (level 0)
//   mid: ResBlock, single-head self-attention (GN, q/k/v/out linears, + x), ResBlock
//   up level i = 0..3 (widths reversed 256, 256, 128, 64): 3 ResBlocks; i < 3: nearest 2x
//        (exact copy) + 3x3 conv at level i+1
//   out = conv_out(SiLU(GN_out(x)))           3x3, 64 -> out_ch at full resolution
// Frames are independent (no temporal shift): the ResBlocks run through the same engines as
// the U-Net's with shift_p = 0 (fused GN-apply + SiLU producer, epilogue box statistics), the
// mid attention through the tcgen05 attention kernel with head_dim = C (256).  conv_out (16-bit)
// is the streaming output head of dvc_conv_out.cu, writing the out_ch channels straight into the
// frames; fp32 (and shapes it does not take) compute a 16-channel tile (zero weight rows) that a
// copy kernel slices.
#include <cstring>
#include <vector>
#include "dvc_attn.cuh"
#include "dvc_conv.cuh"
#include "dvc_norm.cuh"
#include "dvc_resblock.cuh"

using namespace dvc;

namespace {
struct VConv {
    const void *w = nullptr, *b = nullptr;
};
constexpr int kVBlocks = 14;   // mid 2 + 4 levels x 3
}  // namespace

struct dvc_vae {
    dvc_vae_config cfg{};
    void *dweights = nullptr, *dextra = nullptr;
    VConv conv_in, us[3], conv_out16;
    RB blk[kVBlocks];
    int blevel[kVBlocks];
    const void *gno_w = nullptr, *gno_b = nullptr;
    const void *at_gn_w = nullptr, *at_gn_b = nullptr, *at_out_w = nullptr, *at_out_b = nullptr;
    const void *at_q[6] = {};   // q_w, q_b, k_w, k_b, v_w, v_b (blob order)
    void *qkv_w = nullptr, *qkv_b = nullptr;   // concatenated [3C][C], [3C] (dextra)
    int lh[4], lw[4];
};

namespace {

template <typename Take>
void vwalk(dvc_vae &v, Take take) {
    const dvc_vae_config &c = v.cfg;
    const int top = c.width[3];
    auto conv = [&](int cout, int cin, int k) {
        VConv cw;
        cw.w = take((size_t)cout * k * k * cin);
        cw.b = take((size_t)cout);
        return cw;
    };
    int bi = 0;
    auto block = [&](int cin, int cout, int level) {
        RB &r = v.blk[bi];
        r.ca = cin;
        r.cb = 0;
        r.cout = cout;
        r.G = c.groups;
        r.P = 0;   // no temporal shift in the VAE decoder
        r.eps = c.eps;
        r.dt = c.dt;
        r.gn1_w = take(cin);
        r.gn1_b = take(cin);
        r.conv1_w = take((size_t)cout * 9 * cin);
        r.conv1_b = take(cout);
        r.gn2_w = take(cout);
        r.gn2_b = take(cout);
        r.conv2_w = take((size_t)cout * 9 * cout);
        r.conv2_b = take(cout);
        if (cin != cout) {
            r.sc_w = take((size_t)cout * cin);
            r.sc_b = take(cout);
        } else {
            r.sc_w = r.sc_b = nullptr;
        }
        v.blevel[bi++] = level;
    };
    v.conv_in = conv(top, c.c_lat, 3);
    block(top, top, 0);
    if (c.mid_attn) {
        v.at_gn_w = take(top);
        v.at_gn_b = take(top);
        for (int i = 0; i < 3; ++i) {
            v.at_q[2 * i] = take((size_t)top * top);
            v.at_q[2 * i + 1] = take(top);
        }
        v.at_out_w = take((size_t)top * top);
        v.at_out_b = take(top);
    }
    block(top, top, 0);
    int cur = top;
    for (int i = 0; i < 4; ++i) {
        const int ch = c.width[3 - i];
        for (int r = 0; r < 3; ++r) {
            block(cur, ch, i);
            cur = ch;
        }
        if (i < 3) v.us[i] = conv(ch, ch, 3);
    }
    v.gno_w = take(cur);
    v.gno_b = take(cur);
    v.conv_out16 = conv(c.out_ch, cur, 3);   // blob weights; replaced by the padded copy at create
}

dvc_status vvalidate(const dvc_vae_config *c) {
    DVC_CHECK_ARG(c, DVC_ERR_ARG, "null config");
    DVC_CHECK_ARG(dt_valid(c->dt), DVC_ERR_ARG, "bad dtype");
    DVC_CHECK_ARG(c->h >= 1 && c->w >= 1 && c->max_T >= 1 && c->max_T < 256, DVC_ERR_ARG, "bad size / max_T");
    DVC_CHECK_ARG(c->c_lat > 0 && c->out_ch >= 1 && c->out_ch <= 16 && c->groups >= 1, DVC_ERR_ARG,
                  "bad channels (1 <= out_ch <= 16)");
    for (int i = 0; i < 4; ++i) DVC_CHECK_ARG(c->width[i] > 0, DVC_ERR_ARG, "bad width");
    DVC_CHECK_ARG(8 * c->h < 4096 && 8 * c->w < 4096, DVC_ERR_UNSUPPORTED, "frame size < 4096 required");
    if (c->mid_attn) {
        const int C = c->width[3];
        DVC_CHECK_ARG(C == 16 || C == 32 || C == 48 || C == 64 || C == 256, DVC_ERR_UNSUPPORTED,
                      "single-head mid attention needs width[3] in {16,32,48,64,256}");
    }
    return DVC_OK;
}

// workspace: 0/1 ping-pong activations, 2 upsample intermediate / attention scratch, 3 ResBlock
// scratch, 4/5 box statistics of 0/1, 6 padded conv_out tile
constexpr int kVRegions = 7;

size_t vplan(const dvc_vae &v, int T, size_t *offs) {
    const dvc_vae_config &c = v.cfg;
    const size_t es = dt_size(c.dt);
    size_t sz[kVRegions] = {};
    size_t act = 0, st = 0, rbws = 0;
    auto hw = [&](int l) { return (size_t)v.lh[l] * v.lw[l]; };
    for (int l = 0; l < 4; ++l) {
        const int chs[2] = {c.width[3 - l], l > 0 ? c.width[4 - l] : c.width[3]};   // this level's, incoming
        for (int ch : chs) {
            act = std::max(act, T * hw(l) * (size_t)ch);
            st = std::max(st, box_stats_bytes(T, v.lh[l], v.lw[l], ch));
        }
    }
    for (int b = 0; b < kVBlocks; ++b) {
        const RB &r = v.blk[b];
        const int l = v.blevel[b];
        rbws = std::max(rbws, resblock_ws_bytes(r.ca, r.cb, r.cout, r.G, T, v.lh[l], v.lw[l], c.dt));
    }
    sz[0] = sz[1] = act * es;
    // upsample intermediate (level l+1 at the incoming width) or the attention scratch
    size_t scratch = act * es;
    if (c.mid_attn) {
        const int C = c.width[3];
        const size_t px = T * hw(0);
        scratch = std::max(scratch, align256(px * C * es) + align256(px * 3 * C * es) + align256(px * C * es) +
                                        attn_ws_bytes(T, (int)hw(0), C, c.dt) + align256((size_t)T * C * 8));
    }
    sz[2] = scratch;
    sz[3] = std::max(rbws, align256((size_t)T * c.width[0] * 8) + gn_workspace_bytes(T, (int)hw(3), c.groups,
                                                                                      c.width[0]));
    sz[4] = sz[5] = st;
    // padded conv_out tile: only the paths that slice (fp32, shapes the output head does not take)
    sz[6] = conv_out_applicable(c.width[0], c.out_ch, c.dt) ? 0 : T * hw(3) * 16 * es;
    size_t total = 0;
    for (int i = 0; i < kVRegions; ++i) {
        offs[i] = total;
        total += align256(sz[i]);
    }
    return total;
}

// [T][HW][16] -> [T][HW][out_ch]
template <typename T>
__global__ void __launch_bounds__(256) slice_kernel(const T *__restrict__ src, T *__restrict__ dst, long px, int oc) {
    griddep_wait();
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < px * oc; i += (long)gridDim.x * blockDim.x) {
        const long p = i / oc;
        dst[i] = src[p * 16 + (i - p * oc)];
    }
    griddep_launch();
}

dvc_status slice_run(const void *src, void *dst, long px, int oc, dvc_dtype dt, cudaStream_t s) {
    const int blocks = (int)std::min<long>((px * oc + 255) / 256, 148L * 16);
    if (dt == DVC_BF16)
        DVC_CUDA(launch_pdl(slice_kernel<__nv_bfloat16>, dim3(blocks), dim3(256), 0, s, 1,
                            reinterpret_cast<const __nv_bfloat16 *>(src), reinterpret_cast<__nv_bfloat16 *>(dst), px,
                            oc));
    else if (dt == DVC_F16)
        DVC_CUDA(launch_pdl(slice_kernel<__half>, dim3(blocks), dim3(256), 0, s, 1,
                            reinterpret_cast<const __half *>(src), reinterpret_cast<__half *>(dst), px, oc));
    else
        DVC_CUDA(launch_pdl(slice_kernel<float>, dim3(blocks), dim3(256), 0, s, 1, reinterpret_cast<const float *>(src),
                            reinterpret_cast<float *>(dst), px, oc));
    ++g_launches;
    return DVC_OK;
}

}  // namespace

extern "C" {

dvc_status dvc_vae_weight_count(const dvc_vae_config *cfg, size_t *elems) {
    dvc_status st = vvalidate(cfg);
    if (st != DVC_OK) return st;
    DVC_CHECK_ARG(elems, DVC_ERR_ARG, "null elems");
    dvc_vae tmp;
    tmp.cfg = *cfg;
    size_t n = 0;
    vwalk(tmp, [&](size_t e) -> const void * {
        n += e;
        return nullptr;
    });
    *elems = n;
    return DVC_OK;
}

dvc_status dvc_vae_create(const dvc_vae_config *cfg, const void *host_weights, size_t bytes, dvc_vae **out) {
    dvc_status st = vvalidate(cfg);
    if (st != DVC_OK) return st;
    DVC_CHECK_ARG(host_weights && out, DVC_ERR_ARG, "null argument");
    if ((st = check_device()) != DVC_OK) return st;
    size_t elems = 0;
    dvc_vae_weight_count(cfg, &elems);
    const size_t es = dt_size(cfg->dt);
    DVC_CHECK_ARG(bytes == elems * es, DVC_ERR_SHAPE, "weight blob has %zu bytes, config expects %zu", bytes,
                  elems * es);
    dvc_vae *v = new dvc_vae();
    v->cfg = *cfg;
    for (int l = 0; l < 4; ++l) {
        v->lh[l] = cfg->h << l;
        v->lw[l] = cfg->w << l;
    }
    size_t dev_bytes = 0;
    vwalk(*v, [&](size_t e) -> const void * {
        dev_bytes += (e * es + 255) & ~size_t(255);
        return nullptr;
    });
    const int C = cfg->width[3], W0 = cfg->width[0];
    const size_t extra = align256((size_t)16 * 9 * W0 * es) + align256(16 * es) + align256((size_t)3 * C * C * es) +
                         align256((size_t)3 * C * es);
    if (cudaMalloc(&v->dweights, dev_bytes) != cudaSuccess || cudaMalloc(&v->dextra, extra) != cudaSuccess) {
        cudaFree(v->dweights);
        delete v;
        set_error("cudaMalloc of VAE weights failed");
        return DVC_ERR_CUDA;
    }
    size_t src_off = 0, dst_off = 0;
    cudaError_t err = cudaSuccess;
    vwalk(*v, [&](size_t e) -> const void * {
        uint8_t *dst = reinterpret_cast<uint8_t *>(v->dweights) + dst_off;
        if (err == cudaSuccess)
            err = cudaMemcpy(dst, reinterpret_cast<const uint8_t *>(host_weights) + src_off, e * es,
                             cudaMemcpyHostToDevice);
        src_off += e * es;
        dst_off += (e * es + 255) & ~size_t(255);
        return dst;
    });
    // conv_out padded to 16 output channels (zero rows), q|k|v concatenated
    uint8_t *x = reinterpret_cast<uint8_t *>(v->dextra);
    void *w16 = x, *b16 = x + align256((size_t)16 * 9 * W0 * es);
    v->qkv_w = reinterpret_cast<uint8_t *>(b16) + align256(16 * es);
    v->qkv_b = reinterpret_cast<uint8_t *>(v->qkv_w) + align256((size_t)3 * C * C * es);
    if (err == cudaSuccess) err = cudaMemset(v->dextra, 0, extra);
    const size_t oc = cfg->out_ch;
    if (err == cudaSuccess) err = cudaMemcpy(w16, v->conv_out16.w, oc * 9 * W0 * es, cudaMemcpyDeviceToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(b16, v->conv_out16.b, oc * es, cudaMemcpyDeviceToDevice);
    if (cfg->mid_attn)
        for (int i = 0; i < 3 && err == cudaSuccess; ++i) {
            err = cudaMemcpy(reinterpret_cast<uint8_t *>(v->qkv_w) + (size_t)i * C * C * es, v->at_q[2 * i],
                             (size_t)C * C * es, cudaMemcpyDeviceToDevice);
            if (err == cudaSuccess)
                err = cudaMemcpy(reinterpret_cast<uint8_t *>(v->qkv_b) + (size_t)i * C * es, v->at_q[2 * i + 1],
                                 (size_t)C * es, cudaMemcpyDeviceToDevice);
        }
    v->conv_out16.w = w16;
    v->conv_out16.b = b16;
    if (err != cudaSuccess) {
        cudaFree(v->dweights);
        cudaFree(v->dextra);
        delete v;
        set_error("VAE weight upload failed: %s", cudaGetErrorString(err));
        return DVC_ERR_CUDA;
    }
    for (int b = 0; b < kVBlocks; ++b) {
        const int l = v->blevel[b];
        if ((st = resblock_validate(v->blk[b], 1, v->lh[l], v->lw[l])) != DVC_OK) {
            cudaFree(v->dweights);
            cudaFree(v->dextra);
            delete v;
            return st;
        }
    }
    *out = v;
    return DVC_OK;
}

const dvc_vae_config *dvc_vae_get_config(const dvc_vae *v) { return v ? &v->cfg : nullptr; }

dvc_status dvc_vae_destroy(dvc_vae *v) {
    if (!v) return DVC_OK;
    cudaFree(v->dweights);
    cudaFree(v->dextra);
    delete v;
    return DVC_OK;
}

dvc_status dvc_vae_workspace_size(const dvc_vae *v, int T, size_t *bytes) {
    DVC_CHECK_ARG(v && bytes && T >= 1 && T <= v->cfg.max_T, DVC_ERR_ARG, "bad arguments (1 <= T <= max_T)");
    size_t offs[kVRegions];
    *bytes = vplan(*v, T, offs);
    return DVC_OK;
}

dvc_status dvc_vae_decode(dvc_vae *v, const void *lat, int T, void *frames, void *workspace, size_t ws_bytes,
                          void *stream) {
    NvtxRange nv("dvc_vae_decode T=%d", T);
    DVC_CHECK_ARG(v && lat && frames && workspace, DVC_ERR_ARG, "null argument");
    DVC_CHECK_ARG(T >= 1 && T <= v->cfg.max_T, DVC_ERR_ARG, "T=%d outside [1, max_T=%d]", T, v->cfg.max_T);
    DVC_CHECK_ARG(((uintptr_t)workspace & 255) == 0, DVC_ERR_ARG, "workspace must be 256-byte aligned");
    size_t offs[kVRegions];
    const size_t need = vplan(*v, T, offs);
    DVC_CHECK_ARG(ws_bytes >= need, DVC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const dvc_vae_config &c = v->cfg;
    const dvc_dtype dt = c.dt;
    const size_t es = dt_size(dt);
    uint8_t *ws = reinterpret_cast<uint8_t *>(workspace);
    void *buf[2] = {ws + offs[0], ws + offs[1]};
    void *bst[2] = {ws + offs[4], ws + offs[5]};
    void *scr = ws + offs[2], *rbws = ws + offs[3], *pad = ws + offs[6];
    auto conv3 = [&](const void *src, int cin, int H, int W, const VConv &cw, int cout, void *dst, void *stats) {
        ConvDesc d{};
        d.seg[0] = ConvSeg{src, cin, SEG_SAME, H, W, 9, cw.w, 9 * cin, 0, cin};
        d.nseg = 1;
        d.T = T;
        d.ho = H;
        d.wo = W;
        d.cout = cout;
        d.bias0 = cw.b;
        d.out = dst;
        d.stats_out = stats;
        d.dt = dt;
        return conv_run(d, s);
    };
    const int top = c.width[3];
    int cur = 0;   // buf index holding x
    if ((st = conv3(lat, c.c_lat, v->lh[0], v->lw[0], v->conv_in, top, buf[0], bst[0])) != DVC_OK) return st;
    int bi = 0;
    auto block = [&]() -> dvc_status {
        const RB &r = v->blk[bi];
        const int l = v->blevel[bi++];
        dvc_status e = resblock_launch(r, buf[cur], nullptr, T, v->lh[l], v->lw[l], nullptr, nullptr, buf[cur ^ 1],
                                       rbws, s, bst[cur], nullptr, bst[cur ^ 1]);
        cur ^= 1;
        return e;
    };
    // the last ResBlock of an up level writes the exact 2x nearest upsampling of its output straight into
    // the scratch the upsampler conv reads (no nearest kernel, no low-res copy)
    auto block_up2 = [&]() -> dvc_status {
        const RB &r = v->blk[bi];
        const int l = v->blevel[bi++];
        return resblock_launch(r, buf[cur], nullptr, T, v->lh[l], v->lw[l], nullptr, nullptr, scr, rbws, s, bst[cur],
                               nullptr, nullptr, 1);
    };
    if ((st = block()) != DVC_OK) return st;
    if (c.mid_attn) {
        // x += out(softmax(q k^T / sqrt C) v), q|k|v = GN(x) W_qkv^T + b (single head, head_dim = C)
        const int H = v->lh[0], W = v->lw[0], N = H * W;
        const size_t px = (size_t)T * N;
        uint8_t *p = reinterpret_cast<uint8_t *>(scr);
        void *a = p;
        p += align256(px * top * es);
        void *qkv = p;
        p += align256(px * 3 * top * es);
        void *o = p;
        p += align256(px * top * es);
        void *aws = p;
        p += attn_ws_bytes(T, N, top, dt);
        void *coef = p;
        NormArgs na{buf[cur], nullptr, nullptr, top, 0, 0, T, N, c.groups, c.eps, v->at_gn_w, v->at_gn_b, coef, nullptr};
        if ((st = gn_coef_box_run(na, BoxStatsIn{bst[cur], nullptr, nullptr}, H, W, dt, s)) != DVC_OK) return st;
        if ((st = gn_affine_run(buf[cur], coef, T, N, top, dt, a, s)) != DVC_OK) return st;
        ConvDesc d{};
        d.seg[0] = ConvSeg{a, top, SEG_SAME, H, W, 1, v->qkv_w, top, 0, top};
        d.nseg = 1, d.T = T, d.ho = H, d.wo = W, d.cout = 3 * top, d.bias0 = v->qkv_b, d.out = qkv, d.dt = dt;
        if ((st = conv_run(d, s)) != DVC_OK) return st;
        if ((st = attention_run(qkv, T, N, top, top, dt, aws, o, s)) != DVC_OK) return st;
        ConvDesc e{};
        e.seg[0] = ConvSeg{o, top, SEG_SAME, H, W, 1, v->at_out_w, top, 0, top};
        e.nseg = 1, e.T = T, e.ho = H, e.wo = W, e.cout = top, e.bias0 = v->at_out_b, e.residual = buf[cur];
        e.out = buf[cur], e.stats_out = bst[cur], e.dt = dt;   // in place: each tile reads its own residual
        if ((st = conv_run(e, s)) != DVC_OK) return st;
    }
    if ((st = block()) != DVC_OK) return st;
    int ch = top;
    for (int i = 0; i < 4; ++i) {
        const bool fold = i < 3 && v->lh[i + 1] == 2 * v->lh[i] && v->lw[i + 1] == 2 * v->lw[i];
        for (int r = 0; r < 3; ++r)
            if ((st = (fold && r == 2) ? block_up2() : block()) != DVC_OK) return st;
        ch = c.width[3 - i];
        if (i < 3) {
            // nearest 2x (exact copy; folded into the block above when the sizes double) then 3x3
            if (!fold &&
                (st = nearest_run(buf[cur], scr, T, v->lh[i], v->lw[i], v->lh[i + 1], v->lw[i + 1], ch, dt, s)) !=
                    DVC_OK)
                return st;
            if ((st = conv3(scr, ch, v->lh[i + 1], v->lw[i + 1], v->us[i], ch, buf[cur ^ 1], bst[cur ^ 1])) != DVC_OK)
                return st;
            cur ^= 1;
        }
    }
    // out = conv_out(SiLU(GN_out(x))): GN-apply + SiLU fused into conv_out's operand producer when
    // the fused engine applies, else materialised; 16-channel tile, then the out_ch slice
    const int H = v->lh[3], W = v->lw[3];
    if (conv_out_applicable(ch, c.out_ch, dt)) {   // streaming output head, straight into the frames
        float2 *coef = reinterpret_cast<float2 *>(rbws);
        NormArgs na{buf[cur], nullptr, nullptr, ch, 0, 0, T, H * W, c.groups, c.eps, v->gno_w, v->gno_b, coef, nullptr};
        if ((st = gn_coef_box_run(na, BoxStatsIn{bst[cur], nullptr, nullptr}, H, W, dt, s)) != DVC_OK) return st;
        ConvDesc prof{};
        prof.seg[0] = ConvSeg{buf[cur], ch, SEG_SAME, H, W, 9, v->conv_out16.w, 9 * ch, 0, ch};
        prof.nseg = 1, prof.T = T, prof.ho = H, prof.wo = W, prof.cout = c.out_ch;
        ProfSlot slot = prof_begin(s);
        st = conv_out_run(buf[cur], coef, T, H, W, ch, v->conv_out16.w, v->conv_out16.b, c.out_ch, frames, dt, s);
        prof_end(slot, s, conv_flops(prof), "conv_out", prof);
        return st;
    }
    if (conv_fz_applicable(H, W, dt)) {
        float2 *coef = reinterpret_cast<float2 *>(rbws);
        NormArgs na{buf[cur], nullptr, nullptr, ch, 0, 0, T, H * W, c.groups, c.eps, v->gno_w, v->gno_b, coef, nullptr};
        if ((st = gn_coef_box_run(na, BoxStatsIn{bst[cur], nullptr, nullptr}, H, W, dt, s)) != DVC_OK) return st;
        FzDesc f{};
        f.seg[0] = FzDesc::Seg{buf[cur], ch, 0, 9, 1, 0, v->conv_out16.w, 9 * ch, 0, ch, 0};
        f.nseg = 1;
        f.T = T;
        f.H = H;
        f.W = W;
        f.cout = 16;
        f.coef = coef;
        f.cop = ch;
        f.bias0 = v->conv_out16.b;
        f.out = pad;
        f.dt = dt;
        ConvDesc prof{};
        prof.seg[0] = ConvSeg{buf[cur], ch, SEG_SAME, H, W, 9, v->conv_out16.w, 9 * ch, 0, ch};
        prof.nseg = 1, prof.T = T, prof.ho = H, prof.wo = W, prof.cout = c.out_ch;
        ProfSlot slot = prof_begin(s);
        st = conv_fz_run(f, s);
        prof_end(slot, s, conv_flops(prof), "fz_out", prof);
        if (st != DVC_OK) return st;
    } else {
        uint8_t *gnws = reinterpret_cast<uint8_t *>(rbws);
        void *op = scr;
        NormArgs na{buf[cur], nullptr, nullptr, ch, 0, 0, T, H * W, c.groups, c.eps, v->gno_w, v->gno_b, op, gnws};
        if ((st = gn_silu_box_run(na, BoxStatsIn{bst[cur], nullptr, nullptr}, H, W, dt, s)) != DVC_OK) return st;
        if ((st = conv3(op, ch, H, W, v->conv_out16, 16, pad, nullptr)) != DVC_OK) return st;
    }
    return slice_run(pad, frames, (long)T * H * W, c.out_ch, dt, s);
}

}  // extern "C"
