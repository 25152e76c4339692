// dvc_unet.cu -- a9/a10/e: the pruned U-Net ResBlock skeleton over a group of
// frames (reading R1, R11) and the multi-GPU halo.
//
// Topology (the product's own statement of reading R1; SD-2.1-base U-Net with
// widths x0.75, 2 ResBlocks per down level, 3 per up level, 2 mid):
//   conv_in(concat(Lbar, Cm)) -> x0 (push)
//   level l = 0..3: 2 ResBlocks (push each); l < 3: 3x3 stride-2 conv (push)
//   mid: 2 ResBlocks
//   up u = 0..3 (level 3-u): 3 ResBlocks on concat(h, pop()); u < 3: nearest
//   resize to the next skip's size + 3x3 conv
//   out = conv_out(SiLU(GN_out(h)))
// Multi-GPU: a chain's frames are split into contiguous chunks, one
// per rank; before ResBlock k, rank r sends the C_in/P-channel slice of its
// last frame's block input to rank r+1 and receives rank r-1's (dvc_halo.cu:
// copy-engine peer copies + stream memory flags, or NCCL, on a comm stream).
// Weights are replicated.
#include <cstring>
#include <cstdlib>
#include <vector>
#include "dvc_conv.cuh"
#include "dvc_norm.cuh"
#include "dvc_resblock.cuh"
#include "dvc_attn.cuh"
#include "dvc_halo.cuh"

using namespace dvc;

// ----------------------------------------------------------------- the network
struct ConvW {
    const void *w, *b;
    const void *pk = nullptr;   // packed image (dvc_pack.cu) for the TMA engines, or null
};

struct dvc_unet {
    dvc_unet_config cfg;
    void *dweights = nullptr;
    void *dpacked = nullptr;   // packed weight images (16-bit configs)
    void *dff1i = nullptr;     // f1: FF1 weights / biases interleaved for the GEGLU epilogue
    size_t welems = 0;
    ConvW conv_in, ds[3], us[3], conv_out;
    const void *gno_w = nullptr, *gno_b = nullptr;
    RB blk[22];
    int blevel[22];
    TF tf[16];      // f1: Transformer2D blocks (cfg.head_dim > 0)
    int tf_of[22];  // index into tf of the block following ResBlock b, or -1
    int ntf = 0;
    int lh[4], lw[4];
    size_t carry_off[22];
    size_t carry_total = 0;
};

namespace {

// Walks the topology; for every tensor calls take(elements) which returns its
// device pointer.  Also fills the block table.
template <typename Take>
void walk(dvc_unet &n, Take take) {
    const dvc_unet_config &c = n.cfg;
    const int *W = c.width;
    auto conv = [&](int cout, int cin, int k) {
        ConvW cw;
        cw.w = take((size_t)cout * k * k * cin);
        cw.b = take((size_t)cout);
        return cw;
    };
    int bi = 0;
    auto block = [&](int cin, int cout, int level, int cb) {
        RB &r = n.blk[bi];
        r.ca = cin - cb;
        r.cb = cb;
        r.cout = cout;
        r.G = c.groups;
        r.P = c.shift_p;
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
        n.blevel[bi] = level;
        n.tf_of[bi] = -1;
        ++bi;
    };
    // f1 (R26): a Transformer2D block after the ResBlock just walked; tensors follow its weights
    n.ntf = 0;
    auto tfb = [&](int C) {
        if (c.head_dim <= 0) return;
        TF &t = n.tf[n.ntf];
        t.c = C;
        t.groups = c.groups;
        t.head_dim = c.head_dim;
        t.eps_gn = 1e-6f;
        t.eps_ln = 1e-5f;
        t.dt = c.dt;
        t.gn_w = take(C);
        t.gn_b = take(C);
        t.proj_in_w = take((size_t)C * C);
        t.proj_in_b = take(C);
        t.ln1_w = take(C);
        t.ln1_b = take(C);
        t.qkv_w = take((size_t)3 * C * C);
        t.out_w = take((size_t)C * C);
        t.out_b = take(C);
        t.ln2_w = take(C);
        t.ln2_b = take(C);
        t.ff1_w = take((size_t)8 * C * C);
        t.ff1_b = take((size_t)8 * C);
        t.ff2_w = take((size_t)4 * C * C);
        t.ff2_b = take(C);
        t.proj_out_w = take((size_t)C * C);
        t.proj_out_b = take(C);
        n.tf_of[bi - 1] = n.ntf++;
    };
    n.conv_in = conv(W[0], c.c_lat + c.c_ctx, 3);
    std::vector<int> skips{W[0]};
    int cur = W[0];
    for (int l = 0; l < 4; ++l) {
        for (int r = 0; r < 2; ++r) {
            block(cur, W[l], l, 0);
            cur = W[l];
            if (l < 3) tfb(cur);
            skips.push_back(cur);
        }
        if (l < 3) {
            n.ds[l] = conv(cur, cur, 3);
            skips.push_back(cur);
        }
    }
    for (int r = 0; r < 2; ++r) {
        block(cur, cur, 3, 0);
        if (r == 0) tfb(cur);
    }
    for (int u = 0; u < 4; ++u) {
        const int l = 3 - u;
        for (int r = 0; r < 3; ++r) {
            const int sk = skips.back();
            skips.pop_back();
            block(cur + sk, W[l], l, sk);
            cur = W[l];
            if (u > 0) tfb(cur);
        }
        if (u < 3) n.us[u] = conv(cur, cur, 3);
    }
    n.gno_w = take(cur);
    n.gno_b = take(cur);
    n.conv_out = conv(c.c_lat, cur, 3);
}

dvc_status validate_cfg(const dvc_unet_config *c) {
    DVC_CHECK_ARG(c, DVC_ERR_ARG, "null config");
    DVC_CHECK_ARG(dt_valid(c->dt), DVC_ERR_ARG, "bad dtype");
    DVC_CHECK_ARG(c->h >= 8 && c->w >= 8 && c->max_T >= 1 && c->max_T < 256, DVC_ERR_ARG,
                  "latent size >= 8x8 and 1 <= max_T < 256 required");
    DVC_CHECK_ARG(c->groups >= 1 && c->shift_p >= 1 && c->c_lat > 0 && c->c_ctx > 0, DVC_ERR_ARG, "bad config");
    for (int i = 0; i < 4; ++i) DVC_CHECK_ARG(c->width[i] > 0, DVC_ERR_ARG, "bad width");
    DVC_CHECK_ARG(c->head_dim == 0 || c->head_dim == 16 || c->head_dim == 32 || c->head_dim == 48 || c->head_dim == 64,
                  DVC_ERR_UNSUPPORTED, "head_dim must be 0 (attention elided) or 16/32/48/64");
    return DVC_OK;
}

// Workspace regions: 0..11 skips, 12/13 ping-pong h, 14 ResBlock scratch (also the
// GN_out operand and the nearest-resize operand), 15 halo send/recv, 16..27 box
// statistics of the skips, 28/29 box statistics of the ping-pong buffers.
constexpr int kRegions = 30;

size_t plan_workspace(const dvc_unet &n, int T, size_t *offs /* kRegions */) {
    const dvc_unet_config &c = n.cfg;
    const size_t es = dt_size(c.dt);
    const int *W = c.width;
    size_t sz[kRegions] = {};
    auto hw = [&](int l) { return (size_t)n.lh[l] * n.lw[l]; };
    auto bst = [&](int l, int C) { return box_stats_bytes(T, n.lh[l], n.lw[l], C); };
    int k = 0;
    sz[k] = T * hw(0) * W[0] * es;
    sz[16 + k++] = bst(0, W[0]);
    for (int l = 0; l < 4; ++l) {
        for (int r = 0; r < 2; ++r) {
            sz[k] = T * hw(l) * W[l] * es;
            sz[16 + k++] = bst(l, W[l]);
        }
        if (l < 3) {
            sz[k] = T * hw(l + 1) * W[l] * es;
            sz[16 + k++] = bst(l + 1, W[l]);
        }
    }
    size_t hmax = 0, smax = 0;
    for (int l = 0; l < 4; ++l) {
        hmax = std::max(hmax, T * hw(l) * (size_t)W[l]);
        smax = std::max(smax, bst(l, W[l]));
    }
    for (int l = 1; l < 4; ++l) {
        hmax = std::max(hmax, T * hw(l - 1) * (size_t)W[l]);
        smax = std::max(smax, bst(l - 1, W[l]));
    }
    hmax = std::max(hmax, T * hw(0) * (size_t)c.c_lat);
    sz[12] = sz[13] = hmax * es;
    sz[28] = sz[29] = smax;
    size_t rbws = 0;
    for (int b = 0; b < 22; ++b) {
        const RB &r = n.blk[b];
        const int l = n.blevel[b];
        rbws = std::max(rbws, resblock_ws_bytes(r.ca, r.cb, r.cout, r.G, T, n.lh[l], n.lw[l], c.dt));
    }
    rbws = std::max(rbws, align256(gn_workspace_bytes(T, (int)hw(0), c.groups, W[0])) + T * hw(0) * W[0] * es);
    for (int l = 1; l < 4; ++l) rbws = std::max(rbws, T * hw(l - 1) * (size_t)W[l] * es);
    if (c.head_dim > 0)
        for (int l = 0; l < 4; ++l) rbws = std::max(rbws, transformer_ws_bytes(W[l], T, n.lh[l], n.lw[l], c.dt));
    sz[14] = rbws;
    sz[15] = (n.carry_total * 2 + 2 * hw(0) * 2048) * es;
    size_t total = 0;
    for (int i = 0; i < kRegions; ++i) {
        offs[i] = total;
        total += align256(sz[i]);
    }
    return total;
}

// Packed K-chunk-major weight images for every same-resolution conv (TMA engines): one
// contiguous block per (tap, 64-channel chunk) weight tile.  Multi-segment convs (concat
// inputs) pack segment a's rows then segment b's rows in one block.
dvc_status pack_all(dvc_unet &n) {
    const dvc_unet_config &c = n.cfg;
    const size_t es = dt_size(c.dt);
    struct Job {
        const void *w;
        int cout, taps, cin, off, cs;
        const void **dst;
        size_t base;   // element offset of this segment inside its block
        size_t block;  // element offset of the block
    };
    std::vector<Job> jobs;
    size_t total = 0;
    auto add = [&](const void *w, int cout, int taps, int ca, int cb, const void **dst) {
        const size_t a = packed_elems(cout, taps, ca);
        const size_t blk = total;
        jobs.push_back(Job{w, cout, taps, ca + cb, 0, ca, dst, 0, blk});
        if (cb > 0) jobs.push_back(Job{w, cout, taps, ca + cb, ca, cb, nullptr, a, blk});
        total += a + (cb > 0 ? packed_elems(cout, taps, cb) : 0);
        total = (total + 127) & ~size_t(127);   // 256-byte aligned blocks
    };
    const int *W = c.width;
    add(n.conv_in.w, W[0], 9, c.c_lat, c.c_ctx, &n.conv_in.pk);
    for (int b = 0; b < 22; ++b) {
        RB &r = n.blk[b];
        add(r.conv1_w, r.cout, 9, r.ca, r.cb, &r.conv1_pk);
        add(r.conv2_w, r.cout, 9, r.cout, 0, &r.conv2_pk);
        if (r.sc_w) add(r.sc_w, r.cout, 1, r.ca, r.cb, &r.sc_pk);
    }
    for (int u = 0; u < 3; ++u) add(n.us[u].w, W[3 - u], 9, W[3 - u], 0, &n.us[u].pk);
    add(n.conv_out.w, c.c_lat, 9, W[0], 0, &n.conv_out.pk);
    if (cudaMalloc(&n.dpacked, total * es) != cudaSuccess) {
        set_error("cudaMalloc of %zu packed weight bytes failed", total * es);
        return DVC_ERR_CUDA;
    }
    uint8_t *base = reinterpret_cast<uint8_t *>(n.dpacked);
    for (const Job &j : jobs) {
        void *dst = base + (j.block + j.base) * es;
        dvc_status st = pack_weights_run(j.w, c.dt, j.cout, j.taps, j.cin, j.off, j.cs, dst, 0);
        if (st != DVC_OK) return st;
        if (j.dst) *j.dst = base + j.block * es;
    }
    DVC_CUDA(cudaDeviceSynchronize());
    return DVC_OK;
}

}  // namespace

extern "C" {

dvc_status dvc_unet_weight_count(const dvc_unet_config *cfg, size_t *elems) {
    dvc_status st = validate_cfg(cfg);
    if (st != DVC_OK) return st;
    DVC_CHECK_ARG(elems, DVC_ERR_ARG, "null elems");
    dvc_unet tmp;
    tmp.cfg = *cfg;
    size_t n = 0;
    walk(tmp, [&](size_t e) -> const void * {
        n += e;
        return nullptr;
    });
    *elems = n;
    return DVC_OK;
}

dvc_status dvc_unet_create(const dvc_unet_config *cfg, const void *host_weights, size_t bytes, dvc_unet **out) {
    dvc_status st = validate_cfg(cfg);
    if (st != DVC_OK) return st;
    DVC_CHECK_ARG(host_weights && out, DVC_ERR_ARG, "null argument");
    if ((st = check_device()) != DVC_OK) return st;
    size_t elems = 0;
    dvc_unet_weight_count(cfg, &elems);
    const size_t es = dt_size(cfg->dt);
    DVC_CHECK_ARG(bytes == elems * es, DVC_ERR_SHAPE, "weight blob has %zu bytes, config expects %zu", bytes,
                  elems * es);
    dvc_unet *n = new dvc_unet();
    n->cfg = *cfg;
    n->lh[0] = cfg->h;
    n->lw[0] = cfg->w;
    for (int l = 1; l < 4; ++l) {   // 3x3 stride 2 pad 1: ceil halving (R11)
        n->lh[l] = (n->lh[l - 1] - 1) / 2 + 1;
        n->lw[l] = (n->lw[l - 1] - 1) / 2 + 1;
    }
    // each tensor gets a 16-byte aligned slot in one device allocation
    size_t dev_bytes = 0;
    walk(*n, [&](size_t e) -> const void * {
        dev_bytes += (e * es + 255) & ~size_t(255);
        return nullptr;
    });
    if (cudaMalloc(&n->dweights, dev_bytes) != cudaSuccess) {
        delete n;
        set_error("cudaMalloc of %zu weight bytes failed", dev_bytes);
        return DVC_ERR_CUDA;
    }
    size_t src_off = 0, dst_off = 0;
    cudaError_t err = cudaSuccess;
    walk(*n, [&](size_t e) -> const void * {
        uint8_t *dst = reinterpret_cast<uint8_t *>(n->dweights) + dst_off;
        if (err == cudaSuccess)
            err = cudaMemcpy(dst, reinterpret_cast<const uint8_t *>(host_weights) + src_off, e * es,
                             cudaMemcpyHostToDevice);
        src_off += e * es;
        dst_off += (e * es + 255) & ~size_t(255);
        return dst;
    });
    if (err != cudaSuccess) {
        cudaFree(n->dweights);
        delete n;
        set_error("weight upload failed: %s", cudaGetErrorString(err));
        return DVC_ERR_CUDA;
    }
    for (int b = 0; b < 22; ++b) {
        const RB &r = n->blk[b];
        const int l = n->blevel[b];
        st = resblock_validate(r, 1, n->lh[l], n->lw[l]);
        if (st != DVC_OK) {
            cudaFree(n->dweights);
            delete n;
            return st;
        }
        if (n->tf_of[b] >= 0 && (st = transformer_validate(n->tf[n->tf_of[b]], 1, n->lh[l], n->lw[l])) != DVC_OK) {
            cudaFree(n->dweights);
            delete n;
            return st;
        }
        n->carry_off[b] = n->carry_total;
        n->carry_total += (size_t)n->lh[l] * n->lw[l] * ((r.ca + r.cb) / r.P);
    }
    n->welems = elems;
    if (cfg->head_dim > 0 && cfg->dt != DVC_F32 && g_ws_cg != 0) {
        // f1: FF1 rows interleaved once for the GEGLU epilogue (16 value + 16 gate rows per block)
        size_t tot = 0;
        for (int i = 0; i < n->ntf; ++i) tot += align256((size_t)8 * n->tf[i].c * n->tf[i].c * es) +
                                               align256((size_t)8 * n->tf[i].c * es);
        if (cudaMalloc(&n->dff1i, tot) != cudaSuccess) {
            cudaFree(n->dweights);
            delete n;
            set_error("cudaMalloc of %zu interleaved FF1 bytes failed", tot);
            return DVC_ERR_CUDA;
        }
        uint8_t *q = reinterpret_cast<uint8_t *>(n->dff1i);
        for (int i = 0; i < n->ntf && st == DVC_OK; ++i) {
            TF &t = n->tf[i];
            void *wi = q, *bi = q + align256((size_t)8 * t.c * t.c * es);
            q += align256((size_t)8 * t.c * t.c * es) + align256((size_t)8 * t.c * es);
            st = interleave_ff1(t, wi, bi, 0);
            t.ff1_wi = wi, t.ff1_bi = bi;
        }
        if (st == DVC_OK && cudaDeviceSynchronize() != cudaSuccess) st = DVC_ERR_CUDA;
        if (st != DVC_OK) {
            cudaFree(n->dweights);
            cudaFree(n->dff1i);
            delete n;
            return st;
        }
    }
    // Packed weight images (contiguous weight tiles) measured slower than the OHWI rows on B200
    // (r1 profiles), so they are opt-in: DVC_PACK_WEIGHTS=1.
    const char *pe = dvc_knob("DVC_PACK_WEIGHTS");
    if (cfg->dt != DVC_F32 && pe && pe[0] == '1') {
        st = pack_all(*n);
        if (st != DVC_OK) {
            cudaFree(n->dweights);
            cudaFree(n->dpacked);
            delete n;
            return st;
        }
    }
    *out = n;
    return DVC_OK;
}

dvc_status dvc_unet_destroy(dvc_unet *n) {
    if (!n) return DVC_OK;
    cudaFree(n->dweights);
    cudaFree(n->dpacked);
    cudaFree(n->dff1i);
    delete n;
    return DVC_OK;
}

const dvc_unet_config *dvc_unet_get_config(const dvc_unet *n) { return n ? &n->cfg : nullptr; }

dvc_status dvc_unet_carry_size(const dvc_unet *n, size_t *elems) {
    DVC_CHECK_ARG(n && elems, DVC_ERR_ARG, "null argument");
    *elems = n->carry_total;
    return DVC_OK;
}

dvc_status dvc_unet_workspace_size(const dvc_unet *n, int T, size_t *bytes) {
    DVC_CHECK_ARG(n && bytes && T >= 1 && T <= n->cfg.max_T, DVC_ERR_ARG, "bad arguments (1 <= T <= max_T)");
    size_t offs[kRegions];
    *bytes = plan_workspace(*n, T, offs);
    return DVC_OK;
}

dvc_status dvc_unet_decode_gop(dvc_unet *n, dvc_comm *comm, const void *lat, const void *ctx, int T,
                               const void *carry_in, void *carry_out, void *out, void *workspace, size_t ws_bytes,
                               void *stream) {
    NvtxRange nv("dvc_unet_decode_gop T=%d", T);
    DVC_CHECK_ARG(n && lat && ctx && out && workspace, DVC_ERR_ARG, "null argument");
    DVC_CHECK_ARG(T >= 1 && T <= n->cfg.max_T, DVC_ERR_ARG, "T_local=%d outside [1, max_T=%d]", T, n->cfg.max_T);
    DVC_CHECK_ARG(((uintptr_t)workspace & 255) == 0, DVC_ERR_ARG, "workspace must be 256-byte aligned");
    size_t offs[kRegions];
    const size_t need = plan_workspace(*n, T, offs);
    DVC_CHECK_ARG(ws_bytes >= need, DVC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    const int world = comm_world(comm), rank = comm_rank(comm);
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const dvc_unet_config &c = n->cfg;
    const dvc_dtype dt = c.dt;
    const size_t es = dt_size(dt);
    const int *W = c.width;
    uint8_t *ws = reinterpret_cast<uint8_t *>(workspace);
    void *skip[12], *skst[12];
    for (int i = 0; i < 12; ++i) {
        skip[i] = ws + offs[i];
        skst[i] = ws + offs[16 + i];
    }
    void *hb[2] = {ws + offs[12], ws + offs[13]};
    void *hbst[2] = {ws + offs[28], ws + offs[29]};
    void *rbws = ws + offs[14];
    if (world > 1 && (st = halo_call_begin(comm, n->carry_total * es, ws + offs[15], s)) != DVC_OK) return st;
    (void)rank;
    auto hw = [&](int l) { return n->lh[l] * n->lw[l]; };

    int bi = 0;
    // one ResBlock with its halo exchange; sa/sb/sy: box statistics of x_a, x_b, y
    // up2: y receives the exact 2x nearest upsampling of the block output (no statistics, no
    // Transformer2D after the block)
    auto run_block = [&](const void *xa, const void *xb, void *y, const void *sa, const void *sb, void *sy,
                         int up2 = 0, int up_ho = 0, int up_wo = 0) -> dvc_status {
        const RB &r = n->blk[bi];
        const int l = n->blevel[bi];
        const int H = n->lh[l], Wd = n->lw[l];
        NvtxRange nvb("block %02d level %d", bi, l);
        const int cs = (r.ca + r.cb) / r.P;
        const size_t off = n->carry_off[bi] * es;
        const void *cin_ptr = carry_in ? reinterpret_cast<const uint8_t *>(carry_in) + off : nullptr;
        if (world > 1) {   // rank > 0: the carry is rank-1's slice; rank < world-1: send mine onward
            const HaloSlice sl{reinterpret_cast<const uint8_t *>(xa) + (size_t)(T - 1) * H * Wd * r.ca * es,
                               (size_t)r.ca * es, (size_t)cs * es, (size_t)H * Wd, off};
            dvc_status e = halo_exchange(comm, bi, sl, s, &cin_ptr);
            if (e != DVC_OK) return e;
        }
        void *cout_ptr = nullptr;
        if (carry_out && rank == world - 1) cout_ptr = reinterpret_cast<uint8_t *>(carry_out) + off;
        if (up2 && n->tf_of[bi] >= 0) {
            set_error("internal: upsampled block output before a Transformer2D block");
            return DVC_ERR_UNSUPPORTED;
        }
        dvc_status e = resblock_launch(r, xa, xb, T, H, Wd, cin_ptr, cout_ptr, y, rbws, s, sa, sb, up2 ? nullptr : sy,
                                       up2, up_ho, up_wo);
        // f1: the Transformer2D block after this ResBlock, in place on y (its statistics refreshed)
        if (e == DVC_OK && n->tf_of[bi] >= 0)
            e = transformer_launch(n->tf[n->tf_of[bi]], y, T, H, Wd, y, rbws, s, sy, sy);
        if (e == DVC_OK && world > 1) e = halo_block_done(comm, bi, s);
        ++bi;
        return e;
    };
    auto conv3 = [&](const void *src, int cin, int mode, int hi, int wi, const ConvW &cw, int cout, int ho, int wo,
                     void *dst, void *dst_stats) {
        ConvDesc d{};
        if (mode == SEG_SAME && cw.pk && conv_ws_applicable_dims(dt))
            d.seg[0] = ConvSeg{src, cin, mode, hi, wi, 9, cw.pk, 64, 0, 0, 1};
        else
            d.seg[0] = ConvSeg{src, cin, mode, hi, wi, 9, cw.w, 9 * cin, 0, cin};
        d.nseg = 1;
        d.T = T;
        d.ho = ho;
        d.wo = wo;
        d.cout = cout;
        d.bias0 = cw.b;
        d.out = dst;
        d.stats_out = dst_stats;
        d.dt = dt;
        return conv_run(d, s);
    };

    // conv_in on concat(Lbar, Cm): two K segments, no materialised concat
    {
        ConvDesc d{};
        const int cc = c.c_lat + c.c_ctx;
        if (n->conv_in.pk && conv_ws_applicable_dims(dt)) {
            const int rows_a = 9 * ((c.c_lat + 63) / 64) * W[0];
            d.seg[0] = ConvSeg{lat, c.c_lat, SEG_SAME, n->lh[0], n->lw[0], 9, n->conv_in.pk, 64, 0, 0, 1};
            d.seg[1] = ConvSeg{ctx, c.c_ctx, SEG_SAME, n->lh[0], n->lw[0], 9, n->conv_in.pk, 64, rows_a, 0, 1};
        } else {
            d.seg[0] = ConvSeg{lat, c.c_lat, SEG_SAME, n->lh[0], n->lw[0], 9, n->conv_in.w, 9 * cc, 0, cc};
            d.seg[1] = ConvSeg{ctx, c.c_ctx, SEG_SAME, n->lh[0], n->lw[0], 9, n->conv_in.w, 9 * cc, c.c_lat, cc};
        }
        d.nseg = 2;
        d.T = T;
        d.ho = n->lh[0];
        d.wo = n->lw[0];
        d.cout = W[0];
        d.bias0 = n->conv_in.b;
        d.out = skip[0];
        d.stats_out = skst[0];
        d.dt = dt;
        if ((st = conv_run(d, s)) != DVC_OK) return st;
    }
    int k = 1;
    const void *h = skip[0];
    const void *hs = skst[0];
    for (int l = 0; l < 4; ++l) {
        for (int r = 0; r < 2; ++r) {
            if ((st = run_block(h, nullptr, skip[k], hs, nullptr, skst[k])) != DVC_OK) return st;
            h = skip[k];
            hs = skst[k++];
        }
        if (l < 3) {
            if ((st = conv3(h, W[l], SEG_STRIDE2, n->lh[l], n->lw[l], n->ds[l], W[l], n->lh[l + 1], n->lw[l + 1],
                            skip[k], skst[k])) != DVC_OK)
                return st;
            h = skip[k];
            hs = skst[k++];
        }
    }
    int pp = 0;
    for (int r = 0; r < 2; ++r) {
        if ((st = run_block(h, nullptr, hb[pp], hs, nullptr, hbst[pp])) != DVC_OK) return st;
        h = hb[pp];
        hs = hbst[pp];
        pp ^= 1;
    }
    for (int u = 0; u < 4; ++u) {
        const int l = 3 - u;
        // an upsampler to 2H (- 1) x 2W (- 1) -- every level of the U-Net (R11: nearest_to onto the skip's
        // size = the 2x phase replication clipped at the far edge; 720p: 12x20 -> 23x40 -> 45x80 -> 90x160)
        // with no Transformer2D after the level's last ResBlock: that block's conv2 epilogue writes the
        // upsampled tensor itself (no nearest kernel, no low-res copy); the hb buffers are sized for the
        // upsampled tensors
        const bool fold = u < 3 && g_ws_cg != 0 && c.head_dim == 0 &&
                          (n->lh[l - 1] == 2 * n->lh[l] || n->lh[l - 1] == 2 * n->lh[l] - 1) &&
                          (n->lw[l - 1] == 2 * n->lw[l] || n->lw[l - 1] == 2 * n->lw[l] - 1);
        for (int r = 0; r < 3; ++r) {
            --k;
            if ((st = run_block(h, skip[k], hb[pp], hs, skst[k], hbst[pp], fold && r == 2, fold ? n->lh[l - 1] : 0,
                                fold ? n->lw[l - 1] : 0)) != DVC_OK)
                return st;
            h = hb[pp];
            hs = hbst[pp];
            pp ^= 1;
        }
        if (u < 3) {
            void *nst = (u < 3) ? hbst[pp] : nullptr;
            if (fold) {   // h already holds nearest_to(block output, next skip size)
                st = conv3(h, W[l], SEG_SAME, n->lh[l - 1], n->lw[l - 1], n->us[u], W[l], n->lh[l - 1], n->lw[l - 1],
                           hb[pp], nst);
            } else if (g_ws_cg != 0) {
                // materialise nearest_to(h, next skip size) (exact copy) so the 3x3 conv runs on the TMA engine
                if ((st = nearest_run(h, rbws, T, n->lh[l], n->lw[l], n->lh[l - 1], n->lw[l - 1], W[l], dt, s)) !=
                    DVC_OK)
                    return st;
                st = conv3(rbws, W[l], SEG_SAME, n->lh[l - 1], n->lw[l - 1], n->us[u], W[l], n->lh[l - 1],
                           n->lw[l - 1], hb[pp], nst);
            } else {
                st = conv3(h, W[l], SEG_UPNEAREST, n->lh[l], n->lw[l], n->us[u], W[l], n->lh[l - 1], n->lw[l - 1],
                           hb[pp], nst);
            }
            if (st != DVC_OK) return st;
            h = hb[pp];
            hs = hbst[pp];
            pp ^= 1;
        }
    }
    // out = conv_out(SiLU(GN_out(h)))
    if (conv_fz_applicable(n->lh[0], n->lw[0], dt) && (W[0] / c.groups) > 0) {
        // fused: GN_out coefficients from h's box statistics, GN-apply + SiLU inside conv_out's
        // operand producer (no GN_out tensor in HBM)
        float2 *coef = reinterpret_cast<float2 *>(rbws);
        NormArgs na{h, nullptr, nullptr, W[0], 0, 0, T, hw(0), c.groups, c.eps, n->gno_w, n->gno_b, coef, nullptr};
        if ((st = gn_coef_box_run(na, BoxStatsIn{hs, nullptr, nullptr}, n->lh[0], n->lw[0], dt, s)) != DVC_OK)
            return st;
        FzDesc f{};
        if (n->conv_out.pk) f.seg[0] = FzDesc::Seg{h, W[0], 0, 9, 1, 0, n->conv_out.pk, 64, 0, 0, 1};
        else f.seg[0] = FzDesc::Seg{h, W[0], 0, 9, 1, 0, n->conv_out.w, 9 * W[0], 0, W[0], 0};
        f.nseg = 1;
        f.T = T;
        f.H = n->lh[0];
        f.W = n->lw[0];
        f.cout = c.c_lat;
        f.coef = coef;
        f.cop = W[0];
        f.bias0 = n->conv_out.b;
        f.out = out;
        f.dt = dt;
        ConvDesc prof{};
        prof.seg[0] = ConvSeg{h, W[0], SEG_SAME, n->lh[0], n->lw[0], 9, n->conv_out.w, 9 * W[0], 0, W[0]};
        prof.nseg = 1, prof.T = T, prof.ho = n->lh[0], prof.wo = n->lw[0], prof.cout = c.c_lat;
        ProfSlot slot = prof_begin(s);
        st = conv_fz_run(f, s);
        prof_end(slot, s, conv_flops(prof), "fz_out", prof);
        if (st != DVC_OK) return st;
    } else {
        uint8_t *gnws = reinterpret_cast<uint8_t *>(rbws);
        void *op = gnws + align256(gn_workspace_bytes(T, hw(0), c.groups, W[0]));
        NormArgs na{h, nullptr, nullptr, W[0], 0, 0, T, hw(0), c.groups, c.eps, n->gno_w, n->gno_b, op, gnws};
        if ((st = gn_silu_box_run(na, BoxStatsIn{hs, nullptr, nullptr}, n->lh[0], n->lw[0], dt, s)) != DVC_OK)
            return st;
        if ((st = conv3(op, W[0], SEG_SAME, n->lh[0], n->lw[0], n->conv_out, c.c_lat, n->lh[0], n->lw[0], out,
                        nullptr)) != DVC_OK)
            return st;
    }
    if (world > 1 && (st = halo_call_end(comm, s)) != DVC_OK) return st;
    return DVC_OK;
}

}  // extern "C"
