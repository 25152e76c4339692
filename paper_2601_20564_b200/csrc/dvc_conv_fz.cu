// dvc_conv_fz.cu -- tcgen05 implicit-GEMM 3x3 convolution whose A operand
// producer is fused with GroupNorm-apply + SiLU and the Batch-dimension
// temporal shift (SURVEY a3/a4/a5 and a6/a7/a8 in one kernel).
//
// Output tiles are 8-wide x 16-tall pixel boxes (128 MMA rows).  For every
// 64-channel chunk of the operand a producer warp TMA-loads the raw 10 x 18 halo
// of the box as eight 8-channel boxes {8, 10, 18} (no swizzle, out-of-bounds zero
// fill) -- each lands as one 180-row core-matrix column of a K-major UMMA tile --
// together with the chunk's 64 GN coefficients.  The transform warps then rewrite
// the tile in place (shared memory only, no global-load latency on their path):
//     H = SiLU(X * sc[t][c] + b[t][c])   (0 outside the frame: conv padding after
//                                          the transform, H3)
// The nine taps are nine UMMA descriptors into that one tile: row offset
// (1+dy)*10 + (1+dx), 8-row groups 160 B apart (one image row each) -- the halo
// is transformed once instead of nine times and no H tensor reaches HBM.
// The temporal shift is addressing of those TMA boxes: channels [0, C_in/P) of
// frame t come from frame t-1, from the carry at t = 0, or (no carry) from an
// out-of-bounds box = zeros; the one 8-channel group straddling C_in/P is merged
// from a side buffer.  The 1x1 shortcut segments (raw, unshifted X) are TMA'd as
// SW128 boxes straight into a slot (centre tap only).
//
// Warps (512 threads): 1 TMEM allocator + MMA issuer (leader CTA), 2 weight TMA
// producer, 3 operand-tile TMA producer, 4-7 epilogue (bias / 16-bit
// store / box statistics), 8-15 transform.  CTA pairs (cta_group::2, M=256),
// double-buffered TMEM accumulators, as in dvc_conv_ws.cu.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "dvc_conv.cuh"
#include "dvc_ptx.cuh"
#include "dvc_boxstats.cuh"
#include "dvc_epilogue.cuh"

namespace dvc {

constexpr int FZ_BX = 8, FZ_BY = 16;
constexpr int FZ_HX = FZ_BX + 2, FZ_HY = FZ_BY + 2;
constexpr int FZ_HROWS = FZ_HX * FZ_HY;      // 180 halo pixels
constexpr int FZ_COLB = FZ_HROWS * 16;        // one 8-channel halo column (TMA box bytes, 2880)
constexpr int FZ_LBO = 2944;                  // column stride: 2880 rounded up to the TMA's 128-B alignment
// tile slot: [8][FZ_LBO] halo tile | [FZ_LBO] shift side buffer | [64] float2 GN coefficients
constexpr int FZ_SIDE = 8 * FZ_LBO;           // 23552
constexpr int FZ_COEF = FZ_SIDE + FZ_LBO;     // 26496
constexpr int FZ_SLOT = 27648;                // 1024-aligned
constexpr int FZ_RAW_SLOT = 128 * 128;        // one raw SW128 box {64, 8, 16}
constexpr int FZ_SBO = FZ_HX * 16;            // between 8-row groups (image rows)
constexpr int FZ_MAX_BSTAGES = 24;
constexpr int FZ_MAX_NTF = 6;   // even: keeps the barrier block a multiple of 16 B
constexpr int FZ_MAX_RAW = 4;   // raw (1x1) ring slots
#ifndef FZ_TFW
#define FZ_TFW 8   // transform warps: 8 (one per 8-channel column) or 16 (two per column, rows split;
                   // measured slower: 768 threads cap registers at 80 and the epilogue spills)
#endif
constexpr int kFzThreads = 256 + 32 * FZ_TFW;

struct FzSeg {
    const void *src;   // raw operand tensor [T][H][W][c]
    int c;          // channels of this segment
    int cglob0;     // first operand channel (coef index) of this segment
    int taps;       // 9 (GN/SiLU operand) or 1 (raw shortcut)
    int transform;  // 1: GN-apply + SiLU + padding zero; 0: copy
    int shift;      // 1: channels [0, cs) of the segment come from frame t-1 / carry
    int bidx, col0, tapstride, packed;
};

struct FzParams {
    CUtensorMap bmap[2];   // weights, box {64, BN/CG}
    CUtensorMap smap[4];   // raw (transform == 0) segments: box {64, 8, 16, 1}, SW128 -> straight into a tile slot
    CUtensorMap hmap[4];   // transform segments: 8-channel halo box {8, 10, 18, 1}, no swizzle, OOB zero
    CUtensorMap wmap[4];   // transform segments: 64-channel halo box {64, 10, 18, 1}, SW128, OOB zero
    CUtensorMap cmap;      // padded carry [1][H][W][cs_pad], same box (if has_carry)
    FzSeg seg[4];
    int nseg, cs, has_carry, cs_pad;
    const void *carry_pad; // [H][W][cs_pad] (16-byte rows)
    const float2 *coef;    // [T][C_op] = (scale, shift) of the GN affine, beta and mean folded in
    int cop;               // channels of the fused operand
    int T, H, W, cout, bn, tiles_x, tiles_y, nbox, ntile_n, nwork;
    const void *bias0, *bias1;
    void *out;
    float *stats;
    uint32_t idesc;
    int ntf, nraw, nb;   // tile slots, raw slots (0 or 2..4), weight stages (sized from the shared-memory budget)
    unsigned long long *prof;   // [6][4] wait/total cycles per role (PROF kernels only)
    int sw_mode;                // 0: 8-channel no-swizzle boxes only; 1/2: SW128 whole-chunk box for unshifted chunks (2: base offset)
    int nsteps;                 // K loop of a work item: (segment, 64-channel chunk) steps in issue order,
    unsigned char ord[64];      //   ord[i] = seg << 6 | chunk (raw 1x1 chunks interleaved among the 3x3 ones)
    int up2;                    // output = exact 2x nearest upsampling (four strided TMA stores per chunk)
    int epi_tma;                // 1: epilogue stages 32-column chunks in shared memory, TMA-stores them and reads
                                //    the box statistics back column-wise; 0: per-thread row stores + butterflies
    CUtensorMap omap[2];        // output [T][H][W][cout]: box {32, 8, 16, 1} SW64 / {16, 8, 16, 1} SW32
    int wres;                   // 1: one N tile and nb == the weight stages of a work item: the weights are
                                //    loaded once and stay resident (no per-item weight stream)
};

// UMMA descriptor, K-major, no swizzle: core matrices of 8 rows x 16 B
__device__ __forceinline__ uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version; layout type 0 = SWIZZLE_NONE
    return d;
}

// SiLU(z) = z * rcp(1 + ex2(u)) with u = -z*log2(e) from its own FFMA: two MUFU ops
// (ex2.approx, rcp.approx; <= 2 ulp fp32 each), far below the 16-bit rounding of H (R23)
__device__ __forceinline__ float fz_ex2(float u) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(u));
    return e;
}
// SiLU(z) = z * sigmoid(z) = hz + hz * tanh(hz) with hz = z / 2: ONE MUFU op (tanh.approx,
// max rel. error 2^-11) and two FMAs per element, from an affine pre-scaled by 1/2.  The MUFU
// count is what bounds the in-place transform when a convolution has few output channels (the VAE
// decoder's 64-channel full-resolution convs: 2 MUFU ops per input element outran the MMAs).
#ifndef FZ_SILU_TANH
#define FZ_SILU_TANH 1
#endif
__device__ __forceinline__ float fz_tanh(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fz_rcp(float d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return r;
}
// an unshifted transform chunk is one SW128 halo box {64, 10, 18} (rows of 128 B); chunks holding
// shifted channels keep the 8-channel no-swizzle columns (per-group source selection)
__device__ __forceinline__ bool fz_sw_chunk(const FzParams &p, const FzSeg &sg, int c0) {
    return p.sw_mode != 0 && (!sg.shift || c0 >= p.cs);
}
template <typename T> struct Pk;
template <> struct Pk<__nv_bfloat16> {
    static __device__ __forceinline__ void unpack(uint32_t w, float &a, float &b) {
        a = __uint_as_float(w << 16);
        b = __uint_as_float(w & 0xFFFF0000u);
    }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};
template <> struct Pk<__half> {
    static __device__ __forceinline__ void unpack(uint32_t w, float &a, float &b) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w));
        a = f.x;
        b = f.y;
    }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};

struct FzBox {
    int t, y0, x0;
    bool valid;
};
__device__ __forceinline__ FzBox fz_box(const FzParams &p, int box) {
    FzBox b;
    b.valid = box < p.nbox;
    if (!b.valid) {
        b.t = p.T;   // fully out of bounds: TMA zero fill
        b.y0 = b.x0 = 0;
        return b;
    }
    const int per = p.tiles_x * p.tiles_y;
    b.t = box / per;
    const int rem = box - b.t * per;
    b.y0 = (rem / p.tiles_x) * FZ_BY;
    b.x0 = (rem % p.tiles_x) * FZ_BX;
    return b;
}

// PROF: clock64 accounting of the pipeline waits per warp role (DVC_FZ_PROF=1; diagnostics only)
template <typename T, int CG, bool PROF>
__global__ void __launch_bounds__(kFzThreads, 1) conv_fz_kernel(const __grid_constant__ FzParams p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so the compiler keeps the
    // shared address space (an integer round trip would turn every access generic)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int BN = p.bn, BNH = p.bn / CG;
    const int B_STAGE = BNH * 128;
    // transform tile slots (4 unless overridden), a separate 2-slot ring for the raw 1x1 segments
    // (so short raw chunks never hold back the transform prefetch), weight stages filling the
    // rest of the 227 KB
    const int NTF = p.ntf, NRAW = p.nraw, FZ_BSTAGES = p.nb;
    uint8_t *sTf = smem;                        // [NTF] transformed operand tiles
    uint8_t *sRaw = sTf + NTF * FZ_SLOT;        // [NRAW] raw SW128 boxes (16 KB)
    uint8_t *sStage = sRaw + NRAW * FZ_RAW_SLOT;   // [2] epilogue staging (8 KB each, epi_tma)
    uint8_t *sB = sStage + (p.epi_tma ? 2 * kEpiStage : 0);   // [FZ_BSTAGES] weight tiles
    uint64_t *tf_full = reinterpret_cast<uint64_t *>(sB + FZ_BSTAGES * B_STAGE);
    uint64_t *tf_empty = tf_full + FZ_MAX_NTF;
    uint64_t *b_full = tf_empty + FZ_MAX_NTF;
    uint64_t *b_empty = b_full + FZ_BSTAGES;
    uint64_t *tfull = b_empty + FZ_BSTAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *raw_full = tempty + 2;   // [4] halo TMA (+ coefficients) landed in slot tb (local CTA)
    uint64_t *rw_full = raw_full + FZ_MAX_NTF;  // [NRAW] raw box landed (leader; both CTAs' bytes)
    uint64_t *rw_empty = rw_full + FZ_MAX_RAW;  // [NRAW] raw slot free (MMA commit, both CTAs)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rw_empty + FZ_MAX_RAW);
    float *red = reinterpret_cast<float *>(tmem_slot + 4);   // [2][2][4][32] box-statistics staging
    float *sbias = red + 512;   // [2][cout] bias0, bias1 in fp32 (16-byte aligned: the barrier block is
                                // 1024-aligned and holds an even number of 8-byte barriers)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const int cluster_id = blockIdx.x / CG, nclusters = gridDim.x / CG;
    const uint32_t ncols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < FZ_MAX_NTF; ++i) {
            mbar_init(&tf_full[i], CG);
            mbar_init(&tf_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], CG * 4);
        }
        for (int s = 0; s < FZ_BSTAGES; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int i = 0; i < FZ_MAX_NTF; ++i) mbar_init(&raw_full[i], 1);
        for (int i = 0; i < FZ_MAX_RAW; ++i) {
            mbar_init(&rw_full[i], CG);
            mbar_init(&rw_empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    if (warp == 1) tmem_alloc<CG>(smem_u32(tmem_slot), ncols);
    for (int i = tid; i < p.cout; i += kFzThreads) {
        sbias[i] = p.bias0 ? Elem<T>::to_f(reinterpret_cast<const T *>(p.bias0)[i]) : 0.f;
        sbias[p.cout + i] = p.bias1 ? Elem<T>::to_f(reinterpret_cast<const T *>(p.bias1)[i]) : 0.f;
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();     // predecessor grid complete: activations may be read / written
    griddep_launch();   // the successor may be scheduled on SMs that free up
    unsigned long long pacc[4] = {0, 0, 0, 0};
    const long long tstart = PROF ? clock64() : 0;
#define FZ_TIMED(slot, stmt)                                  \
    do {                                                      \
        const long long t0_ = PROF ? clock64() : 0;           \
        stmt;                                                 \
        if constexpr (PROF) pacc[slot] += clock64() - t0_;    \
    } while (0)

    if (warp == 2) {
        // ===================== weight producer =====================
        // converged warp; lane 0 issues through guard predicates (no divergent region per stage)
        int bs = 0;
        uint32_t bph = 0;
        const uint32_t tx = (uint32_t)CG * (uint32_t)B_STAGE;
        const uint32_t issue = lane == 0, expect = issue && rank == 0;
        const uint32_t bfull0 = smem_u32(b_full), bempty0 = smem_u32(b_empty), sB0 = smem_u32(sB);
        const uint32_t lead_bfull0 = CG == 2 ? mapa_shared(bfull0, 0) : bfull0;
        for (int w = cluster_id; w < p.nwork; w += nclusters) {
            if (p.wres && w != cluster_id) break;   // resident weights: one pass
            const int nt = w % p.ntile_n;
            const int n0 = nt * BN + (int)rank * BNH;
            for (int st_i = 0; st_i < p.nsteps; ++st_i) {
                const int s = p.ord[st_i] >> 6, ch = p.ord[st_i] & 63;
                const FzSeg &sg = p.seg[s];
                const int nch = (sg.c + 63) >> 6;
                const CUtensorMap *bm = &p.bmap[sg.bidx];
                for (int tap = 0; tap < sg.taps; ++tap) {
                    FZ_TIMED(0, mbar_wait_spin_addr(bempty0 + 8 * bs, bph ^ 1));
                    // packed weights: the (tap, chunk) tile is one contiguous row block
                    const int col = sg.packed ? 0 : sg.col0 + tap * sg.tapstride + ch * 64;
                    const int row = sg.packed ? sg.col0 + (tap * nch + ch) * p.cout + n0 : n0;
                    mbar_expect_tx_if(expect, bfull0 + 8 * bs, tx);
                    tma_load_2d_if<CG>(issue, sB0 + bs * B_STAGE, bm, lead_bfull0 + 8 * bs, col, row);
                    if (++bs == FZ_BSTAGES) {
                        bs = 0;
                        bph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 3 || warp == 0) {
        // ===================== operand tile producers (TMA) =====================
        // warp 3: transformed segments (tf ring); warp 0: raw 1x1 segments (raw ring).  Two
        // producers so that neither ring's back-pressure holds up the other's prefetch.
        // transform segments: per 8-channel group one halo box {8 ch, 10, 18} of frame t (or of
        // frame t-1 / the carry / zeros for the shifted channels) straight into its core-matrix
        // column, plus the 64 GN coefficients; raw 1x1 segments: one SW128 box into the slot,
        // completing on the leader's tf_full.
        int tb = 0, rb = 0;
        uint32_t tph = 0, rph = 0;
        const uint32_t issue = lane == 0;
        const uint32_t rw_full_leader = CG == 2 ? mapa_shared(smem_u32(&rw_full[0]), 0) : smem_u32(&rw_full[0]);
        const bool raw_role = warp == 0;
        for (int w = cluster_id; w < p.nwork; w += nclusters) {
            const FzBox bx = fz_box(p, (w / p.ntile_n) * CG + (int)rank);
            for (int st_i = 0; st_i < p.nsteps; ++st_i) {
                const int s = p.ord[st_i] >> 6, ch = p.ord[st_i] & 63;
                const FzSeg &sg = p.seg[s];
                const int nch = (sg.c + 63) >> 6;
                if (raw_role == (sg.transform != 0)) continue;   // the other producer's segment
                if (!sg.transform) {   // raw ring
                    FZ_TIMED(0, mbar_wait(&rw_empty[rb], rph ^ 1));
                    if (issue) {
                        const uint32_t fb = rw_full_leader + (uint32_t)(rb * 8);
                        const uint32_t dst = smem_u32(sRaw + rb * FZ_RAW_SLOT);
                        if constexpr (CG == 1) {
                            mbar_arrive_expect_tx_addr(fb, FZ_RAW_SLOT);
                            tma_load_4d(dst, &p.smap[s], fb, ch * 64, bx.x0, bx.y0, bx.t);
                        } else {
                            mbar_arrive_expect_tx_cluster(fb, FZ_RAW_SLOT);
                            tma_load_4d_cg2(dst, &p.smap[s], fb, ch * 64, bx.x0, bx.y0, bx.t);
                        }
                    }
                    __syncwarp();
                    if (++rb == NRAW) {
                        rb = 0;
                        rph ^= 1;
                    }
                    continue;
                }
                FZ_TIMED(0, mbar_wait(&tf_empty[tb], tph ^ 1));
                const uint32_t slot = smem_u32(sTf + tb * FZ_SLOT);
                if (issue) {
                    const int c0 = ch * 64;
                    const int ngrp = min(8, (sg.c - c0) >> 3);
                    const uint32_t rb = smem_u32(&raw_full[tb]);
                    const uint32_t coef_bytes = bx.valid ? (uint32_t)ngrp * 64u : 0u;
                    if (fz_sw_chunk(p, sg, c0)) {
                        mbar_arrive_expect_tx_addr(rb, (uint32_t)FZ_HROWS * 128u + coef_bytes);
                        tma_load_4d(slot, &p.wmap[s], rb, c0, bx.x0 - 1, bx.y0 - 1, bx.t);
                        if (coef_bytes)
                            bulk_load(slot + FZ_COEF, p.coef + (size_t)bx.t * p.cop + sg.cglob0 + c0, coef_bytes, rb);
                        goto produced;
                    }
                    {
                    int nside = 0;
                    for (int g = 0; g < ngrp; ++g) {
                        const int nprev = sg.shift ? min(max(p.cs - (c0 + 8 * g), 0), 8) : 0;
                        nside += nprev > 0 && nprev < 8;
                    }
                    mbar_arrive_expect_tx_addr(rb, (uint32_t)(ngrp + nside) * FZ_COLB + coef_bytes);
                    for (int g = 0; g < ngrp; ++g) {
                        const int cl = c0 + 8 * g;
                        const int nprev = sg.shift ? min(max(p.cs - cl, 0), 8) : 0;
                        const uint32_t dst = slot + (uint32_t)(g * FZ_LBO);
                        if (nprev < 8)
                            tma_load_4d(dst, &p.hmap[s], rb, cl, bx.x0 - 1, bx.y0 - 1, bx.t);
                        if (nprev > 0) {
                            // shifted channels: frame t-1, the carry at t = 0, or (no carry) a fully
                            // out-of-bounds box = zeros
                            const uint32_t pd = nprev < 8 ? slot + FZ_SIDE : dst;
                            if (bx.t > 0 || !p.has_carry)
                                tma_load_4d(pd, &p.hmap[s], rb, cl, bx.x0 - 1, bx.y0 - 1, bx.t > 0 ? bx.t - 1 : -1);
                            else
                                tma_load_4d(pd, &p.cmap, rb, cl, bx.x0 - 1, bx.y0 - 1, 0);
                        }
                    }
                    if (coef_bytes)
                        bulk_load(slot + FZ_COEF, p.coef + (size_t)bx.t * p.cop + sg.cglob0 + c0, coef_bytes, rb);
                    }
                produced:;
                }
                __syncwarp();
                if (++tb == NTF) {
                    tb = 0;
                    tph ^= 1;
                }
            }
        }
    } else if (warp >= 8) {
        // ===================== transform warps: in place, H = SiLU(GN(X)) =====================
        const int kg = (warp - 8) & 7;                     // 8-channel core-matrix column of this warp
        const int row0 = FZ_TFW == 16 ? ((warp - 8) >> 3) * 96 : 0;   // 16 warps: rows [0,96) / [96,180)
        int tb = 0;
        uint32_t tph = 0;
        uint32_t rph = 0;   // raw_full phase per slot: only transform chunks complete raw_full
        const uint32_t tf_full_leader = CG == 2 ? mapa_shared(smem_u32(&tf_full[0]), 0) : smem_u32(&tf_full[0]);
        for (int w = cluster_id; w < p.nwork; w += nclusters) {
            const FzBox bx = fz_box(p, (w / p.ntile_n) * CG + (int)rank);
            for (int st_i = 0; st_i < p.nsteps; ++st_i) {
                const int s = p.ord[st_i] >> 6, ch = p.ord[st_i] & 63;
                const FzSeg &sg = p.seg[s];
                const int nch = (sg.c + 63) >> 6;
                if (!sg.transform) continue;   // raw segments use their own ring
                const int cl = ch * 64 + kg * 8;   // first channel (segment-local) of this warp
                uint8_t *slot = sTf + tb * FZ_SLOT;
                FZ_TIMED(0, mbar_wait(&raw_full[tb], (rph >> tb) & 1u));
                rph ^= 1u << tb;
                if (cl < sg.c) {   // warp-uniform; groups past the segment are never read by the MMA
                    // GN affine of frame t for the 8 channels, z = v*sc + sh, and the same affine
                    // pre-scaled by -log2(e) so that e^-z = ex2(v*sc2 + sh2) costs one FFMA
                    float sc[8], sh[8], sc2[8], sh2[8];
                    if (bx.valid) {
                        const float4 *cf = reinterpret_cast<const float4 *>(slot + FZ_COEF + kg * 64);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float4 q = cf[i];
                            sc[2 * i] = q.x, sh[2 * i] = q.y, sc[2 * i + 1] = q.z, sh[2 * i + 1] = q.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) sc[i] = 1.f, sh[i] = 0.f;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if constexpr (FZ_SILU_TANH) sc[i] *= 0.5f, sh[i] *= 0.5f;   // hz = z / 2
                        sc2[i] = sc[i] * -1.4426950408889634f, sh2[i] = sh[i] * -1.4426950408889634f;
                    }
                    // a group straddling C_in/P: its first nprev channels come from the side buffer.
                    // C_in/P is even (C_in % 16 == 0): merge per 32-bit word.
                    const int nprev = sg.shift ? min(max(p.cs - cl, 0), 8) : 0;
                    const bool straddle = nprev > 0 && nprev < 8;
                    uint32_t msk[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) msk[j] = 2 * j < nprev ? 0xFFFFFFFFu : 0u;
                    // row r of this warp's 8 channels: SW128 chunk -> 16-byte unit kg ^ (r & 7) of the
                    // 128-byte row r (the TMA swizzle); else row r of core-matrix column kg
                    const bool sw = fz_sw_chunk(p, sg, ch * 64);
                    auto roff = [&](int r) -> int { return sw ? r * 128 + ((kg ^ (r & 7)) << 4) : kg * FZ_LBO + r * 16; };
                    constexpr int NR = FZ_TFW == 16 ? 3 : (FZ_HROWS + 31) / 32;   // halo rows per lane
                    // all rows' words first (independent shared loads in flight), then two rows
                    // (16 independent ex2 / rcp chains) per step
                    uint32_t wv[NR][4];
#pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        const int r = row0 + lane + 32 * k;
                        uint4 cu = make_uint4(0, 0, 0, 0);
                        if (r < FZ_HROWS) {
                            cu = *reinterpret_cast<const uint4 *>(slot + roff(r));
                            if (straddle) {
                                const uint4 pv = *reinterpret_cast<const uint4 *>(slot + FZ_SIDE + r * 16);
                                cu.x = (pv.x & msk[0]) | (cu.x & ~msk[0]);
                                cu.y = (pv.y & msk[1]) | (cu.y & ~msk[1]);
                                cu.z = (pv.z & msk[2]) | (cu.z & ~msk[2]);
                                cu.w = (pv.w & msk[3]) | (cu.w & ~msk[3]);
                            }
                        }
                        wv[k][0] = cu.x, wv[k][1] = cu.y, wv[k][2] = cu.z, wv[k][3] = cu.w;
                    }
#pragma unroll
                    for (int k0 = 0; k0 < NR; k0 += 2) {
                        float z[2][8], e[2][8];
#pragma unroll
                        for (int k = 0; k < 2; ++k)
                            if (k0 + k < NR)
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                float v0, v1;
                                Pk<T>::unpack(wv[k0 + k][j], v0, v1);
                                z[k][2 * j] = fmaf(v0, sc[2 * j], sh[2 * j]);
                                z[k][2 * j + 1] = fmaf(v1, sc[2 * j + 1], sh[2 * j + 1]);
                                if constexpr (FZ_SILU_TANH) {   // z holds hz = z / 2; e = tanh(hz)
                                    e[k][2 * j] = fz_tanh(z[k][2 * j]);
                                    e[k][2 * j + 1] = fz_tanh(z[k][2 * j + 1]);
                                } else if constexpr (FZ_TFW == 16) {   // register budget: u = -z log2(e) from z
                                    e[k][2 * j] = fz_ex2(z[k][2 * j] * -1.4426950408889634f);
                                    e[k][2 * j + 1] = fz_ex2(z[k][2 * j + 1] * -1.4426950408889634f);
                                } else {
                                    e[k][2 * j] = fz_ex2(fmaf(v0, sc2[2 * j], sh2[2 * j]));
                                    e[k][2 * j + 1] = fz_ex2(fmaf(v1, sc2[2 * j + 1], sh2[2 * j + 1]));
                                }
                            }
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const int r = row0 + lane + 32 * (k0 + k);
                            if (k0 + k >= NR || r >= FZ_HROWS) continue;
                            const int hy = r / FZ_HX, hx = r - hy * FZ_HX;
                            const int y = bx.y0 - 1 + hy, x = bx.x0 - 1 + hx;
                            // conv zero padding applies AFTER the transform (H3): out of frame -> 0
                            const bool live = bx.valid && y >= 0 && y < p.H && x >= 0 && x < p.W;
                            uint32_t o[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                float h0, h1;
                                if constexpr (FZ_SILU_TANH) {
                                    h0 = fmaf(z[k][2 * j], e[k][2 * j], z[k][2 * j]);
                                    h1 = fmaf(z[k][2 * j + 1], e[k][2 * j + 1], z[k][2 * j + 1]);
                                } else {
                                    h0 = z[k][2 * j] * fz_rcp(1.0f + e[k][2 * j]);
                                    h1 = z[k][2 * j + 1] * fz_rcp(1.0f + e[k][2 * j + 1]);
                                }
                                o[j] = live ? Pk<T>::pack(h0, h1) : 0u;
                            }
                            *reinterpret_cast<uint4 *>(slot + roff(r)) = make_uint4(o[0], o[1], o[2], o[3]);
                        }
                    }
                }
                FZ_TIMED(2, fence_proxy_async());   // generic-proxy smem writes -> visible to the tensor core
                FZ_TIMED(1, asm volatile("bar.sync 2, %0;" ::"n"(32 * FZ_TFW) : "memory"));   // the transform warps
                if (warp == 8 && elect_one()) {
                    if constexpr (CG == 1)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tf_full[tb]))
                                     : "memory");
                    else mbar_arrive_cluster(tf_full_leader + (uint32_t)(tb * 8));
                }
                __syncwarp();
                if (++tb == NTF) {
                    tb = 0;
                    tph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA) =====================
        // converged warp; mma_stage() elects the issuing lane inside its asm
        if (rank == 0) {
            int bs = 0, tb = 0, rb = 0, it = 0;
            uint32_t bph = 0, tph = 0, rph = 0;
            const uint32_t rwfull0 = smem_u32(rw_full), rwempty0 = smem_u32(rw_empty), sR0 = smem_u32(sRaw);
            const uint32_t bfull0 = smem_u32(b_full), bempty0 = smem_u32(b_empty);
            const uint32_t tffull0 = smem_u32(tf_full), tfempty0 = smem_u32(tf_empty);
            const uint32_t b_lo0 = desc_lo(smem_u32(sB), 16), sT0 = smem_u32(sTf);
            const uint32_t b_inc = (uint32_t)(B_STAGE >> 4);
            uint32_t b_lo = b_lo0;   // descriptor word of weight stage bs
            for (int w = cluster_id; w < p.nwork; w += nclusters, ++it) {
                const int buf = it & 1;
                const uint32_t use = (uint32_t)(it >> 1) & 1;
                FZ_TIMED(0, mbar_wait_spin(&tempty[buf], use ^ 1));
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * BN);
                uint32_t acc = 0;
                for (int st_i = 0; st_i < p.nsteps; ++st_i) {
                    const int s = p.ord[st_i] >> 6, ch = p.ord[st_i] & 63;
                    const FzSeg &sg = p.seg[s];
                    const int nch = (sg.c + 63) >> 6;
                    const uint32_t klast = (uint32_t)(sg.c - 64 * (nch - 1)) >> 4;
                    // transformed tile: K step of 16 channels = two 8-channel core-matrix columns of
                    // the halo layout (no swizzle); raw segment: the TMA box in SW128
                    const bool tf = sg.transform != 0;
                    const uint32_t ks = ch == nch - 1 ? klast : 4u;
                    if (!tf) {   // raw 1x1 chunk from the raw ring (SW128 box): one tap
                        FZ_TIMED(1, mbar_wait_spin_addr(rwfull0 + 8 * rb, rph));
                        tc_fence_after();
                        if (!p.wres || it == 0) FZ_TIMED(2, mbar_wait_spin_addr(bfull0 + 8 * bs, bph));
                        tc_fence_after();
                        mma_stage<CG>(d, desc_lo(sR0 + (uint32_t)(rb * FZ_RAW_SLOT), 16), kDescHiSw128, 2u, b_lo,
                                      kDescHiSw128, p.idesc, ks, acc, bempty0 + 8 * bs);
                        acc = 1;
                        commit_elected<CG>(rwempty0 + 8 * rb);
                        b_lo += b_inc;
                        if (++bs == FZ_BSTAGES) {
                            bs = 0;
                            bph ^= 1;
                            b_lo = b_lo0;
                        }
                        if (++rb == NRAW) {
                            rb = 0;
                            rph ^= 1;
                        }
                        continue;
                    }
                    FZ_TIMED(1, mbar_wait_spin_addr(tffull0 + 8 * tb, tph));
                    tc_fence_after();
                    // transformed tile (no swizzle, 8-channel core-matrix columns FZ_LBO apart, image
                    // rows FZ_SBO apart): tap (dy, dx) starts (1+dy)*10 + (1+dx) halo rows in; a K step
                    // of 16 channels = two core-matrix columns
                    // SW128 chunk: rows of 128 B, image rows FZ_HX * 128 B apart, tap offset in
                    // whole rows, K step +32 B
                    const bool sw = fz_sw_chunk(p, sg, ch * 64);
                    const uint32_t a_base = sT0 + (uint32_t)(tb * FZ_SLOT);
                    const uint32_t a_lo0 = sw ? desc_lo(a_base, 16) : desc_lo(a_base, FZ_LBO);
                    const uint32_t a_hi = sw ? desc_hi_sw128(FZ_HX * 128) : desc_hi_noswz(FZ_SBO);
                    const uint32_t a_step = sw ? 2u : (uint32_t)(2 * FZ_LBO) >> 4;
                    const uint32_t a_row = sw ? 8u : 1u;   // one halo row in 16-byte units
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap) {
                        if (!p.wres || it == 0) FZ_TIMED(2, mbar_wait_spin_addr(bfull0 + 8 * bs, bph));
                        tc_fence_after();
                        const uint32_t roff16 = (uint32_t)((tap / 3) * FZ_HX + tap % 3) * a_row;
                        // optional matrix base offset (bits 49-51): the 1024-B pattern phase of the start
                        const uint32_t bo = sw && p.sw_mode == 2 ? (((a_base >> 7) + roff16 / 8) & 7u) << 17 : 0u;
                        mma_stage<CG>(d, a_lo0 + roff16, a_hi | bo, a_step, b_lo, kDescHiSw128, p.idesc, ks, acc,
                                      bempty0 + 8 * bs);
                        acc = 1;
                        b_lo += b_inc;
                        if (++bs == FZ_BSTAGES) {
                            bs = 0;
                            bph ^= 1;
                            b_lo = b_lo0;
                        }
                    }
                    commit_elected<CG>(tfempty0 + 8 * tb);   // the tile slot is free once its taps retire
                    if (++tb == NTF) {
                        tb = 0;
                        tph ^= 1;
                    }
                }
                commit_elected<CG>(smem_u32(&tfull[buf]));
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===================== epilogue (both CTAs) =====================
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const int by = r / FZ_BX, bxp = r - by * FZ_BX;
        const float *sb0 = p.bias0 ? sbias : nullptr;
        const float *sb1 = p.bias1 ? sbias + p.cout : nullptr;
        T *out = reinterpret_cast<T *>(p.out);
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
        int it = 0;
        // staging-buffer / reduction parity, kept across work items: an odd chunk count per item (narrow
        // N tiles) must not restart on the buffer whose TMA store may still be reading it
        int par = 0;
        for (int w = cluster_id; w < p.nwork; w += nclusters, ++it) {
            const int buf = it & 1;
            const uint32_t use = (uint32_t)(it >> 1) & 1;
            const int q = w / p.ntile_n, nt = w - q * p.ntile_n;
            const int box = q * CG + (int)rank;
            const FzBox bx = fz_box(p, box);
            long m = -1;
            if (bx.valid) {
                const int y = bx.y0 + by, x = bx.x0 + bxp;
                if (y < p.H && x < p.W) m = ((long)bx.t * p.H + y) * p.W + x;
            }
            FZ_TIMED(1, mbar_wait(&tfull[buf], use));
            tc_fence_after();
            const bool want_stats = p.stats != nullptr && bx.valid;
            const int per = p.tiles_x * p.tiles_y;
            float *stats_box = want_stats ? p.stats + ((size_t)bx.t * per + (box - bx.t * per)) * p.cout * 2 : nullptr;
            // one 16-column chunk: + bias (fp32, shared memory), 16-bit store; returns (in x) this
            // row's statistics contribution of the stored values
            auto chunk = [&](const uint32_t (&v)[16], int n, float (&x)[32]) {
                float f[16];
                if (m >= 0) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
                    if (sb0) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            const float4 e = *reinterpret_cast<const float4 *>(sb0 + n + i);
                            f[i] += e.x, f[i + 1] += e.y, f[i + 2] += e.z, f[i + 3] += e.w;
                        }
                    }
                    if (sb1) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            const float4 e = *reinterpret_cast<const float4 *>(sb1 + n + i);
                            f[i] += e.x, f[i + 1] += e.y, f[i + 2] += e.z, f[i + 3] += e.w;
                        }
                    }
                    Vec8<T> lo, hi;
                    round_store16<T>(f, lo, hi);   // f <- the stored values (statistics, R17)
                    *reinterpret_cast<Vec8<T> *>(out + m * p.cout + n) = lo;
                    *reinterpret_cast<Vec8<T> *>(out + m * p.cout + n + 8) = hi;
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = 0.f;   // rows outside the frame count as 0
                }
                if (want_stats) box_row_values(f, true, x);
            };
            const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * BN);
            if (p.epi_tma) {
                // Staged epilogue, per 32-column chunk: TMEM -> registers (thread = box row) -> + bias,
                // 16-bit rounding -> a swizzled [128 rows][32 cols] tile in shared memory (zeros for rows
                // outside the frame) -> one TMA store of the {32, 8, 16, 1} box (the hardware clips the
                // out-of-frame rows); the box statistics are then read back column-wise (lane = column,
                // warp q4 = rows 32*q4..32*q4+31) and reduced with the canonical tree of dvc_boxstats.cuh
                // (pairs of rows differing in bit 4, then 3, 2, 1, 0; warps combined ((w0+w1)+w2)+w3),
                // i.e. bit for bit what the butterfly produced, without the 62 shuffles per 16 columns.
                const bool issuer = warp == 4 && lane == 0;
#pragma unroll 1
                for (int cc = 0; cc < BN; cc += 32, par ^= 1) {
                    const bool two = cc + 16 < BN;   // warp-uniform: 32 or 16 columns
                    const int n = nt * BN + cc;
                    uint32_t va[16], vb[16];
                    tmem_ld16_nowait(taddr + (uint32_t)cc, va);
                    if (two) tmem_ld16_nowait(taddr + (uint32_t)(cc + 16), vb);
                    tmem_wait16(va);
                    if (two) tmem_wait16(vb);
                    if (cc + 32 >= BN) {   // the accumulator is drained: the MMA may reuse it
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            tmem_drained_arrive(CG == 2 ? tempty_leader + (uint32_t)(buf * 8) : smem_u32(&tempty[buf]), CG == 2);
                        }
                    }
                    float f[32];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        f[i] = __uint_as_float(va[i]);
                        f[16 + i] = __uint_as_float(vb[i]);
                    }
                    if (sb0) epi_add_bias(f, sb0 + n, two);   // bias0 then bias1, as the other paths
                    if (sb1) epi_add_bias(f, sb1 + n, two);
                    epi_stage_chunk<T>(f, m >= 0, two, r, q4, lane, sStage + par * kEpiStage, &p.omap[0], &p.omap[1],
                                       issuer, bx.valid, n, bx.x0, bx.y0, bx.t,
                                       want_stats ? stats_box + (size_t)n * 2 : nullptr, red + par * 256, p.up2 != 0);
                }
                continue;
            }
            // TMEM -> registers 32 columns at a time (two 16-column loads in flight); the box
            // statistics of both chunks are reduced together (two independent butterflies, one
            // barrier per 32 columns) and combined by warps 0 / 1 (canonical order, dvc_boxstats.cuh)
#pragma unroll 1
            for (int cc = 0; cc < BN; cc += 32, par ^= 1) {
                const bool two = cc + 16 < BN;   // warp-uniform
                uint32_t va[16], vb[16];
                tmem_ld16_nowait(taddr + (uint32_t)cc, va);
                if (two) tmem_ld16_nowait(taddr + (uint32_t)(cc + 16), vb);
                tmem_wait16(va);
                float *rr = red + par * 256;   // [2 chunks][4 warps][32]
                float x[32];
                chunk(va, nt * BN + cc, x);
                if (want_stats) rr[q4 * 32 + lane] = box_reduce_scatter32(x, lane);
                if (two) {
                    tmem_wait16(vb);
                    chunk(vb, nt * BN + cc + 16, x);
                    if (want_stats) rr[128 + q4 * 32 + lane] = box_reduce_scatter32(x, lane);
                }
                if (want_stats) {
                    FZ_TIMED(2, asm volatile("bar.sync 1, 128;" ::: "memory"));
                    if (q4 < (two ? 2 : 1)) {
                        const int n = nt * BN + cc + 16 * q4;
                        stats_box[(n + (lane & 15)) * 2 + (lane >> 4)] = box_combine4(rr + q4 * 128, lane);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                tmem_drained_arrive(CG == 2 ? tempty_leader + (uint32_t)(buf * 8) : smem_u32(&tempty[buf]), CG == 2);
            }
        }
    }
#undef FZ_TIMED
    if (p.epi_tma && warp == 4 && lane == 0) bulk_wait_group<0>();   // every staged store has landed
    if constexpr (PROF) {
        const int role = warp == 1 ? 0 : warp == 4 ? 1 : warp == 8 ? 2 : warp == 3 ? 3 : warp == 2 ? 4 : -1;
        if (role >= 0 && lane == 0 && !(role == 0 && rank != 0)) {
            pacc[3] = clock64() - tstart;
            for (int i = 0; i < 4; ++i) atomicAdd(p.prof + role * 4 + i, pacc[i]);
        }
        if (tid == 0) atomicAdd(p.prof + 20, 1ull);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem, ncols);
    }
}

// ----------------------------------------------------------------- host side
PFN_encodeTiled_t get_encode_fn();
dvc_status make_bmap_rows(CUtensorMap *map, const void *ptr, dvc_dtype dt, long rows, long cols, int box_rows);
extern int g_ws_cg;

dvc_status make_box_map(CUtensorMap *map, const void *ptr, dvc_dtype dt, int T, int H, int W, int C, int BX, int BY);

static int fz_off_from_env() {   // DVC_NO_FZ=1: never use the fused engine (A/B experiments)
    const char *e = dvc_knob("DVC_NO_FZ");
    return e && e[0] == '1';
}
static const int g_fz_off = fz_off_from_env();
static int fz_min_h_from_env() {   // DVC_FZ_MIN_H: smallest frame height on the fused engine (A/B experiments)
    const char *e = dvc_knob("DVC_FZ_MIN_H");
    return e ? atoi(e) : 32;
}
static const int g_fz_min_h = fz_min_h_from_env();
bool conv_fz_applicable(int H, int W, dvc_dtype dt) {
    return !g_fz_off && g_ws_cg == 2 && dt != DVC_F32 && H >= g_fz_min_h && W >= 8;
}

static int g_fz_sms = 0;

// 8-channel halo box {8, 10, 18, 1} of a [T][H][W][C] tensor, no swizzle: lands as one 180-row
// core-matrix column of the UMMA tile; out-of-bounds rows (and frames) are zero-filled
static dvc_status make_halo_map(CUtensorMap *map, const void *ptr, dvc_dtype dt, int T, int H, int W, int C,
                                 int box_c = 8) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && C % 8 == 0, DVC_ERR_ARG, "fused conv: halo source alignment");
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)FZ_HX, (cuuint32_t)FZ_HY, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                     const_cast<void *>(ptr), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     box_c == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     box_c == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (halo) failed (%d)", (int)r);
    return DVC_OK;
}

// output box {c, 8, 16, 1} of a [T][H][W][cout] tensor for the staged epilogue's TMA store: 32 channels
// (64-byte rows, SWIZZLE_64B) or 16 (32-byte rows, SWIZZLE_32B), matching the staging layout
// up = 2: the tensor is the 2x upsampled output [T][2H][2W][C], walked with element stride 2 in x and
// y so that a staged 8 x 16 box lands on one phase of the upsampled grid
static dvc_status make_out_map(CUtensorMap *map, void *ptr, dvc_dtype dt, int T, int H, int W, int C, int box_c,
                               int up = 1, int up_ho = 0, int up_wo = 0) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && C % 8 == 0, DVC_ERR_ARG, "fused conv: output alignment");
    // up = 2: the real upsampled extent (2H - 1 clips the last phase-1 row)
    const cuuint64_t Ho = up == 2 && up_ho ? up_ho : (cuuint64_t)H * up, Wo = up == 2 && up_wo ? up_wo : (cuuint64_t)W * up;
    cuuint64_t gdim[4] = {(cuuint64_t)C, Wo, Ho, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C * 2, Wo * C * 2, Ho * Wo * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)(FZ_BX * up), (cuuint32_t)(FZ_BY * up), 1};
    cuuint32_t estr[4] = {1, (cuuint32_t)up, (cuuint32_t)up, 1};
    CUresult r = enc(map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, ptr,
                     gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     box_c == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed (%d)", (int)r);
    return DVC_OK;
}

dvc_status conv_fz_run(const FzDesc &d, cudaStream_t stream) {
    // identity skips are X . I segments (an epilogue residual add measured slower: its per-row loads
    // made the epilogue the bottleneck, fz2 0.97 -> 1.48 ms at 720p level 0)
    DVC_CHECK_ARG(d.nseg >= 1 && d.nseg <= 4 && d.T >= 1 && d.T < 256 && d.cout % 16 == 0 && d.residual == nullptr,
                  DVC_ERR_UNSUPPORTED, "fused conv: bad descriptor (identity skips are 1x1 segments, not residuals)");
    FzParams p;
    memset(&p, 0, sizeof(p));
    constexpr int CG = 2;
    const int bn = choose_bn(d.cout, CG, 16);
    DVC_CHECK_ARG(bn >= 16 && (bn / CG) % 8 == 0, DVC_ERR_UNSUPPORTED, "no N tile for cout=%d", d.cout);
    p.bn = bn;
    p.T = d.T;
    p.H = d.H;
    p.W = d.W;
    p.cout = d.cout;
    p.tiles_x = (d.W + FZ_BX - 1) / FZ_BX;
    p.tiles_y = (d.H + FZ_BY - 1) / FZ_BY;
    p.nbox = d.T * p.tiles_x * p.tiles_y;
    p.ntile_n = d.cout / bn;
    p.nwork = ((p.nbox + CG - 1) / CG) * p.ntile_n;
    {   // few frames per call: narrower N tiles while the call fills less than half a wave (as the TMA
        // engine; N-splitting keeps each output's K order, results stay bit-identical for any T)
        if (g_fz_sms == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&g_fz_sms, cudaDevAttrMultiProcessorCount, dev);
        }
        const char *e = dvc_knob("DVC_FZ_NARROW");
        const bool narrow = e ? atoi(e) != 0 : true;
        const int half_wave = g_fz_sms / CG / 2, mboxes = (p.nbox + CG - 1) / CG;
        while (narrow && mboxes * p.ntile_n < half_wave) {
            int nb = 0;
            for (int c = p.bn - 16; c >= 64 && !nb; c -= 16)
                if (d.cout % c == 0 && (c / CG) % 8 == 0) nb = c;
            if (!nb) break;
            p.bn = nb;
            p.ntile_n = d.cout / nb;
            p.nwork = mboxes * p.ntile_n;
        }
    }
    p.bias0 = d.bias0;
    p.bias1 = d.bias1;
    p.out = d.out;
    p.stats = reinterpret_cast<float *>(d.stats_out);
    if (dvc_knob("DVC_FZ_XNOSTATS")) p.stats = nullptr;   // timing experiment only: results are wrong
    p.coef = reinterpret_cast<const float2 *>(d.coef);
    DVC_CHECK_ARG(((uintptr_t)d.coef & 15) == 0 && d.cop % 2 == 0, DVC_ERR_ARG, "fused conv: coefficient alignment");
    p.cop = d.cop;
    p.cs = d.cs;
    p.has_carry = d.carry_pad != nullptr;
    p.carry_pad = d.carry_pad;
    p.cs_pad = d.cs_pad;
    p.nseg = d.nseg;
    dvc_status st;
    DVC_CHECK_ARG(!p.has_carry || (((uintptr_t)d.carry_pad & 15) == 0 && d.cs_pad % 8 == 0), DVC_ERR_ARG,
                  "fused conv: padded carry must have 16-byte rows");
    int nb = 0;
    const void *bw[2] = {nullptr, nullptr};
    for (int s = 0; s < d.nseg; ++s) {
        const FzDesc::Seg &g = d.seg[s];
        DVC_CHECK_ARG(g.c % 16 == 0 && g.src != nullptr && ((uintptr_t)g.src & 15) == 0 && g.cglob0 % 2 == 0,
                      DVC_ERR_UNSUPPORTED, "fused conv: segment channels / alignment");
        int idx = -1;
        for (int k = 0; k < nb; ++k)
            if (bw[k] == g.w) idx = k;
        if (idx < 0) {
            DVC_CHECK_ARG(nb < 2, DVC_ERR_UNSUPPORTED, "at most two weight matrices per conv");
            idx = nb++;
            bw[idx] = g.w;
            if (g.packed) {
                long rows = 0;   // the map covers every segment sharing this packed block
                for (int s2 = 0; s2 < d.nseg; ++s2)
                    if (d.seg[s2].w == g.w) {
                        const long r = d.seg[s2].col0 + (long)d.seg[s2].taps * ((d.seg[s2].c + 63) / 64) * d.cout;
                        if (r > rows) rows = r;
                    }
                st = make_bmap_rows(&p.bmap[idx], g.w, d.dt, rows, 64, p.bn / CG);
            } else
                st = make_bmap_rows(&p.bmap[idx], g.w, d.dt, d.cout, g.w_ld, p.bn / CG);
            if (st != DVC_OK) return st;
        }
        p.seg[s] = FzSeg{g.src, g.c, g.cglob0, g.taps, g.transform, g.shift, idx, g.col0, g.tapstride, g.packed};
        if (!g.transform) {
            DVC_CHECK_ARG(g.taps == 1, DVC_ERR_UNSUPPORTED, "fused conv: raw segments are 1x1");
            st = make_box_map(&p.smap[s], g.src, d.dt, d.T, d.H, d.W, g.c, FZ_BX, FZ_BY);
        } else {
            DVC_CHECK_ARG(g.taps == 9, DVC_ERR_UNSUPPORTED, "fused conv: transformed segments are 3x3");
            st = make_halo_map(&p.hmap[s], g.src, d.dt, d.T, d.H, d.W, g.c);
            if (st == DVC_OK) st = make_halo_map(&p.wmap[s], g.src, d.dt, d.T, d.H, d.W, g.c, 64);
        }
        if (st != DVC_OK) return st;
    }
    if (p.has_carry) {
        st = make_halo_map(&p.cmap, d.carry_pad, d.dt, 1, d.H, d.W, d.cs_pad);
        if (st != DVC_OK) return st;
    }
    p.idesc = make_idesc(d.dt == DVC_BF16, 128 * CG, p.bn);
    {
        static const int sw_env = dvc_knob("DVC_FZ_SW") ? atoi(dvc_knob("DVC_FZ_SW")) : 1;
        p.sw_mode = sw_env;
    }
    // shared memory: tile slots, weight stages, residual tile; fill the 227 KB budget with weight stages
    {
        const char *e = dvc_knob("DVC_FZ_NTF");
        p.ntf = e ? atoi(e) : 4;
        if (p.ntf < 2 || p.ntf > FZ_MAX_NTF) p.ntf = 4;
    }
    p.nraw = 0;
    for (int s = 0; s < d.nseg; ++s)
        if (!d.seg[s].transform) p.nraw = 2;
    if (p.nraw) {
        // raw-heavy convs (1x1 shortcut chunks >= 2x the 3x3 chunks, e.g. up3.r0's 720 -> 240 conv2):
        // one transform slot less, one raw slot more (same-box A/B: 0.665 -> 0.528 ms); DVC_FZ_NRAW
        // (experiment builds) overrides the depth
        int ntfc = 0, nrawc = 0;
        for (int s = 0; s < d.nseg; ++s) (d.seg[s].transform ? ntfc : nrawc) += (d.seg[s].c + 63) / 64;
        if (nrawc >= 2 * ntfc && !dvc_knob("DVC_FZ_NTF")) p.ntf = 3, p.nraw = 3;
        const char *e = dvc_knob("DVC_FZ_NRAW");
        if (e && atoi(e) >= 2 && atoi(e) <= FZ_MAX_RAW) p.nraw = atoi(e);
    }
    // K-loop order of a work item: the 3x3 (transformed) chunks in segment order, with the raw 1x1
    // chunks spread evenly among them, so the 2-slot raw ring refills during the 9-tap chunks instead
    // of stalling the MMA on back-to-back raw chunks at the end (DVC_FZ_ILV=0: segment order)
    {
        std::vector<int> tfs, raws;
        for (int s = 0; s < d.nseg; ++s)
            for (int ch = 0; ch < (d.seg[s].c + 63) / 64; ++ch) (d.seg[s].transform ? tfs : raws).push_back(s << 6 | ch);
        DVC_CHECK_ARG(!tfs.empty() && tfs.size() + raws.size() <= 64, DVC_ERR_UNSUPPORTED,
                      "fused conv: 1..64 chunks with a 3x3 segment first");
        const char *e = dvc_knob("DVC_FZ_ILV");
        const bool ilv = e ? atoi(e) != 0 : true;
        std::vector<int> ord;
        if (!ilv) {
            for (int s = 0; s < d.nseg; ++s)
                for (int ch = 0; ch < (d.seg[s].c + 63) / 64; ++ch) ord.push_back(s << 6 | ch);
        } else {
            const size_t nt = tfs.size(), nr = raws.size();
            size_t r = 0;
            for (size_t k = 0; k < nt; ++k) {
                ord.push_back(tfs[k]);
                for (const size_t r1 = (k + 1) * nr / nt; r < r1; ++r) ord.push_back(raws[r]);
            }
        }
        DVC_CHECK_ARG(d.seg[ord[0] >> 6].transform, DVC_ERR_UNSUPPORTED, "fused conv: K loop must start with a 3x3 chunk");
        p.nsteps = (int)ord.size();
        for (size_t i = 0; i < ord.size(); ++i) p.ord[i] = (unsigned char)ord[i];
    }
    {   // staged TMA-store epilogue (default; DVC_FZ_EPI=0 in experiment builds: per-thread row stores)
        const char *e = dvc_knob("DVC_FZ_EPI");
        p.epi_tma = e ? atoi(e) : 1;
    }
    p.up2 = d.up2;
    DVC_CHECK_ARG(!d.up2 || (p.epi_tma && d.stats_out == nullptr), DVC_ERR_UNSUPPORTED,
                  "fused conv: the 2x-upsampled output needs the staged epilogue and no statistics");
    DVC_CHECK_ARG(!d.up2 || ((d.up_ho == 0 || d.up_ho == 2 * d.H || d.up_ho == 2 * d.H - 1) &&
                             (d.up_wo == 0 || d.up_wo == 2 * d.W || d.up_wo == 2 * d.W - 1)),
                  DVC_ERR_UNSUPPORTED, "fused conv: upsampled output must be 2H (- 1) x 2W (- 1)");
    if (p.epi_tma) {
        st = make_out_map(&p.omap[0], d.out, d.dt, d.T, d.H, d.W, d.cout, 32, d.up2 ? 2 : 1, d.up_ho, d.up_wo);
        if (st == DVC_OK) st = make_out_map(&p.omap[1], d.out, d.dt, d.T, d.H, d.W, d.cout, 16, d.up2 ? 2 : 1, d.up_ho, d.up_wo);
        if (st != DVC_OK) return st;
    }
    const size_t fixed = 1024 + (size_t)p.ntf * FZ_SLOT + (size_t)p.nraw * FZ_RAW_SLOT +
                         (p.epi_tma ? 2 * kEpiStage : 0) + 8 * (4 + 2 * FZ_MAX_RAW + 3 * FZ_MAX_NTF + 2 * FZ_MAX_BSTAGES) +
                         16 + 2048 /* red */ +
                         1024 /* static */ + 16 + (size_t)2 * d.cout * 4 /* bias */;
    const size_t bstage = (size_t)(p.bn / CG) * 128;
    int nbst = (int)((227 * 1024 - fixed) / bstage);
    {
        const char *e = dvc_knob("DVC_FZ_NB");
        if (e && atoi(e) >= 2 && atoi(e) < nbst) nbst = atoi(e);
    }
    if (nbst > FZ_MAX_BSTAGES) nbst = FZ_MAX_BSTAGES;
    DVC_CHECK_ARG(nbst >= 2, DVC_ERR_UNSUPPORTED, "fused conv: shared memory too small");
    {   // resident weights when one N tile's stages for a whole work item fit (the VAE's 64-channel
        // full-resolution convs: 9-18 stages of 4 KB); DVC_FZ_WRES=0 in experiment builds disables
        int per_item = 0;
        for (int i = 0; i < p.nsteps; ++i) per_item += d.seg[p.ord[i] >> 6].transform ? 9 : 1;
        const char *e = dvc_knob("DVC_FZ_WRES");
        p.wres = (e ? atoi(e) != 0 : true) && p.ntile_n == 1 && per_item <= nbst ? 1 : 0;
        if (p.wres) nbst = per_item;
    }
    p.nb = nbst;
    const size_t smem = fixed - 1024 + (size_t)nbst * bstage;
    static const bool prof = dvc_knob("DVC_FZ_PROF") != nullptr && atoi(dvc_knob("DVC_FZ_PROF")) != 0;
    static unsigned long long *prof_buf = nullptr;
    if (prof) {
        if (!prof_buf) DVC_CUDA(cudaMalloc(&prof_buf, 24 * sizeof(unsigned long long)));
        DVC_CUDA(cudaMemsetAsync(prof_buf, 0, 24 * sizeof(unsigned long long), stream));
        p.prof = prof_buf;
    }
    auto kern = d.dt == DVC_BF16 ? (prof ? conv_fz_kernel<__nv_bfloat16, 2, true> : conv_fz_kernel<__nv_bfloat16, 2, false>)
                                 : (prof ? conv_fz_kernel<__half, 2, true> : conv_fz_kernel<__half, 2, false>);
    {   // host cost: the attribute is set once per kernel / size
        dvc_status ss_ = ensure_smem((const void *)kern, (int)smem);
        if (ss_ != DVC_OK) return ss_;
    }
    if (g_fz_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_fz_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int clusters = g_fz_sms / CG;
    if (clusters > p.nwork) clusters = p.nwork;
    DVC_CUDA(launch_pdl(kern, dim3(clusters * CG), dim3(kFzThreads), smem, stream, CG, p));
    ++g_launches;
    if (prof) {   // diagnostics: per-role wait / total cycles averaged over CTAs (stderr)
        unsigned long long h[24];
        DVC_CUDA(cudaMemcpyAsync(h, prof_buf, sizeof(h), cudaMemcpyDeviceToHost, stream));
        DVC_CUDA(cudaStreamSynchronize(stream));
        const double n = (double)(h[20] ? h[20] : 1), nl = n / CG;
        fprintf(stderr,
                "fzprof T=%d %dx%d K=%d N=%d segs=%d | mma(leader) tempty %.0f tffull %.0f bfull %.0f tot %.0f | "
                "epi resfull %.0f tfull %.0f statbar %.0f tot %.0f | tf rawfull %.0f bar %.0f fence %.0f tot %.0f | "
                "prod tfempty %.0f tot %.0f | bprod bempty %.0f tot %.0f\n",
                d.T, d.H, d.W, 0, d.cout, d.nseg, h[0] / nl, h[1] / nl, h[2] / nl, h[3] / nl,
                h[4] / n, h[5] / n, h[6] / n, h[7] / n, h[8] / n, h[9] / n, h[10] / n, h[11] / n, h[12] / n, h[15] / n, h[16] / n,
                h[19] / n);
    }
    return check_launch("conv_fz_kernel");
}

}  // namespace dvc
