// dvc_conv_ws.cu -- persistent, warp-specialised tcgen05 implicit-GEMM
// convolution for same-resolution 3x3 / 1x1 convolutions (the ResBlock convs
// a5/a7/a8 and conv_in/conv_out).
//
// GEMM view: M = output pixels, tiled per frame into spatial boxes of
// BY x BX <= 128 pixels (one 128-row MMA tile each); N = C_out in tiles of
// BN <= 256; K = sum over segments of taps x C_src in 64-channel stages.
// For tap (dy, dx) the A tile of a box is the TMA box of the NHWC activation
// at (x0+dx, y0+dy): the tensor map's out-of-bounds zero fill IS the conv's
// zero padding, so no address arithmetic runs on the SMs.
//
// CG = 2 (default): a CTA pair (cluster of 2) runs tcgen05.mma.cta_group::2
// with M = 256 (each CTA's box = 128 rows) and N = BN; each CTA stages its own
// A box and HALF of the weight tile, halving per-SM weight traffic.
// Per CTA: 2 TMEM accumulator buffers of BN fp32 columns, so the epilogue of
// tile i overlaps the MMAs of tile i+1.
//
// Warp roles (256 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer (leader CTA only issues), warps 4-7 epilogue (TMEM -> registers ->
// bias / residual -> global), warps 2-3 idle.
#include <cuda.h>
#include <cstdlib>
#include "dvc_conv.cuh"
#include "dvc_ptx.cuh"
#include "dvc_boxstats.cuh"
#include "dvc_epilogue.cuh"

namespace dvc {

struct WsParams {
    CUtensorMap amap[4];   // per segment: 4D {C, W, H, T}, box {64, BX, BY, 1}, SW128, OOB zero
    CUtensorMap bmap[2];   // weights 2D {K, C_out}, box {64, BN/CG}, SW128
    int bidx[4], seg_c[4], seg_taps[4], seg_col0[4], seg_tapstride[4], seg_packed[4];
    int seg_nch[4], seg_klast[4];
    int seg_stride[4];   // 1: same resolution; 2: stride-2 conv (TMA element stride 2 over the input)   // 64-channel stages per tap; K=16 steps in the last one
    int nseg;
    int T, H, W, cout, bn;
    int BX, BY, tiles_x, tiles_y, nbox, ntile_n, nwork;
    const void *bias0, *bias1, *residual;
    void *out;
    uint32_t idesc;
    float *stats;   // per-channel box statistics of the output (dvc_boxstats.cuh), or null
    int geglu;      // ConvDesc::geglu: 32-column batches = 16 values + 16 gates -> 16 outputs
    int fp8;        // ConvDesc::fp8: E4M3 operands, 128 channels per 128-byte stage row, kind::f8f6f4
    int chw;        // channels per stage: 64 (16-bit) or 128 (fp8)
    float out_scale;
    int epi_tma;           // staged epilogue (dvc_epilogue.cuh): TMA-stored 32-column chunks
    CUtensorMap omap[2];   // output [T][H][W][cout], box {32 | 16, BX, BY, 1}, SW64 / SW32
    int up2;               // ConvDesc::up2: omap describes the upsampled output, element stride 2
};

// EG epilogue warpgroups (warps 4-7, and 8-11 when EG = 2): group g drains the 32-column chunks
// g, g + EG, ... of each accumulator with its own staging tiles, named barrier (1 + g) and store issuer,
// so convolutions whose K loop is short (the f1 transformer linears, K = 240 .. 960) are not bound by
// one warpgroup's drain / stage / store round trips per chunk
template <int EG> constexpr int ws_threads() { return 128 + 128 * EG; }

template <typename T, int CG, int STAGES, int EG>
__global__ void __launch_bounds__(ws_threads<EG>(), 1) conv_ws_kernel(const __grid_constant__ WsParams p) {
    constexpr int kWsThreads = ws_threads<EG>();
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so the compiler keeps the
    // shared address space (an integer round trip would turn every access generic)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int BN = p.bn, BNH = p.bn / CG;
    constexpr int A_STAGE = 128 * 128;
    const int B_STAGE = BNH * 128;
    uint8_t *sA = smem;
    uint8_t *sB = sA + STAGES * A_STAGE;
    uint8_t *sStage = sB + STAGES * B_STAGE;   // [EG][2] epilogue staging (epi_tma)
    uint64_t *full = reinterpret_cast<uint64_t *>(sStage + (p.epi_tma ? 2 * EG * kEpiStage : 0));
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    float *red = reinterpret_cast<float *>(tmem_slot + 4);   // [EG][2][2][4][32] box-statistics staging
    float *sbias = red + 512 * EG;   // [1 or 2][cout] bias0 (, bias1) in fp32 (16-byte aligned: even barrier count)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const int cluster_id = blockIdx.x / CG, nclusters = gridDim.x / CG;
    const uint32_t ncols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], CG * 4 * EG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
        for (int s = 0; s < p.nseg; ++s) tma_prefetch(&p.amap[s]);
        tma_prefetch(&p.bmap[0]);
    }
    if (warp == 1) tmem_alloc<CG>(smem_u32(tmem_slot), ncols);
    for (int i = tid; i < p.cout; i += kWsThreads) {
        sbias[i] = p.bias0 ? Elem<T>::to_f(reinterpret_cast<const T *>(p.bias0)[i]) : 0.f;
        if (p.bias1) sbias[p.cout + i] = Elem<T>::to_f(reinterpret_cast<const T *>(p.bias1)[i]);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();     // predecessor grid complete: activations may be read / written
    griddep_launch();   // the successor may be scheduled on SMs that free up

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        // the whole warp walks the (warp-uniform) loop; lane 0 issues through guard
        // predicates (no divergent region per stage)
        int stage = 0;
        uint32_t phase = 0;
        const uint32_t a_bytes = (uint32_t)(p.BX * p.BY * 128);
        const uint32_t tx = (uint32_t)CG * (a_bytes + (uint32_t)B_STAGE);
        const uint32_t issue = lane == 0;
        const uint32_t expect = issue && rank == 0;   // the leader's barrier counts both CTAs' bytes
        const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
        const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
        const uint32_t lead_full0 = CG == 2 ? mapa_shared(full0, 0) : full0;
        for (int w = cluster_id; w < p.nwork; w += nclusters) {
            const int q = w / p.ntile_n, nt = w - q * p.ntile_n;
            const int n0 = nt * BN + (int)rank * BNH;
            const int box = q * CG + (int)rank;
            int t, y0, x0;
            if (box < p.nbox) {
                const int per = p.tiles_x * p.tiles_y;
                t = box / per;
                const int rem = box - t * per;
                y0 = (rem / p.tiles_x) * p.BY;
                x0 = (rem % p.tiles_x) * p.BX;
            } else {   // padding box of the last pair: fully out of bounds -> zeros
                t = p.T;
                y0 = x0 = 0;
            }
            for (int s = 0; s < p.nseg; ++s) {
                const int nch = p.seg_nch[s], taps = p.seg_taps[s], sst = p.seg_stride[s];
                const CUtensorMap *am = &p.amap[s];
                const CUtensorMap *bm = &p.bmap[p.bidx[s]];
                const bool packed = p.seg_packed[s] != 0;
                for (int tap = 0; tap < taps; ++tap) {
                    const int dy = taps == 9 ? tap / 3 - 1 : 0;
                    const int dx = taps == 9 ? tap % 3 - 1 : 0;
                    // weight tile origin: column block of this tap, or (packed) its row block
                    const int bc0 = packed ? 0 : p.seg_col0[s] + tap * p.seg_tapstride[s];
                    const int br0 = packed ? p.seg_col0[s] + tap * nch * p.cout + n0 : n0;
                    const int bcs = packed ? 0 : p.chw, brs = packed ? p.cout : 0;
                    for (int ch = 0; ch < nch; ++ch) {
                        mbar_wait_spin_addr(empty0 + 8 * stage, phase ^ 1);
                        const uint32_t lb = CG == 2 ? lead_full0 + 8 * stage : full0 + 8 * stage;
                        mbar_expect_tx_if(expect, full0 + 8 * stage, tx);
                        tma_load_4d_if<CG>(issue, sA0 + stage * A_STAGE, am, lb, ch * p.chw, sst * x0 + dx, sst * y0 + dy, t);
                        tma_load_2d_if<CG>(issue, sB0 + stage * B_STAGE, bm, lb, bc0 + ch * bcs, br0 + ch * brs);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA) =====================
        // converged warp; mma_stage() elects the issuing lane inside its asm
        if (rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
            const uint32_t a_lo0 = desc_lo(smem_u32(sA), 16), b_lo0 = desc_lo(smem_u32(sB), 16);
            for (int w = cluster_id; w < p.nwork; w += nclusters, ++it) {
                const int buf = it & 1;
                const uint32_t use = (uint32_t)(it >> 1) & 1;
                mbar_wait_spin(&tempty[buf], use ^ 1);   // epilogues of both CTAs drained this buffer
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * BN);
                uint32_t acc = 0;
                for (int s = 0; s < p.nseg; ++s) {
                    const int nch = p.seg_nch[s], taps = p.seg_taps[s];
                    const uint32_t klast = (uint32_t)p.seg_klast[s];
                    for (int tap = 0; tap < taps; ++tap) {
                        for (int ch = 0; ch < nch; ++ch) {
                            mbar_wait_spin_addr(full0 + 8 * stage, phase);
                            tc_fence_after();
                            if (p.fp8)
                                mma_stage_f8<CG>(d, a_lo0 + (uint32_t)stage * (A_STAGE >> 4), kDescHiSw128, 2u,
                                                 b_lo0 + (uint32_t)(stage * (B_STAGE >> 4)), kDescHiSw128, p.idesc,
                                                 ch == nch - 1 ? klast : 4u, acc, empty0 + 8 * stage);
                            else
                                mma_stage<CG>(d, a_lo0 + (uint32_t)stage * (A_STAGE >> 4), kDescHiSw128, 2u,
                                              b_lo0 + (uint32_t)(stage * (B_STAGE >> 4)), kDescHiSw128, p.idesc,
                                              ch == nch - 1 ? klast : 4u, acc, empty0 + 8 * stage);
                            acc = 1;
                            if (++stage == STAGES) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                    }
                }
                commit_elected<CG>(smem_u32(&tfull[buf]));
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs) =====================
        const int q4 = warp & 3;                 // TMEM lane quadrant of this warp
        const int g = (warp - 4) >> 2;           // epilogue warpgroup: chunks g, g + EG, ...
        const uint32_t gbar = 1u + (uint32_t)g;  // its named barrier
        float *const gred = red + 512 * g;
        const int r = q4 * 32 + lane;            // accumulator row = pixel of this CTA's box
        const int by = r / p.BX, bx = r - by * p.BX;
        const float *sb0 = p.bias0 ? sbias : nullptr;
        const float *sb1 = p.bias1 ? sbias + p.cout : nullptr;
        const T *res = reinterpret_cast<const T *>(p.residual);
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
            const int per = p.tiles_x * p.tiles_y;
            long m = -1;
            if (box < p.nbox && r < p.BX * p.BY) {
                const int t = box / per, rem = box - t * per;
                const int y = (rem / p.tiles_x) * p.BY + by, x = (rem % p.tiles_x) * p.BX + bx;
                if (y < p.H && x < p.W) m = ((long)t * p.H + y) * p.W + x;
            }
            mbar_wait(&tfull[buf], use);   // long wait (a whole main loop): sleep, leave the issue slots
            tc_fence_after();
            const bool want_stats = p.stats != nullptr && box < p.nbox;   // warp-uniform
            float *stats_box = want_stats ? p.stats + (size_t)box * p.cout * 2 : nullptr;   // box = t * per + bi
            // one 16-column chunk: + bias (fp32, shared memory) + residual, 16-bit store; x = this
            // row's statistics contribution of the stored values
            auto chunk = [&](const uint32_t (&v)[16], int n, float (&x)[32]) {
                float f[16];
                if (m >= 0) {
                    float rv[16];
                    if (res) {   // issue the residual loads first
                        load8(res + m * p.cout + n, *reinterpret_cast<float(*)[8]>(&rv[0]));
                        load8(res + m * p.cout + n + 8, *reinterpret_cast<float(*)[8]>(&rv[8]));
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) * p.out_scale;
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
                    if (res) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] += rv[i];
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
            // 32 columns per step: two tcgen05.ld in flight, two butterflies, one barrier, and the
            // combine split over warps 0 / 1 (canonical order, dvc_boxstats.cuh)
            const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * BN);
            if (p.geglu) {   // f1 GEGLU epilogue: out[m][n/2 + i] = (v_i + b) * gelu(g_i + b')
                const int half = p.cout / 2;
#pragma unroll 1
                for (int cc = 32 * g; cc < BN; cc += 32 * EG) {
                    uint32_t va[16], vb[16];
                    tmem_ld16_nowait(taddr + (uint32_t)cc, va);
                    tmem_ld16_nowait(taddr + (uint32_t)(cc + 16), vb);
                    tmem_wait16(va);
                    tmem_wait16(vb);
                    if (m >= 0) {
                        const int n = nt * BN + cc;
                        float f[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            float a = __uint_as_float(va[i]), gt = __uint_as_float(vb[i]);   // value, gate
                            if (sb0) a += sb0[n + i], gt += sb0[n + 16 + i];
                            f[i] = a * (0.5f * gt * (1.f + erff(gt * 0.70710678118654752f)));
                        }
                        Vec8<T> lo, hi;
                        round_store16<T>(f, lo, hi);
                        *reinterpret_cast<Vec8<T> *>(out + m * half + n / 2) = lo;
                        *reinterpret_cast<Vec8<T> *>(out + m * half + n / 2 + 8) = hi;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    tmem_drained_arrive(CG == 2 ? tempty_leader + (uint32_t)(buf * 8) : smem_u32(&tempty[buf]), CG == 2);
                }
                continue;
            }
            if (p.epi_tma) {   // staged epilogue (dvc_epilogue.cuh)
                const bool issuer = warp == 4 + 4 * g && lane == 0;
                if (32 * g >= BN) {   // no chunk for this group: the accumulator is drained as far as it goes
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        tmem_drained_arrive(CG == 2 ? tempty_leader + (uint32_t)(buf * 8) : smem_u32(&tempty[buf]), CG == 2);
                    continue;
                }
                int bt = p.T, bx0 = 0, by0 = 0;
                if (box < p.nbox) {
                    bt = box / per;
                    const int rem = box - bt * per;
                    by0 = (rem / p.tiles_x) * p.BY;
                    bx0 = (rem % p.tiles_x) * p.BX;
                }
#pragma unroll 1
                for (int cc = 32 * g; cc < BN; cc += 32 * EG, par ^= 1) {
                    const bool two = cc + 16 < BN;   // warp-uniform: 32 or 16 columns
                    const int n = nt * BN + cc;
                    uint32_t va[16], vb[16];
                    tmem_ld16_nowait(taddr + (uint32_t)cc, va);
                    if (two) tmem_ld16_nowait(taddr + (uint32_t)(cc + 16), vb);
                    float rv[32];
                    if (res && m >= 0) {   // the residual loads overlap the TMEM loads
                        load8(res + m * p.cout + n, *reinterpret_cast<float(*)[8]>(&rv[0]));
                        load8(res + m * p.cout + n + 8, *reinterpret_cast<float(*)[8]>(&rv[8]));
                        if (two) {
                            load8(res + m * p.cout + n + 16, *reinterpret_cast<float(*)[8]>(&rv[16]));
                            load8(res + m * p.cout + n + 24, *reinterpret_cast<float(*)[8]>(&rv[24]));
                        }
                    }
                    tmem_wait16(va);
                    if (two) tmem_wait16(vb);
                    if (cc + 32 * EG >= BN) {   // this group's last chunk: its part of the accumulator is drained
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            tmem_drained_arrive(CG == 2 ? tempty_leader + (uint32_t)(buf * 8) : smem_u32(&tempty[buf]), CG == 2);
                        }
                    }
                    float f[32];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        f[i] = __uint_as_float(va[i]) * p.out_scale;
                        f[16 + i] = __uint_as_float(vb[i]) * p.out_scale;
                    }
                    if (sb0) epi_add_bias(f, sb0 + n, two);   // bias0 then bias1, as the other paths
                    if (sb1) epi_add_bias(f, sb1 + n, two);
                    if (res && m >= 0) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) f[i] += rv[i];
                    }
                    epi_stage_chunk<T>(f, m >= 0, two, r, q4, lane, sStage + (2 * g + par) * kEpiStage, &p.omap[0],
                                       &p.omap[1], issuer, box < p.nbox, n, bx0, by0, bt,
                                       want_stats ? stats_box + (size_t)n * 2 : nullptr, gred + par * 256, p.up2 != 0,
                                       gbar);
                }
                continue;
            }
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
                    asm volatile("bar.sync 1, 128;" ::: "memory");   // the 4 epilogue warps
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
    if (p.epi_tma && (warp == 4 || warp == 8) && lane == 0) bulk_wait_group<0>();   // every staged store has landed
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

dvc_status make_box_map(CUtensorMap *map, const void *ptr, dvc_dtype dt, int T, int H, int W, int C, int BX, int BY);
// box {64, BX, BY} of output pixels over a [T][H][W][C] input; stride 2: the TMA walks the input
// with element stride 2 (box {64, 2 BX, 2 BY}, every other pixel), i.e. the stride-2 conv's taps
static dvc_status make_amap(CUtensorMap *map, const void *ptr, dvc_dtype dt, int T, int H, int W, int C, int BX,
                            int BY, int stride) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && (C * 2) % 16 == 0 && (stride == 1 || stride == 2), DVC_ERR_ARG,
                  "activation must be 16-byte aligned");
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)(BX * stride), (cuuint32_t)(BY * stride), 1};
    cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    CUresult r = enc(map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                     const_cast<void *>(ptr), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (activation) failed (%d)", (int)r);
    return DVC_OK;
}
dvc_status make_box_map(CUtensorMap *map, const void *ptr, dvc_dtype dt, int T, int H, int W, int C, int BX, int BY) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && (C * 2) % 16 == 0, DVC_ERR_ARG, "activation must be 16-byte aligned");
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)BX, (cuuint32_t)BY, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                     const_cast<void *>(ptr), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (activation) failed (%d)", (int)r);
    return DVC_OK;
}

dvc_status make_bmap_rows(CUtensorMap *map, const void *ptr, dvc_dtype dt, long rows, long cols, int box_rows);

// Spatial box minimising the number of 128-row MMA tiles per frame.  Frames
// with H >= 32 use the fused engine's 8 x 16 box (dvc_conv_fz.cu) so that every
// producer of a tensor shares one box decomposition (box statistics).
void choose_box(int H, int W, int *BX, int *BY) {
    if (H >= 32 && W >= 8) {
        *BX = 8;
        *BY = 16;
        return;
    }
    long best = -1;
    for (int bx = 1; bx <= W && bx <= 128; ++bx) {
        int by = 128 / bx;
        if (by > H) by = H;
        if (by < 1) continue;
        long cost = (long)((H + by - 1) / by) * ((W + bx - 1) / bx);
        if (best < 0 || cost < best || (cost == best && bx * by > *BX * *BY)) {
            best = cost;
            *BX = bx;
            *BY = by;
        }
    }
}

static int g_num_sms = 0;

template <int CG, int STAGES, int EG>
static size_t ws_smem_bytes(const WsParams &p) {
    return 1024 + (size_t)STAGES * (128 * 128 + (p.bn / CG) * 128) + (p.epi_tma ? 2 * EG * kEpiStage : 0) +
           8 * (2 * STAGES + 4) + 16 + 2048 * EG + (size_t)(p.bias1 ? 2 : 1) * p.cout * 4;   // bias1 staged only when present
}

template <typename T, int CG, int STAGES, int EG>
static dvc_status launch_ws(const WsParams &p, cudaStream_t stream) {
    const size_t smem = ws_smem_bytes<CG, STAGES, EG>(p);
    auto kern = conv_ws_kernel<T, CG, STAGES, EG>;
    {   // host cost: the attribute is set once per kernel / size
        dvc_status ss_ = ensure_smem((const void *)kern, (int)smem);
        if (ss_ != DVC_OK) return ss_;
    }
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int clusters = g_num_sms / CG;
    if (clusters > p.nwork) clusters = p.nwork;
    DVC_CUDA(launch_pdl(kern, dim3(clusters * CG), dim3(ws_threads<EG>()), smem, stream, CG, p));
    ++g_launches;
    return check_launch("conv_ws_kernel");
}

// fp8 (E4M3 bytes) variants of the activation / weight tensor maps: 128 channels = 128 bytes per row
static dvc_status make_amap8(CUtensorMap *map, const void *ptr, int T, int H, int W, int C, int BX, int BY,
                             int stride) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && C % 16 == 0, DVC_ERR_ARG, "fp8 activation must be 16-byte aligned");
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
    cuuint32_t box[4] = {128, (cuuint32_t)(BX * stride), (cuuint32_t)(BY * stride), 1};
    cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(ptr), gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (fp8 activation) failed (%d)", (int)r);
    return DVC_OK;
}
static dvc_status make_bmap8(CUtensorMap *map, const void *ptr, long rows, long cols, int box_rows) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && cols % 16 == 0, DVC_ERR_ARG, "fp8 weights: 16-byte rows");
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)cols};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (fp8 weights) failed (%d)", (int)r);
    return DVC_OK;
}

// output box {c, BX, BY, 1} of a [T][H][W][C] 16-bit tensor for the staged epilogue's TMA store: 32 channels
// (64-byte rows, SWIZZLE_64B) or 16 (32-byte rows, SWIZZLE_32B), matching dvc_epilogue.cuh's staging
// up = 2: (H, W) are the upsampled extents and the map walks x and y with element stride 2, so a
// staged BX x BY box lands on one phase of the 2x grid (the far row / column clipped when H or W is odd)
dvc_status make_out_map_box(CUtensorMap *map, void *ptr, dvc_dtype dt, int T, int H, int W, int C, int box_c, int BX,
                            int BY, int up) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && C % 8 == 0, DVC_ERR_ARG, "conv output alignment");
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)(BX * up), (cuuint32_t)(BY * up), 1};
    cuuint32_t estr[4] = {1, (cuuint32_t)up, (cuuint32_t)up, 1};
    CUresult r = enc(map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, ptr,
                     gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     box_c == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : box_c == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed (%d)", (int)r);
    return DVC_OK;
}

static int engine_from_env() {
    const char *e = dvc_knob("DVC_CONV_ENGINE");
    if (e && (e[0] == '0' || e[0] == '1' || e[0] == '2') && e[1] == 0) return e[0] - '0';
    return 2;
}
int g_ws_cg = engine_from_env();   // 2: CTA-pair MMA (default), 1: single-CTA MMA, 0: gather engine only

bool conv_ws_applicable(const ConvDesc &d) {
    if (g_ws_cg == 0 || d.dt == DVC_F32) return false;
    for (int s = 0; s < d.nseg; ++s) {
        const ConvSeg &g = d.seg[s];
        const bool same = g.mode == SEG_SAME && g.hi == d.ho && g.wi == d.wo;
        // 3x3 / stride 2 / pad 1: ho = ceil(hi / 2)
        const bool down = g.mode == SEG_STRIDE2 && g.taps == 9 && (g.hi + 1) / 2 == d.ho && (g.wi + 1) / 2 == d.wo;
        if (!same && !down) return false;
    }
    return true;
}

dvc_status conv_ws_run(const ConvDesc &d, cudaStream_t stream) {
    dvc_status st = conv_check(d, true);
    if (st != DVC_OK) return st;
    WsParams p;
    memset(&p, 0, sizeof(p));
    const int CG = g_ws_cg == 1 ? 1 : 2;
    const int bn = choose_bn(d.cout, CG, d.geglu ? 32 : 16);   // GEGLU: whole 32-column value/gate blocks
    DVC_CHECK_ARG(bn >= 16 && (bn / CG) % 8 == 0, DVC_ERR_UNSUPPORTED, "no N tile for cout=%d", d.cout);
    DVC_CHECK_ARG(!d.geglu || (bn % 32 == 0 && d.residual == nullptr && d.stats_out == nullptr && d.bias1 == nullptr),
                  DVC_ERR_UNSUPPORTED, "GEGLU epilogue: 32-column tiles, no residual / statistics / second bias");
    p.bn = bn;
    p.geglu = d.geglu;
    p.fp8 = d.fp8;
    p.chw = d.fp8 ? 128 : 64;
    p.out_scale = d.fp8 ? d.out_scale : 1.f;
    p.nseg = d.nseg;
    p.T = d.T;
    p.H = d.ho;
    p.W = d.wo;
    p.cout = d.cout;
    choose_box(d.ho, d.wo, &p.BX, &p.BY);
    p.tiles_x = (d.wo + p.BX - 1) / p.BX;
    p.tiles_y = (d.ho + p.BY - 1) / p.BY;
    p.nbox = d.T * p.tiles_x * p.tiles_y;
    p.ntile_n = d.cout / bn;
    p.nwork = ((p.nbox + CG - 1) / CG) * p.ntile_n;
    {   // few frames per call (streaming / strong scaling: e.g. the 12x20 level at T = 4 has 16 work items
        // for 74 CTA pairs): narrower N tiles while the call fills less than half a wave.  Splitting N
        // leaves every output's K accumulation order unchanged, so results stay bit-identical for any T.
        if (g_num_sms == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        }
        const char *e = dvc_knob("DVC_WS_NARROW");
        const bool narrow = (e ? atoi(e) != 0 : true) && !d.geglu && !d.fp8;
        const int half_wave = g_num_sms / CG / 2, mboxes = (p.nbox + CG - 1) / CG;
        while (narrow && mboxes * p.ntile_n < half_wave) {
            int nb = 0;
            for (int c = p.bn - 16; c >= 64 && !nb; c -= 16)
                if (d.cout % c == 0 && (c / CG) % 8 == 0) nb = c;
            if (!nb) break;
            p.bn = nb;
            p.ntile_n = d.cout / nb;
            p.nwork = mboxes * p.ntile_n;
        }
        const char *eb = dvc_knob("DVC_WS_BN");   // experiment builds: force the N tile
        if (eb && !d.geglu && atoi(eb) >= 16 && d.cout % atoi(eb) == 0 && (atoi(eb) / CG) % 8 == 0) {
            p.bn = atoi(eb);
            p.ntile_n = d.cout / p.bn;
            p.nwork = mboxes * p.ntile_n;
        }
    }
    p.bias0 = d.bias0;
    p.bias1 = d.bias1;
    p.residual = d.residual;
    p.out = d.out;
    int nb = 0;
    const void *bw[2] = {nullptr, nullptr};
    for (int s = 0; s < d.nseg; ++s) {
        const ConvSeg &g = d.seg[s];
        p.seg_stride[s] = g.mode == SEG_STRIDE2 ? 2 : 1;
        st = d.fp8 ? make_amap8(&p.amap[s], g.src, d.T, g.hi, g.wi, g.c_src, p.BX, p.BY, p.seg_stride[s])
                   : make_amap(&p.amap[s], g.src, d.dt, d.T, g.hi, g.wi, g.c_src, p.BX, p.BY, p.seg_stride[s]);
        if (st != DVC_OK) return st;
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
                        const long r = d.seg[s2].w_col0 + (long)d.seg[s2].taps * ((d.seg[s2].c_src + 63) / 64) * d.cout;
                        if (r > rows) rows = r;
                    }
                st = make_bmap_rows(&p.bmap[idx], g.w, d.dt, rows, 64, p.bn / CG);
            } else if (d.fp8)
                st = make_bmap8(&p.bmap[idx], g.w, d.cout, g.w_ld, p.bn / CG);
            else
                st = make_bmap_rows(&p.bmap[idx], g.w, d.dt, d.cout, g.w_ld, p.bn / CG);
            if (st != DVC_OK) return st;
        }
        p.bidx[s] = idx;
        p.seg_packed[s] = g.packed;
        p.seg_c[s] = g.c_src;
        p.seg_nch[s] = (g.c_src + p.chw - 1) / p.chw;
        p.seg_klast[s] = (g.c_src - p.chw * (p.seg_nch[s] - 1)) / (d.fp8 ? 32 : 16);
        p.seg_taps[s] = g.taps;
        p.seg_col0[s] = g.w_col0;
        p.seg_tapstride[s] = g.w_tapstride;
    }
    const int bf = d.dt == DVC_BF16;
    // kind::f8f6f4 with A/B format 0 = E4M3 (the same descriptor fields as kind::f16)
    p.idesc = make_idesc(d.fp8 ? 0 : bf, 128 * CG, p.bn);
    if (d.fp8)
        for (int s = 0; s < d.nseg; ++s)
            DVC_CHECK_ARG(d.seg[s].c_src % 32 == 0 && !d.seg[s].packed && d.seg[s].w_ld % 16 == 0, DVC_ERR_UNSUPPORTED,
                          "fp8 conv: channels multiple of 32, unpacked 16-byte weight rows");
    p.stats = reinterpret_cast<float *>(d.stats_out);
    {   // staged TMA-store epilogue (DVC_WS_EPI=0 in experiment builds: per-thread row stores)
        const char *e = dvc_knob("DVC_WS_EPI");
        p.epi_tma = !d.geglu && (e ? atoi(e) != 0 : true);
    }
    p.up2 = d.up2;
    DVC_CHECK_ARG(!d.up2 || (p.epi_tma && !d.fp8 && d.stats_out == nullptr && (d.up_ho == 2 * d.ho || d.up_ho == 2 * d.ho - 1) &&
                             (d.up_wo == 2 * d.wo || d.up_wo == 2 * d.wo - 1)),
                  DVC_ERR_UNSUPPORTED, "conv: upsampled output needs the staged epilogue, no statistics, 2H(-1) x 2W(-1)");
    if (p.epi_tma) {
        const int oh = d.up2 ? d.up_ho : d.ho, ow = d.up2 ? d.up_wo : d.wo, up = d.up2 ? 2 : 1;
        st = make_out_map_box(&p.omap[0], d.out, d.dt, d.T, oh, ow, d.cout, 32, p.BX, p.BY, up);
        if (st == DVC_OK) st = make_out_map_box(&p.omap[1], d.out, d.dt, d.T, oh, ow, d.cout, 16, p.BX, p.BY, up);
        if (st != DVC_OK) return st;
    }
    if (CG == 2) {
        // two epilogue warpgroups for 1x1 convolutions with a short K loop (<= 16 stages of 64 channels:
        // the f1 transformer linears), where one warpgroup's per-chunk drain / stage / store round trips
        // outlast the MMAs (same box, 720p T = 32: 240 -> 720 423 -> 301 us, 240 -> 240 152 -> 113 us,
        // full U-Net 270 -> 275 frames/s; 3x3 convolutions measured neutral to slightly slower and keep
        // one); 5 operand stages when the second group's staging does not fit beside 6 (DVC_WS_EG in
        // experiment builds forces 1 or 2)
        int kst = 0;
        bool pointwise = true;
        for (int s = 0; s < d.nseg; ++s) {
            kst += p.seg_taps[s] * p.seg_nch[s];
            pointwise = pointwise && p.seg_taps[s] == 1;
        }
        const char *e = dvc_knob("DVC_WS_EG");
        const int eg = (p.epi_tma || p.geglu) && (e ? atoi(e) == 2 : pointwise && kst <= 16) ? 2 : 1;
        if (eg == 2) {
            const bool six = ws_smem_bytes<2, 6, 2>(p) <= 227 * 1024;
            if (bf) return six ? launch_ws<__nv_bfloat16, 2, 6, 2>(p, stream) : launch_ws<__nv_bfloat16, 2, 5, 2>(p, stream);
            return six ? launch_ws<__half, 2, 6, 2>(p, stream) : launch_ws<__half, 2, 5, 2>(p, stream);
        }
        if (bf) return launch_ws<__nv_bfloat16, 2, 6, 1>(p, stream);
        return launch_ws<__half, 2, 6, 1>(p, stream);
    }
    if (bf) return launch_ws<__nv_bfloat16, 1, 4, 1>(p, stream);
    return launch_ws<__half, 1, 4, 1>(p, stream);
}

}  // namespace dvc
