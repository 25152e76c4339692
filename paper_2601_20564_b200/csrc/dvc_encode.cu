// dvc_encode.cu -- a1 + a2 in one persistent tcgen05 kernel: PixelUnshuffle (s = 8) fused with the
// Latent Channel Expansion 1x1 conv (192 -> c_lat, + bias), SURVEY a1/a2 (R12-R14).
//
// The unshuffle is pure TMA addressing.  The frames [T][3][H][W] are viewed as the 4D tensor
//     (x: W, dy: 8, hb: H/8, tc: 3T)     (x fastest; strides 2 B, 2W B, 16W B, 2HW B)
// and one box {64, 8, 16, 3} (no swizzle; 128-byte rows = 64 pixels = 8 latent columns) is the
// 8 x 16 latent-pixel output box with all 192 unshuffled channels k = c*64 + dy*8 + dx.  With
// x = 8 wb + dx it lands in shared memory as
//     [c][hb][dy][wb][dx]
// which IS the canonical K-major no-swizzle UMMA layout of the A tile: a core matrix (8 latent
// pixels of one row x 8 consecutive k) is 128 contiguous bytes, core matrices adjacent in K (dy,
// dy+1) are 128 B apart (LBO), adjacent in M (next latent row) 1024 B apart (SBO); channel c
// starts 16 KB further.  So the 192-channel latent never exists in memory, and no thread touches
// the A operand: the frames go HBM -> TMA -> tensor core.
//
// GEMM per tile: M = 128 latent pixels, N = c_lat (<= 256), K = 192 (12 MMAs of K = 16); the
// expansion weights [c_lat][192] stay resident in shared memory (3 SW128 boxes).  Two TMEM
// accumulators (2 x N fp32 columns) let the epilogue (bias, 16-bit store) of tile i overlap the
// MMAs of tile i+1.  The A operand streams through a ring of 16 KB colour planes (one
// {64, 8, 16, 1} box = one K block of 64 each, three per tile), each refilled as soon as its four
// MMAs retire.  The epilogue stages 64 columns at a time (SWIZZLE_128B, 128-byte output rows = whole
// L2 lines) and keeps up to four TMA stores in flight; the stores are the bound (measured on the
// B200, 720p x 32: 94 us with 32-column chunks and 2 stores in flight -> 82 us; loads alone 49 us).
// Warps (256 threads): 0 TMA producer, 1 TMEM allocator + MMA issuer, 4-7 epilogue.
// HBM-bound by design: per tile 48 KB of frames in, 128 x c_lat x 2 B of latent out.
#include <cuda.h>
#include <cstdlib>
#include "dvc_conv.cuh"
#include "dvc_ptx.cuh"
#include "dvc_epilogue.cuh"

namespace dvc {

constexpr int ENC_BX = 8, ENC_BY = 16;         // latent pixels per tile (128 MMA rows)
constexpr int ENC_A_BYTES = 3 * 64 * 128 * 2;  // 49152: {64, 8, 16, 3} 16-bit box
constexpr int ENC_PLANE = 64 * 128 * 2;         // 16384: one colour plane {64, 8, 16, 1}
constexpr int ENC_NPLANE = 2 * ENC_A_BYTES / ENC_PLANE;   // 6: A-region capacity in colour planes
constexpr int ENC_THREADS = 384;                // 16-bit frames: warps 4-7 and 8-11 = two epilogue groups
constexpr int ENC_U8_THREADS = 384;             // + warps 8-11: the u8 -> 16-bit converters
constexpr int ENC_U8_HALF = 64 * 192;           // u8 staging slot: 64 frame rows x 64 pixels x 3 bytes

template <typename T> struct Pk2;
template <> struct Pk2<__nv_bfloat16> {
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};
template <> struct Pk2<__half> {
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};

struct EncParams {
    CUtensorMap amap;   // 4D frames view, box {64, 8, 16, 3}, no swizzle (u8: 3D bytes view, box {192, 64, 1})
    CUtensorMap bmap;   // expansion weights [c_lat][192], box {64, c_lat}, SW128
    int T, h, w, c_lat;
    int tiles_x, tiles_y, ntiles;
    const void *bias;
    void *out;          // latent [T][h][w][c_lat]
    CUtensorMap omap[3];   // latent, box {32 | 16, 8, 16, 1} SW64 / SW32, [2]: {64, 8, 16, 1} SW128 (staged epilogue)
    int wide;              // c_lat % 64 == 0: 64-column chunks, 128-byte output rows (omap[2], 16 KB staging)
    int nplane;            // 16-bit path: A ring depth in colour planes (wide: 4, the last two planes'
                           // 32 KB hold two more staging tiles -> 4 stores in flight; else 6)
    uint32_t idesc;
};

// U8: the frames are 8-bit HWC [T][H][W][3] (R14: value RNE16(u / 255)).  The TMA cannot convert or
// de-interleave, so warp 0 streams half tiles (64 frame rows x 64 pixels x 3 bytes) into two staging
// slots and four converter warps (8-11) write the same [c][hb][dy][wb][dx] 16-bit A tile the 16-bit
// path gets from the TMA; the MMA and epilogue are shared.
template <typename T, bool U8>
__global__ void __launch_bounds__(U8 ? ENC_U8_THREADS : ENC_THREADS, 1) encode_kernel(const __grid_constant__ EncParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int N = p.c_lat;
    const int B_CHUNK = N * 128;               // one 64-column SW128 box of the weights
    uint8_t *sA = smem;                        // [2][ENC_A_BYTES]
    uint8_t *sB = sA + 2 * ENC_A_BYTES;        // [3][B_CHUNK]
    uint64_t *a_full = reinterpret_cast<uint64_t *>(sB + 3 * B_CHUNK);   // [6] (u8: [2] whole tiles)
    uint64_t *a_empty = a_full + ENC_NPLANE;
    uint64_t *tfull = a_empty + ENC_NPLANE;
    uint64_t *tempty = tfull + 2;
    uint64_t *b_full = tempty + 2;
    uint64_t *u_full = b_full + 2;    // [2] u8 staging slot landed (U8)
    uint64_t *u_empty = u_full + 2;   // [2] u8 staging slot converted (U8)
    uint8_t *sU = sB + 3 * B_CHUNK + 2048;   // [2][ENC_U8_HALF] u8 staging (U8; after barriers + bias)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(u_empty + 2);
    float *sbias = reinterpret_cast<float *>(tmem_slot + 4);   // [c_lat]
    uint8_t *sStage = sB + 3 * B_CHUNK + 2048;   // [2] epilogue staging (16-bit frames; U8 uses it for sU)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ncols = 2 * N <= 128 ? 128 : 2 * N <= 256 ? 256 : 512;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < ENC_NPLANE; ++i) {
            mbar_init(&a_full[i], U8 ? 8 : 1);   // U8: 4 converter warps x 2 half tiles
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], U8 ? 4 : 8);   // epilogue warps (16-bit frames: two groups of 4)
            mbar_init(&u_full[i], 1);
            mbar_init(&u_empty[i], 4);
        }
        mbar_init(&b_full[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
        tma_prefetch(&p.amap);
        tma_prefetch(&p.bmap);
    }
    if (warp == 1) tmem_alloc<1>(smem_u32(tmem_slot), ncols);
    for (int i = tid; i < N; i += (U8 ? ENC_U8_THREADS : ENC_THREADS)) sbias[i] = Elem<T>::to_f(reinterpret_cast<const T *>(p.bias)[i]);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();     // predecessor grid complete: activations may be read / written
    griddep_launch();   // the successor may be scheduled on SMs that free up

    if (warp == 0) {
        // ===================== TMA producer =====================
        const uint32_t issue = lane == 0;
        if (issue) {
            const uint32_t bb = smem_u32(&b_full[0]);
            mbar_arrive_expect_tx_addr(bb, (uint32_t)(3 * B_CHUNK));
            for (int kc = 0; kc < 3; ++kc) tma_load_2d_a(smem_u32(sB + kc * B_CHUNK), &p.bmap, bb, kc * 64, 0);
        }
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int per = p.tiles_x * p.tiles_y;
            const int t = tile / per, rem = tile - t * per;
            const int by = rem / p.tiles_x, bx = rem - by * p.tiles_x;
            if constexpr (U8) {   // two half tiles into the staging slots (the converters free them)
                for (int hh = 0; hh < 2; ++hh) {
                    mbar_wait_spin(&u_empty[stage], phase ^ 1);
                    if (issue) {
                        const uint32_t fb = smem_u32(&u_full[stage]);
                        mbar_arrive_expect_tx_addr(fb, ENC_U8_HALF);
                        tma_load_3d(smem_u32(sU + stage * ENC_U8_HALF), &p.amap, fb, bx * ENC_BX * 8 * 3,
                                    by * ENC_BY * 8 + hh * 64, t);
                    }
                    __syncwarp();
                    if (++stage == 2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                continue;
            }
#pragma unroll 1
            for (int c = 0; c < 3; ++c) {   // one colour plane per ring slot
                mbar_wait_spin(&a_empty[stage], phase ^ 1);
                if (issue) {
                    const uint32_t fb = smem_u32(&a_full[stage]);
                    mbar_arrive_expect_tx_addr(fb, ENC_PLANE);
                    tma_load_4d(smem_u32(sA + stage * ENC_PLANE), &p.amap, fb, bx * ENC_BX * 8, 0, by * ENC_BY, t * 3 + c);
                }
                __syncwarp();
                if (++stage == p.nplane) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
        const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
        int stage = 0, it = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
            const int buf = it & 1;
            const uint32_t use = (uint32_t)(it >> 1) & 1;
            mbar_wait_spin(&tempty[buf], use ^ 1);
            const uint32_t d = tmem + (uint32_t)(buf * N);
            if constexpr (!U8) {
                // colour c = K block of 64 in ring slot `stage` (K step of 16 = dy += 2 = +256 B); B = weight
                // box c (K step = +32 B inside the swizzled 128-byte rows); each plane is released by the
                // commit of its own four MMAs
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    mbar_wait_spin(&a_full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_lo = desc_lo(sA0 + (uint32_t)(stage * ENC_PLANE), 128);
                    const uint32_t b_lo = desc_lo(sB0 + (uint32_t)(c * B_CHUNK), 16);
                    mma_stage<1>(d, a_lo, desc_hi_noswz(1024), 16u, b_lo, kDescHiSw128, p.idesc, 4u, c ? 1u : 0u,
                                 smem_u32(&a_empty[stage]));
                    if (++stage == p.nplane) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                commit_elected<1>(smem_u32(&tfull[buf]));
                continue;
            }
            mbar_wait_spin(&a_full[stage], phase);
            tc_fence_after();
            const uint32_t a_base = sA0 + (uint32_t)(stage * ENC_A_BYTES);
            // colour c = K block of 64: A at +16 KB per colour (K step of 16 = dy += 2 = +256 B),
            // B = weight box c (K step = +32 B inside the swizzled 128-byte rows)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint32_t a_lo = desc_lo(a_base + (uint32_t)(c * 16384), 128);
                const uint32_t b_lo = desc_lo(sB0 + (uint32_t)(c * B_CHUNK), 16);
                if (c < 2)
                    mma_stage_nc<1>(d, a_lo, desc_hi_noswz(1024), 16u, b_lo, kDescHiSw128, p.idesc, 4u, c ? 1u : 0u);
                else
                    mma_stage<1>(d, a_lo, desc_hi_noswz(1024), 16u, b_lo, kDescHiSw128, p.idesc, 4u, 1u,
                                 smem_u32(&a_empty[stage]));
            }
            commit_elected<1>(smem_u32(&tfull[buf]));
            if (++stage == 2) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else if (U8 && warp >= 8) {
        // ===================== u8 -> 16-bit converters (R14) =====================
        // half tile hh = frame rows [64 hh, 64 hh + 64) of the tile = latent rows hb in [8 hh, 8 hh + 8);
        // thread item j: (hbl, dy, wb) reads the 24 bytes of 8 pixels x 3 colours of frame row
        // 8 hbl + dy and writes three 16-byte core-matrix rows (one per colour) of the A tile.
        // u / 255 as fp32 product with the fp32 constant 1/255, rounded once to 16 bits: equal to the
        // exactly rounded RNE16(u / 255) for all 256 values in fp16 and bf16 (tests: exhaustive, G2).
        const int ct = tid - 256;
        int astage = 0, ustage = 0;
        uint32_t aphase = 0, uphase = 0;
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            mbar_wait(&a_empty[astage], aphase ^ 1);
            uint8_t *A = sA + astage * ENC_A_BYTES;
            for (int hh = 0; hh < 2; ++hh) {
                mbar_wait(&u_full[ustage], uphase);
                const uint8_t *U = sU + ustage * ENC_U8_HALF;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = ct + 128 * k;
                    const int wb = j & 7, dy = (j >> 3) & 7, hbl = j >> 6;
                    const uint2 *src = reinterpret_cast<const uint2 *>(U + (hbl * 8 + dy) * 192 + wb * 24);
                    const uint2 q0 = src[0], q1 = src[1], q2 = src[2];
                    const uint32_t wv[6] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y};
                    uint32_t o[3][4];
#pragma unroll
                    for (int dx = 0; dx < 8; dx += 2) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const int b0 = 3 * dx + c, b1 = 3 * (dx + 1) + c;
                            const float f0 = (float)((wv[b0 >> 2] >> (8 * (b0 & 3))) & 0xFFu) * (1.0f / 255.0f);
                            const float f1 = (float)((wv[b1 >> 2] >> (8 * (b1 & 3))) & 0xFFu) * (1.0f / 255.0f);
                            o[c][dx >> 1] = Pk2<T>::pack(f0, f1);
                        }
                    }
                    const int hb = hh * 8 + hbl;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        *reinterpret_cast<uint4 *>(A + c * 16384 + hb * 1024 + dy * 128 + wb * 16) =
                            make_uint4(o[c][0], o[c][1], o[c][2], o[c][3]);
                }
                fence_proxy_async();   // generic smem writes -> the tensor core (async proxy)
                __syncwarp();
                if (lane == 0) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&u_empty[ustage])) : "memory");
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&a_full[astage])) : "memory");
                }
                if (++ustage == 2) {
                    ustage = 0;
                    uphase ^= 1;
                }
            }
            if (++astage == 2) {
                astage = 0;
                aphase ^= 1;
            }
        }
    } else if (warp >= 4 && (warp < 8 || !U8)) {
        // ===================== epilogue: + bias, 16-bit store =====================
        // 16-bit frames: two warpgroups (warps 4-7, 8-11) take alternate 64-column chunks, each with its
        // own two staging tiles, named barrier and store issuer (the stores are the bound)
        const int q4 = warp & 3;
        const int g = (warp - 4) >> 2;
        const int r = q4 * 32 + lane;   // accumulator row = latent pixel (r / 8, r % 8) of the box
        T *out = reinterpret_cast<T *>(p.out);
        int it = 0;
        int wpar = 0;   // wide staging tile, cycled across tiles (a tile may have fewer chunks than tiles)
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
            const int buf = it & 1;
            const uint32_t use = (uint32_t)(it >> 1) & 1;
            const int per = p.tiles_x * p.tiles_y;
            const int t = tile / per, rem = tile - t * per;
            const int y = (rem / p.tiles_x) * ENC_BY + r / ENC_BX, x = (rem % p.tiles_x) * ENC_BX + r % ENC_BX;
            const bool live = y < p.h && x < p.w;
            T *orow = out + (((size_t)t * p.h + y) * p.w + x) * N;
            mbar_wait(&tfull[buf], use);
            tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * N);
            if constexpr (!U8) {   // staged epilogue (dvc_epilogue.cuh): one TMA store per 32 columns
                const bool issuer = warp == 4 + 4 * g && lane == 0;
                const int bx0 = (rem % p.tiles_x) * ENC_BX, by0 = (rem / p.tiles_x) * ENC_BY;
                int par = 0;
                if (g == 1 && (!p.wide || N <= 64)) {   // the second group has no chunk of this tile
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
                    continue;
                }
                if (p.wide) {
                    // 64 columns per chunk: one SWIZZLE_128B [128 rows][128 B] staging tile (16-byte unit j of
                    // row r at j ^ (r & 7)) and one TMA store of the {64, 8, 16, 1} box -- whole 128-byte
                    // output rows (full L2 lines) and half the barrier round trips of the 32-column form
                    // four staging tiles (two in the A region, nplane == 4): group g cycles tiles 2g, 2g + 1
#pragma unroll 1
                    for (int cc = 64 * g; cc < N; cc += 128, wpar ^= 1) {
                        const int par = 2 * g + wpar;
                        uint32_t v[4][16];
#pragma unroll
                        for (int k = 0; k < 4; ++k) tmem_ld16_nowait(taddr + (uint32_t)(cc + 16 * k), v[k]);
#pragma unroll
                        for (int k = 0; k < 4; ++k) tmem_wait16(v[k]);
                        if (cc + 128 >= N) {   // this group's part of the accumulator is drained
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0)
                                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
                        }
                        uint8_t *st = par < 2 ? sStage + par * (2 * kEpiStage) : sA + (par + 2) * ENC_PLANE;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int c = cc + 8 * j;
                            const uint32_t *w = &v[j >> 1][(j & 1) * 8];
                            uint4 u;
                            u.x = live ? Pk2<T>::pack(__uint_as_float(w[0]) + sbias[c], __uint_as_float(w[1]) + sbias[c + 1]) : 0u;
                            u.y = live ? Pk2<T>::pack(__uint_as_float(w[2]) + sbias[c + 2], __uint_as_float(w[3]) + sbias[c + 3]) : 0u;
                            u.z = live ? Pk2<T>::pack(__uint_as_float(w[4]) + sbias[c + 4], __uint_as_float(w[5]) + sbias[c + 5]) : 0u;
                            u.w = live ? Pk2<T>::pack(__uint_as_float(w[6]) + sbias[c + 6], __uint_as_float(w[7]) + sbias[c + 7]) : 0u;
                            *reinterpret_cast<uint4 *>(st + r * 128 + ((j ^ (r & 7)) << 4)) = u;
                        }
                        fence_proxy_async_smem();
                        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");   // this group's barrier
                        if (issuer) {
                            tma_store_4d(&p.omap[2], smem_u32(st), cc, bx0, by0, t);
                            bulk_commit_group();
                            bulk_wait_group_read<1>();   // the group's other staging tile is reusable
                        }
                        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
                    }
                    continue;
                }
#pragma unroll 1
                for (int cc = 0; cc < N; cc += 32, par ^= 1) {
                    uint32_t va[16], vb[16];
                    const bool two = cc + 16 < N;
                    tmem_ld16_nowait(taddr + (uint32_t)cc, va);
                    if (two) tmem_ld16_nowait(taddr + (uint32_t)(cc + 16), vb);
                    tmem_wait16(va);
                    if (two) tmem_wait16(vb);
                    if (cc + 32 >= N) {   // accumulator drained
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
                    }
                    float f[32];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        f[i] = __uint_as_float(va[i]) + sbias[cc + i];
                        f[16 + i] = two ? __uint_as_float(vb[i]) + sbias[cc + 16 + i] : 0.f;
                    }
                    epi_stage_chunk<T>(f, live, two, r, q4, lane, sStage + par * kEpiStage, &p.omap[0], &p.omap[1],
                                       issuer, true, cc, bx0, by0, t, nullptr, nullptr);
                }
                continue;
            }
#pragma unroll 1
            for (int cc = 0; cc < N; cc += 32) {
                uint32_t va[16], vb[16];
                const bool two = cc + 16 < N;
                tmem_ld16_nowait(taddr + (uint32_t)cc, va);
                if (two) tmem_ld16_nowait(taddr + (uint32_t)(cc + 16), vb);
                tmem_wait16(va);
                if (two) tmem_wait16(vb);
                if (live) {
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        if (h2 == 1 && !two) break;
                        const uint32_t *v = h2 ? vb : va;
                        const int n = cc + 16 * h2;
                        Vec8<T> lo, hi;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            lo.v[i] = Elem<T>::from_f(__uint_as_float(v[i]) + sbias[n + i]);
                            hi.v[i] = Elem<T>::from_f(__uint_as_float(v[8 + i]) + sbias[n + 8 + i]);
                        }
                        *reinterpret_cast<Vec8<T> *>(orow + n) = lo;
                        *reinterpret_cast<Vec8<T> *>(orow + n + 8) = hi;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
        }
    }
    if (!U8 && (warp == 4 || warp == 8) && lane == 0) bulk_wait_group<0>();   // every staged store has landed
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<1>(tmem, ncols);
    }
}

// ----------------------------------------------------------------- host side
PFN_encodeTiled_t get_encode_fn();
dvc_status make_bmap_rows(CUtensorMap *map, const void *ptr, dvc_dtype dt, long rows, long cols, int box_rows);
dvc_status make_out_map_box(CUtensorMap *map, void *ptr, dvc_dtype dt, int T, int H, int W, int C, int box_c, int BX,
                            int BY, int up = 1);

bool encode_tma_applicable(dvc_dtype dt, int H, int W, int s, int c_lat) {
    return (dt == DVC_BF16 || dt == DVC_F16) && s == 8 && H % 8 == 0 && W % 8 == 0 && c_lat >= 16 && c_lat <= 256 &&
           c_lat % 16 == 0 && (W / 8) >= 1;
}

static int g_enc_sms = 0;

// frame_dt: DVC_BF16 / DVC_F16 ([T][3][H][W], must equal dt) or DVC_U8 ([T][H][W][3] bytes, W % 16 == 0)
dvc_status encode_tma_run(const void *frames, dvc_dtype frame_dt, int T, int H, int W, const void *w_exp,
                          const void *b_exp, int c_lat, void *latent, dvc_dtype dt, cudaStream_t stream) {
    const bool u8 = frame_dt == DVC_U8;
    DVC_CHECK_ARG(encode_tma_applicable(dt, H, W, 8, c_lat) && (u8 ? W % 16 == 0 : frame_dt == dt),
                  DVC_ERR_UNSUPPORTED, "encode: unsupported shape / dtype combination");
    DVC_CHECK_ARG(((uintptr_t)frames & 15) == 0 && ((uintptr_t)latent & 15) == 0, DVC_ERR_ARG,
                  "encode: frames / latent must be 16-byte aligned");
    EncParams p;
    memset(&p, 0, sizeof(p));
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUresult r;
    if (u8) {   // bytes [T][H][3W], box {192 bytes = 64 pixels x 3, 64 rows, 1}
        cuuint64_t gdim[3] = {(cuuint64_t)W * 3, (cuuint64_t)H, (cuuint64_t)T};
        cuuint64_t gstride[2] = {(cuuint64_t)W * 3, (cuuint64_t)H * W * 3};
        cuuint32_t box[3] = {ENC_BX * 8 * 3, 64, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        r = enc(&p.amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(frames), gdim, gstride, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {    // frames [T][3][H][W] as (x, dy, hb, t*3 + c)
        cuuint64_t gdim[4] = {(cuuint64_t)W, 8, (cuuint64_t)(H / 8), (cuuint64_t)T * 3};
        cuuint64_t gstride[3] = {(cuuint64_t)W * 2, (cuuint64_t)W * 16, (cuuint64_t)H * W * 2};
        cuuint32_t box[4] = {ENC_BX * 8, 8, ENC_BY, 1};   // one colour plane per TMA
        cuuint32_t estr[4] = {1, 1, 1, 1};
        r = enc(&p.amap, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                const_cast<void *>(frames), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (frames) failed (%d)", (int)r);
    dvc_status st = make_bmap_rows(&p.bmap, w_exp, dt, c_lat, 192, c_lat);
    if (st != DVC_OK) return st;
    p.T = T;
    p.h = H / 8;
    p.w = W / 8;
    p.c_lat = c_lat;
    p.tiles_x = (p.w + ENC_BX - 1) / ENC_BX;
    p.tiles_y = (p.h + ENC_BY - 1) / ENC_BY;
    p.ntiles = T * p.tiles_x * p.tiles_y;
    p.bias = b_exp;
    p.out = latent;
    p.idesc = make_idesc(dt == DVC_BF16, 128, c_lat);
    const size_t smem = u8 ? 1024 + 2 * ENC_A_BYTES + 3 * (size_t)c_lat * 128 + 2048 + 2 * ENC_U8_HALF
                           : 1024 + 2 * ENC_A_BYTES + 3 * (size_t)c_lat * 128 + 2048 + 4 * kEpiStage;
    if (!u8) {
        st = make_out_map_box(&p.omap[0], latent, dt, T, H / 8, W / 8, c_lat, 32, ENC_BX, ENC_BY);
        if (st == DVC_OK) st = make_out_map_box(&p.omap[1], latent, dt, T, H / 8, W / 8, c_lat, 16, ENC_BX, ENC_BY);
        p.wide = c_lat % 64 == 0;
        if (st == DVC_OK && p.wide) st = make_out_map_box(&p.omap[2], latent, dt, T, H / 8, W / 8, c_lat, 64, ENC_BX, ENC_BY);
        p.nplane = p.wide ? 4 : ENC_NPLANE;
        if (st != DVC_OK) return st;
    }
    auto kern = dt == DVC_BF16 ? (u8 ? encode_kernel<__nv_bfloat16, true> : encode_kernel<__nv_bfloat16, false>)
                               : (u8 ? encode_kernel<__half, true> : encode_kernel<__half, false>);
    {   // host cost: the attribute is set once per kernel / size
        dvc_status ss_ = ensure_smem((const void *)kern, (int)smem);
        if (ss_ != DVC_OK) return ss_;
    }
    if (g_enc_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_enc_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = p.ntiles < g_enc_sms ? p.ntiles : g_enc_sms;
    ProfSlot s0 = prof_begin(stream);
    DVC_CUDA(launch_pdl(kern, dim3(grid), dim3(u8 ? ENC_U8_THREADS : ENC_THREADS), smem, stream, 1, p));
    ++g_launches;
    prof_end_aux(s0, stream, u8 ? "encode_u8" : "encode");
    return check_launch("encode_kernel");
}

}  // namespace dvc
