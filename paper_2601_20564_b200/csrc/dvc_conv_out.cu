// dvc_conv_out.cu -- the Pruned VAE Decoder's output head (f2, P:110 / Table 8; readings
// R29-R31): out = conv3x3(SiLU(GN_out(x))) + b, x = [T][H][W][C] at full resolution (C = width[0],
// 64 at the paper's widths), out = [T][H][W][out_ch] (out_ch = 3 RGB channels).
//
// Why its own kernel.  With 3 output channels the conv does 3 * 9 * C * 2 = 3456 FLOP per pixel against
// 2C = 128 bytes of x: 27 FLOP/byte, far below the tensor-core ridge (~190 FLOP/byte), so it is bound
// by reading x once from HBM (118 MB per 720p frame) and by the GN + SiLU transform (one MUFU op per
// element), not by MMAs.  The fused engine (dvc_conv_fz.cu) ran it as a 16-channel UMMA tile whose
// per-item pipeline (36 N=16 MMAs and 9 weight stages per 128-pixel box) was latency-bound (ncu:
// issue 33 %, tensor 9 %, memory 13 %, 1.17 ms for 8 frames) and wrote a padded 16-channel tensor a
// copy kernel then sliced.  An implicit GEMM over the 9 taps (K = 9C) would also read every operand
// row 9 times from shared memory (one ldmatrix per tap).  This kernel instead puts the taps in N:
//
//   P[p][tap, o] = sum_c h[p][c] * W[o][tap][c]      for every HALO pixel p (K = C, N = 9 out_ch <= 32)
//   out[y][x][o] = b[o] + sum_{ky,kx} P[(y + ky - 1, x + kx - 1)][(ky, kx), o]
//
// so each transformed operand element is loaded into an MMA fragment exactly once, and the 9-term
// shifted sum is an fp32 epilogue over P in shared memory.  Per CTA (two per SM, persistent, 8
// warps, so that one CTA's transform + MMA phase overlaps the other's epilogue and barriers) and
// per 8 x 32-pixel output tile of one frame:
//   * one TMA halo box {8 ch, 34, 10} per 8-channel group lands unswizzled as [C/8][352 rows][8 ch]
//     (zero-filled outside the tensor); two stages, the tile after next loads while this one runs;
//   * warp w takes halo pixel groups w, w + 8, w + 16 (22 m16 groups = 352 >= 340 rows): ldmatrix of
//     the raw 16-bit rows straight into mma.m16n8k16 A fragments, the transform applied in
//     registers -- hz = x * scale/2 + shift/2 (the GN affine folded, gn_coef_box_run),
//     h = hz + hz * tanh(hz) = SiLU(z) (R23, the fused engine's form), rounded to 16 bit, 0 for halo
//     pixels outside the frame (zero padding applies after the transform, H3) -- then C/16 x 4 MMAs
//     against the n8 weight fragments held in registers (fp32 accumulation);
//   * P (fp32, [9 out_ch][356]) overwrites the consumed stage; the epilogue (one thread per output
//     pixel) sums the 9 shifted taps in fp32, adds the bias, rounds once to 16 bit and writes the
//     out_ch channels straight into the frame tensor (no padded intermediate, no slice launch).
// mma.sync is deliberate: the op is HBM/MUFU-bound at N = 27, tcgen05's throughput would sit idle.
#include <algorithm>
#include <type_traits>
#include "dvc_conv.cuh"
#include "dvc_ptx.cuh"

namespace dvc {

PFN_encodeTiled_t get_encode_fn();

namespace {

constexpr int CO_TH = 8, CO_TW = 32;                   // output tile (rows x columns)
constexpr int CO_HY = CO_TH + 2, CO_HX = CO_TW + 2;    // halo
constexpr int CO_HP = CO_HY * CO_HX;                   // 340 halo pixels
constexpr int CO_NG = (CO_HP + 15) / 16;               // 22 m16 pixel groups
constexpr int CO_ROWS = CO_NG * 16;                    // 352 operand rows per channel group
constexpr int CO_GP = CO_ROWS * 16;                    // 5632 bytes (128-byte multiple)
constexpr int CO_WARPS = 8;                            // groups w, w + 8, w + 16 of warp w
constexpr int CO_GPW = (CO_NG + CO_WARPS - 1) / CO_WARPS;   // 3
constexpr int CO_THREADS = CO_WARPS * 32;               // = one thread per output pixel
constexpr int CO_MAX_OC = 3;                           // N = 9 out_ch <= 32: four n8 tiles
constexpr int CO_NT = 4;
constexpr int CO_PXS = 356;                            // P row pitch (floats): >= 352, = 4 mod 32
static_assert(CO_GP % 128 == 0 && CO_PXS >= CO_ROWS && CO_PXS % 32 == 4 && CO_THREADS == CO_TH * CO_TW,
              "conv_out layout");

struct CoParams {
    const float2 *coef;   // [T][C] (scale, shift)
    const void *w;        // [>= oc][3][3][C] OHWI (rows past oc unused)
    const void *b;        // [>= oc]
    void *out;            // [T][H][W][oc]
    int T, H, W, oc;
    int ntx, nty, ntiles;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr)
                 : "memory");
}

template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint2 b) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
            "{%0, %1, %2, %3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

template <typename T> struct CoPk;
template <> struct CoPk<__nv_bfloat16> {
    static __device__ __forceinline__ void unpack(uint32_t u, float &a, float &b) {
        a = __uint_as_float(u << 16), b = __uint_as_float(u & 0xFFFF0000u);
    }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};
template <> struct CoPk<__half> {
    static __device__ __forceinline__ void unpack(uint32_t u, float &a, float &b) {
        const __half2 h = *reinterpret_cast<const __half2 *>(&u);
        const float2 f = __half22float2(h);
        a = f.x, b = f.y;
    }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};

// SiLU(z) = hz + hz * tanh(hz), hz = z / 2 (one MUFU op; R23)
__device__ __forceinline__ float co_silu_h(float hz) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(hz));
    return fmaf(hz, y, hz);
}

// shared memory: 2 stages of max([C/8][CO_GP] operand, [9 oc][CO_PXS] fp32 P) | 2 mbarriers.  C = 64: the
// operand is ONE SWIZZLE_128B halo box {64, 34, 10} (128-byte rows, 8x fewer TMA row requests than eight
// 16-byte-row boxes), [CO_ROWS][128 B] with 16-byte unit u of row r at u ^ (r & 7); the same bytes.
__host__ __device__ inline int co_stage_bytes(int C) {
    const int op = (C / 8) * CO_GP, pb = 9 * CO_MAX_OC * CO_PXS * 4;
    return ((op > pb ? op : pb) + 1023) / 1024 * 1024;   // 1024-aligned stages (SW128 pattern)
}
__host__ __device__ inline int co_smem_bytes(int C) { return 2 * co_stage_bytes(C) + 16; }

template <typename T, int KS>   // KS = C / 16
__global__ void __launch_bounds__(CO_THREADS, 2) conv_out_kernel(const __grid_constant__ CUtensorMap xmap, CoParams p) {
    constexpr int C = KS * 16;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sbytes = co_stage_bytes(C);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + 2 * sbytes);

    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_prefetch(&xmap);
    }
    // B = [K = C channels][N = 32 columns n = tap * oc + o] in mma.m16n8k16 "col" fragments: lane
    // (column nt*8 + lane/4, q = lane%4) holds W[o][tap][16 ks + 2q, +1] and [16 ks + 8 + 2q, +1]
    const int oc = p.oc, ncol = 9 * oc, q = lane & 3, g = lane >> 2;
    uint2 bw[KS][CO_NT];
    {
        const uint16_t *w = reinterpret_cast<const uint16_t *>(p.w);
#pragma unroll
        for (int nt = 0; nt < CO_NT; ++nt) {
            const int n = nt * 8 + g, tap = n / oc, o = n - tap * oc;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                uint2 v = make_uint2(0u, 0u);
                if (n < ncol) {
                    const uint16_t *row = w + ((size_t)o * 9 + tap) * C + ks * 16 + 2 * q;
                    v.x = (uint32_t)row[0] | ((uint32_t)row[1] << 16);
                    v.y = (uint32_t)row[8] | ((uint32_t)row[9] << 16);
                }
                bw[ks][nt] = v;
            }
        }
    }
    float bias[CO_MAX_OC];
#pragma unroll
    for (int o = 0; o < CO_MAX_OC; ++o) bias[o] = o < oc ? (float)reinterpret_cast<const T *>(p.b)[o] : 0.f;
    __syncthreads();
    griddep_wait();   // x and the GN coefficients come from the preceding launches

    const int per_frame = p.ntx * p.nty;
    auto issue = [&](int tile, int s) {   // thread 0: the halo boxes of one tile into stage s
        const int t = tile / per_frame, rem = tile - t * per_frame;
        const int ty = rem / p.ntx, tx = rem - ty * p.ntx;
        const uint32_t bar = smem_u32(&full[s]);
        mbar_arrive_expect_tx_addr(bar, (uint32_t)(C / 8) * CO_HP * 16u);
        const uint32_t dst = smem_u32(smem + s * sbytes);
        if constexpr (KS == 4) {
            tma_load_4d(dst, &xmap, bar, 0, tx * CO_TW - 1, ty * CO_TH - 1, t);
        } else {
#pragma unroll
            for (int cg = 0; cg < C / 8; ++cg)
                tma_load_4d(dst + cg * CO_GP, &xmap, bar, cg * 8, tx * CO_TW - 1, ty * CO_TH - 1, t);
        }
    };
    int tile = blockIdx.x;
    if (tid == 0) {
        if (tile < p.ntiles) issue(tile, 0);
        if (tile + (int)gridDim.x < p.ntiles) issue(tile + gridDim.x, 1);
    }
    // ldmatrix: lane supplies row (lane % 8) + 8 (mi & 1) of matrix mi = lane / 8, channel half mi >> 1
    const uint32_t lrow = (uint32_t)(((lane & 7) + 8 * ((lane >> 3) & 1)) * 16 + ((lane >> 4) & 1) * CO_GP);

    for (int k = 0; tile < p.ntiles; ++k, tile += gridDim.x) {
        const int s = k & 1;
        const int t = tile / per_frame, rem = tile - t * per_frame;
        const int ty = rem / p.ntx, tx = rem - ty * p.ntx;
        const int y0 = ty * CO_TH, x0 = tx * CO_TW;
        uint8_t *st = smem + s * sbytes;
        // GN affine of this lane's channels 16 ks + 8 h + 2q + {0, 1} (scale, shift; halved at use)
        const float4 *cf = reinterpret_cast<const float4 *>(p.coef + (size_t)t * C + 2 * q);
        mbar_wait(&full[s], (uint32_t)(k >> 1) & 1u);

        // ---- P for the warp's pixel groups: raw rows -> fragments -> SiLU(GN) -> MMAs
        float acc[CO_GPW][CO_NT][4];
        const uint32_t sbase = smem_u32(st) + lrow;
#pragma unroll
        for (int i = 0; i < CO_GPW; ++i) {
            const int grp = warp + i * CO_WARPS;
#pragma unroll
            for (int nt = 0; nt < CO_NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = acc[i][nt][2] = acc[i][nt][3] = 0.f;
            if (grp >= CO_NG) continue;   // warp-uniform
            bool live[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = grp * 16 + g + 8 * h;
                const int hy = r / CO_HX, hx = r - hy * CO_HX;
                const int y = y0 - 1 + hy, x = x0 - 1 + hx;
                live[h] = r < CO_HP && y >= 0 && y < p.H && x >= 0 && x < p.W;
            }
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                uint32_t a[4];
                if constexpr (KS == 4) {   // SW128 rows: this lane's row rr, 8-channel unit 2 ks + (lane >> 4)
                    const uint32_t rr = (uint32_t)(grp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1));
                    const uint32_t u = (uint32_t)(2 * ks + ((lane >> 4) & 1));
                    const uint32_t row_addr = smem_u32(st) + rr * 128u;   // TMA swizzles on absolute address bits
                    ldsm_x4(row_addr + ((u ^ ((row_addr >> 7) & 7u)) << 4), a[0], a[1], a[2], a[3]);
                } else {
                    ldsm_x4(sbase + (uint32_t)(grp * 16 * 16 + 2 * ks * CO_GP), a[0], a[1], a[2], a[3]);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {   // a[j]: row g + 8 (j & 1), channels 16 ks + 8 (j >> 1) + 2q, +1
                    const float4 c = __ldg(cf + ks * 8 + (j >> 1) * 4);
                    float v0, v1;
                    CoPk<T>::unpack(a[j], v0, v1);
                    const uint32_t hv = CoPk<T>::pack(co_silu_h(0.5f * fmaf(v0, c.x, c.y)),
                                                      co_silu_h(0.5f * fmaf(v1, c.z, c.w)));
                    a[j] = live[j & 1] ? hv : 0u;
                }
#pragma unroll
                for (int nt = 0; nt < CO_NT; ++nt) mma16816<T>(acc[i][nt], a, bw[ks][nt]);
            }
        }
        __syncthreads();   // every fragment of stage s read: P may overwrite it

        // ---- P[n][row] (fp32, column-major, pitch CO_PXS): d0/d1 row g, d2/d3 row g + 8
        float *P = reinterpret_cast<float *>(st);
#pragma unroll
        for (int i = 0; i < CO_GPW; ++i)
#pragma unroll
            for (int nt = 0; nt < CO_NT; ++nt) {
                const int n = nt * 8 + 2 * q, r = (warp + i * CO_WARPS) * 16 + g;
                if (r >= CO_ROWS) continue;
                if (n < ncol) P[n * CO_PXS + r] = acc[i][nt][0], P[n * CO_PXS + r + 8] = acc[i][nt][2];
                if (n + 1 < ncol)
                    P[(n + 1) * CO_PXS + r] = acc[i][nt][1], P[(n + 1) * CO_PXS + r + 8] = acc[i][nt][3];
            }
        __syncthreads();

        // ---- out = b + sum of the 9 shifted taps, one thread per output pixel
        {
            const int oy = tid >> 5, ox = tid & 31, y = y0 + oy, x = x0 + ox;
            if (y < p.H && x < p.W) {
                T *out = reinterpret_cast<T *>(p.out) + (((size_t)t * p.H + y) * p.W + x) * oc;
#pragma unroll
                for (int o = 0; o < CO_MAX_OC; ++o) {
                    if (o >= oc) break;
                    float sum = 0.f;
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap) {
                        const int ky = tap / 3, kx = tap % 3;
                        sum += P[(tap * oc + o) * CO_PXS + (oy + ky) * CO_HX + ox + kx];
                    }
                    out[o] = (T)(sum + bias[o]);
                }
            }
        }
        __syncthreads();   // P read: stage s may be refilled
        if (tid == 0 && tile + 2 * (int)gridDim.x < p.ntiles) {
            fence_proxy_async_smem();   // generic accesses to stage s before the async-proxy overwrite
            issue(tile + 2 * gridDim.x, s);
        }
    }
    griddep_launch();
}

int g_co_sms = 0;

}  // namespace

bool conv_out_applicable(int C, int oc, dvc_dtype dt) {
    return dt != DVC_F32 && C % 16 == 0 && C >= 16 && C <= 64 && oc >= 1 && oc <= CO_MAX_OC;
}

// x [T][H][W][C] 16-bit, coef float2 [T][C], w OHWI [>= oc][3][3][C], b [>= oc] -> out [T][H][W][oc]
dvc_status conv_out_run(const void *x, const void *coef, int T, int H, int W, int C, const void *w, const void *b,
                        int oc, void *out, dvc_dtype dt, cudaStream_t stream) {
    DVC_CHECK_ARG(conv_out_applicable(C, oc, dt) && T >= 1 && H >= 1 && W >= 1, DVC_ERR_UNSUPPORTED,
                  "conv_out: C=%d oc=%d dtype %d", C, oc, (int)dt);
    DVC_CHECK_ARG(((uintptr_t)x & 15) == 0 && ((uintptr_t)coef & 15) == 0 && ((uintptr_t)w & 3) == 0, DVC_ERR_ARG,
                  "conv_out: alignment");
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
    cuuint64_t gstride[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    const bool wide = C == 64;   // one SWIZZLE_128B box of all 64 channels (else one 8-channel box per group)
    cuuint32_t box[4] = {wide ? 64u : 8u, (cuuint32_t)CO_HX, (cuuint32_t)CO_HY, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                     const_cast<void *>(x), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     wide ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled (conv_out) failed (%d)", (int)r);

    CoParams p;
    p.coef = reinterpret_cast<const float2 *>(coef);
    p.w = w, p.b = b, p.out = out;
    p.T = T, p.H = H, p.W = W, p.oc = oc;
    p.ntx = (W + CO_TW - 1) / CO_TW, p.nty = (H + CO_TH - 1) / CO_TH;
    const long ntiles = (long)T * p.ntx * p.nty;
    DVC_CHECK_ARG(ntiles < (1L << 31), DVC_ERR_UNSUPPORTED, "conv_out: too many tiles");
    p.ntiles = (int)ntiles;

    const int smem = co_smem_bytes(C);
    using Kern = void (*)(const CUtensorMap, CoParams);
    const bool bf = dt == DVC_BF16;
    const Kern kern = C == 16   ? (bf ? conv_out_kernel<__nv_bfloat16, 1> : conv_out_kernel<__half, 1>)
                      : C == 32 ? (bf ? conv_out_kernel<__nv_bfloat16, 2> : conv_out_kernel<__half, 2>)
                      : C == 48 ? (bf ? conv_out_kernel<__nv_bfloat16, 3> : conv_out_kernel<__half, 3>)
                                : (bf ? conv_out_kernel<__nv_bfloat16, 4> : conv_out_kernel<__half, 4>);
    dvc_status st = ensure_smem(reinterpret_cast<const void *>(kern), smem);
    if (st != DVC_OK) return st;
    if (g_co_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_co_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = (int)std::min<long>(ntiles, 2L * g_co_sms);
    DVC_CUDA(launch_pdl(kern, dim3(grid), dim3(CO_THREADS), smem, stream, 1, map, p));
    ++g_launches;
    return DVC_OK;
}

}  // namespace dvc
