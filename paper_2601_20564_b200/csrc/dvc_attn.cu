// dvc_attn.cu -- f1: the self-attention Transformer2D blocks of the full pruned U-Net
// ("U-Net" of SD-2.1 via AdcSR, P:525 parameter count; readings R24-R27).
//
// One block over X [T][H][W][C] (frames independent, no temporal shift):
//   a  = GN(X)                      gn_affine_kernel  (coefficients from box statistics)
//   h0 = proj_in(a)                 1x1 tensor-core conv (conv_run)
//   l1 = LN1(h0)                    layernorm_kernel  (one warp per pixel)
//   qkv = l1 W_qkv^T                1x1 conv, no bias, [T][N][3C]
//   Qp|Kp|Vp = pack(qkv)            qkv_pack_kernel: per-(frame, head, tile) UMMA images (V transposed)
//   o  = attention(q, k, v)         attn_tc_kernel (tcgen05, S and PV in TMEM)
//   h1 = out(o) + h0                1x1 conv with residual
//   l2 = LN2(h1)
//   f  = ff1(l2)                    1x1 conv C -> 8C
//   g  = f[:4C] * gelu(f[4C:])      geglu_kernel
//   h2 = ff2(g) + h1                1x1 conv 4C -> C with residual
//   Y  = proj_out(h2) + X           1x1 conv with residual (+ box statistics of Y for the next GN)
//
// attn_tc_kernel: one CTA = 256 queries (two 128-row tiles) of one (frame,
// head), warp-specialised: warp 17 streams (K_j, V_j^T) tiles through a 4-stage ring (1D bulk copies of
// the pre-tiled images qkv_pack_kernel writes), warp 16 issues S_t = Q_t K_j^T (M=128, N=128, K=D) and
// O_t += P_t V_j with P read from TMEM, 16 softmax warps (two threads per query row, 64 keys each)
// read S once from TMEM, keep a lazy running maximum (moved only when the tile maximum exceeds it by
// 8 in log2 units, with an in-TMEM rescale of that O row), exponentiate with ex2.approx for 6 of 8
// scores and a degree-3 polynomial on the FMA pipe for 2 of 8 (packed fp32x2 arithmetic), and write P
// as packed 16-bit pairs to TMEM.  TMEM: S0, S1, O0, O1, P0, P1 = 512 columns.  The head_dim-256
// variant (VAE mid attention) keeps one query tile per CTA: S | P | O = 128 + 64 + 256 columns.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include "dvc_conv.cuh"
#include "dvc_norm.cuh"
#include "dvc_ptx.cuh"
#include "dvc_attn.cuh"

namespace dvc {

// ----------------------------------------------------------------- elementwise kernels
template <typename T>
__global__ void __launch_bounds__(256) gn_affine_kernel(const T *__restrict__ x, const float2 *__restrict__ coef,
                                                        T *__restrict__ y, int HW, int C, long total8) {
    griddep_wait();
    const int c8 = C / 8;
    const long stride = (long)gridDim.x * blockDim.x;
    // four independent 16-byte loads in flight per thread per round (the pass is HBM-bound)
    for (long i0 = blockIdx.x * (long)blockDim.x + threadIdx.x; i0 < total8; i0 += 4 * stride) {
        float f[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long i = i0 + u * stride;
            if (i < total8) load8(x + (i / c8) * C + (int)(i % c8) * 8, f[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long i = i0 + u * stride;
            if (i >= total8) break;
            const long pix = i / c8;
            const int c = (int)(i - pix * c8) * 8;
            const float4 *cf = reinterpret_cast<const float4 *>(coef + (size_t)(pix / HW) * C + c);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 s = __ldg(cf + k);   // (scale, shift) of channels c+2k, c+2k+1
                f[u][2 * k] = fmaf(f[u][2 * k], s.x, s.y);
                f[u][2 * k + 1] = fmaf(f[u][2 * k + 1], s.z, s.w);
            }
            store8(y + pix * C + c, f[u]);
        }
    }
    griddep_launch();
}

// LayerNorm over the C channels of each pixel (R24): one warp per pixel, fp32 two-pass
// from registers (C <= 32 * 8 * 4 = 1024).
template <typename T>
__global__ void __launch_bounds__(256) layernorm_kernel(const T *__restrict__ x, const T *__restrict__ gamma,
                                                        const T *__restrict__ beta, T *__restrict__ y, long npix,
                                                        int C, float eps) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const long pix = blockIdx.x * 8L + (threadIdx.x >> 5);
    if (pix < npix) {
        const int c8 = C / 8;
        float v[4][8];
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = (lane + 32 * j) * 8;
            if (c < C) {
                load8(x + pix * C + c, v[j]);
#pragma unroll
                for (int k = 0; k < 8; ++k) s += v[j][k];
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float mean = s / C;
        float q = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = (lane + 32 * j) * 8;
            if (c < C) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float d = v[j][k] - mean;
                    q += d * d;
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        const float rstd = rsqrtf(q / C + eps);
        (void)c8;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = (lane + 32 * j) * 8;
            if (c < C) {
                float g[8], b[8];
                load8(gamma + c, g);
                load8(beta + c, b);
#pragma unroll
                for (int k = 0; k < 8; ++k) v[j][k] = fmaf((v[j][k] - mean) * rstd, g[k], b[k]);
                store8(y + pix * C + c, v[j]);
            }
        }
    }
    griddep_launch();
}

// GEGLU (R24): g[m][j] = f[m][j] * gelu(f[m][C4 + j]), exact erf GELU.
template <typename T>
__global__ void __launch_bounds__(256) geglu_kernel(const T *__restrict__ f, T *__restrict__ g, int C4, long total8) {
    griddep_wait();
    const int c8 = C4 / 8;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total8; i += (long)gridDim.x * blockDim.x) {
        const long m = i / c8;
        const int c = (int)(i - m * c8) * 8;
        float a[8], z[8];
        load8(f + m * (2L * C4) + c, a);
        load8(f + m * (2L * C4) + C4 + c, z);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] *= 0.5f * z[k] * (1.f + erff(z[k] * 0.70710678118654752f));
        store8(g + m * C4 + c, a);
    }
    griddep_launch();
}

// qkv [T][N][3C] -> three pre-tiled operand arrays, one contiguous 128*D block per (frame, head,
// 128-token tile) in exactly the shared-memory image the attention kernel's UMMA descriptors
// read (no-swizzle core matrices), so each tile moves with ONE 1D bulk copy:
//   Qp, Kp [T][heads][ntiles]: element (r, d) of the tile at (d/8)*1024 + r*8 + d%8   (chunk-major)
//   Vp     [T][heads][ntiles]: element (r, d) (key r)  at (r/8)*D*8  + d*8 + r%8    (V^T, K = keys)
// Tokens n >= N of the last tile are zero.  One CTA per (tile, head, frame).
template <typename T, int D, int KT>
__global__ void __launch_bounds__(256) qkv_pack_kernel(const T *__restrict__ qkv, T *__restrict__ qp,
                                                       T *__restrict__ kp, T *__restrict__ vp, int N, int C) {
    griddep_wait();
    constexpr int DCH = D < 64 ? D : 64;   // channels per pass (V^T staged through shared memory)
    __shared__ __align__(16) T sv[128 * DCH];
    const int jt = blockIdx.x, h = blockIdx.y, t = blockIdx.z;
    const int heads = gridDim.y, ntiles = gridDim.x;
    const size_t tile = (((size_t)t * heads + h) * ntiles + jt) * (128 * D);
    constexpr int DC = DCH / 8;
#pragma unroll 1
    for (int d0 = 0; d0 < D; d0 += DCH) {
        for (int i = threadIdx.x; i < 128 * DC; i += 256) {
            const int r = i / DC, kl = i - r * DC, kc = d0 / 8 + kl;
            const int n = jt * 128 + r;
            uint4 q = make_uint4(0, 0, 0, 0), k = q, v = q;
            if (n < N) {
                const T *src = qkv + ((size_t)t * N + n) * 3 * C + h * D + kc * 8;
                q = __ldg(reinterpret_cast<const uint4 *>(src));
                k = __ldg(reinterpret_cast<const uint4 *>(src + C));
                v = __ldg(reinterpret_cast<const uint4 *>(src + 2 * C));
            }
            *reinterpret_cast<uint4 *>(qp + tile + kc * 1024 + r * 8) = q;
            // K in KT-row sub-tiles of the 128-token block (chunk-major inside each)
            *reinterpret_cast<uint4 *>(kp + tile + (r / KT) * (KT * D) + kc * (KT * 8) + (r % KT) * 8) = k;
            *reinterpret_cast<uint4 *>(sv + r * DCH + kl * 8) = v;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 16 * DCH; i += 256) {   // (key chunk, d): 8 consecutive keys of column d
            const int kc = i / DCH, dl = i - kc * DCH;
            Vec8<T> u;
#pragma unroll
            for (int e = 0; e < 8; ++e) u.v[e] = sv[(kc * 8 + e) * DCH + dl];
            const int r0 = kc * 8;   // V^T in KT-key sub-tiles
            *reinterpret_cast<Vec8<T> *>(vp + tile + (r0 / KT) * (KT * D) + ((r0 % KT) / 8) * D * 8 + (d0 + dl) * 8) = u;
        }
        __syncthreads();
    }
    griddep_launch();
}

// FF1 weight / bias rows [8C] -> blocks of 32 = 16 value rows (j) then the 16 gate rows (4C + j),
// the order the GEGLU epilogue of the TMA engine consumes (one row of `cols` elements each)
template <typename T>
__global__ void __launch_bounds__(256) geglu_interleave_kernel(const T *__restrict__ src, T *__restrict__ dst, int C4,
                                                               int cols) {
    griddep_wait();
    const long total = 2L * C4 * cols;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols), c = (int)(i - (long)r * cols);
        const int blk = r >> 5, w = r & 31;
        const int src_row = w < 16 ? blk * 16 + w : C4 + blk * 16 + (w - 16);
        dst[i] = src[(size_t)src_row * cols + c];
    }
    griddep_launch();
}

// ----------------------------------------------------------------- attention, fp32 validation mode
// One thread per (frame, head, query): online softmax over all keys (DVC_F32, R16's 1e-5 gate).
template <int D>
__global__ void __launch_bounds__(128) attn_simt_kernel(const float *__restrict__ qkv, float *__restrict__ out, int N,
                                                        int C, float scale) {
    const int t = blockIdx.z, h = blockIdx.y;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const size_t ld = 3 * (size_t)C;
    const float *q = qkv + ((size_t)t * N + n) * ld + h * D;
    float qr[D], o[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        qr[i] = q[i] * scale;
        o[i] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < N; ++j) {
        const float *k = qkv + ((size_t)t * N + j) * ld + C + h * D;
        const float *v = k + C;
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < D; ++i) s = fmaf(qr[i], k[i], s);
        const float mn = fmaxf(m, s);
        const float a = __expf(m - mn), p = __expf(s - mn);
        l = l * a + p;
#pragma unroll
        for (int i = 0; i < D; ++i) o[i] = fmaf(o[i], a, p * v[i]);
        m = mn;
    }
    float *y = out + ((size_t)t * N + n) * C + h * D;
    const float inv = 1.f / l;
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = o[i] * inv;
}

// ----------------------------------------------------------------- attention, tcgen05
// One CTA = two 128-query tiles (256 queries) of one (frame, head), 18 warps:
//   warps 0-15 softmax: tile (bit 2), TMEM lane quarter (bits 0-1), key half (bit 3); the two
//              threads of a query row each handle 64 of the tile's 128 keys
//   warp 16    MMA issuer (one elected lane): S_t = Q_t K_j^T, PV_t = P_t V_j
//   warp 17    producer: Q tiles once, then a 4-stage ring of (K_j, V_j^T) tiles
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256,+D), O_1 [320,+D), P_0 [384,448),
// P_1 [448,512) (P as packed 16-bit pairs: the PV MMA takes A from TMEM, so neither the P stores
// nor the PV operand reads touch shared memory).
// The MMA warp issues PV_t(j) (accumulating into O_t) then S_t(j+1) as soon as group t has
// written P_t(j) (which also releases S_t(j)), so the two groups drift half an iteration apart.
// TMEM reads are the scarce resource (64 B/clk/SM): each softmax thread reads its S row ONCE
// (128 registers), and O stays in TMEM.  O uses a lazy maximum: a row's reference max m only
// moves (with an in-TMEM rescale of its O row by 2^(m - m_new)) when the tile max exceeds it
// by more than 8 (log2 units), so P <= 2^8 and the rescale is rare.  Because the MMA warp
// issues PV_t(j-1) before S_t(j), the commit that signals S_t(j) also covers PV_t(j-1): when
// group t holds S_t(j), O_t is quiescent and may be rescaled, and P_t may be overwritten.
// Operand tiles arrive as single 1D bulk copies of the pre-tiled blocks qkv_pack_kernel writes
// (a 3D TMA view of the packed qkv moved 16 B per request and capped the kernel at ~2 TB/s of
// L2 reads); all are canonical no-swizzle K-major UMMA layouts:
//   Q/K [rows][D]:  core (r8, kc) at kc*2048 + r8*128   (LBO 2048, SBO 128)
//   V^T [D][keys]:  core (d8, kc) at kc*D*16 + d8*128   (LBO D*16, SBO 128)

// head_dim <= 64: two query tiles per CTA (TMEM S0 S1 | O0 O1 | P0 P1), 4-stage K/V ring, Q double-
// buffered; head_dim 256 (the VAE decoder's single-head mid attention, f2): one tile (S | P | O = 256
// columns), K/V and Q single-buffered (256 KB would not fit twice).
// The kernel is persistent: one CTA per SM walks work items (query-tile group, head, frame) with a
// static stride, keeping its TMEM allocation, barriers and pipelines; the next item's Q load and first
// S MMAs overlap the current item's last PV and output normalisation (a fixed cost that was a third of
// every CTA's time at the 720p level-2 shape, N = 920).
template <int D, int KT = 128>
struct AttnSmem {
    // KT = keys per S tile: 128 (two query tiles per CTA); 64 gives three query tiles per CTA (six
    // softmax warps per SM sub-partition) -- measured slower at 720p level 0 (609 vs 650 TFLOP/s:
    // the per-iteration handshakes double), so only KT = 128 is instantiated
    static constexpr int NT = D <= 64 ? (KT == 64 ? 3 : 2) : 1;   // query tiles per CTA
    static constexpr int STAGES = D <= 64 ? (KT == 64 ? 6 : 4) : 1;
    static constexpr int QB = D <= 64 ? 2 : 1;                     // Q buffers (items in flight)
    static constexpr int THREADS = (8 * NT + 2) * 32;     // 8 softmax warps per tile + MMA + TMA
    static constexpr int Q = 128 * D * 2;        // one query tile
    static constexpr int K = KT * D * 2;         // one key tile
    static constexpr int V = D * KT * 2;         // one transposed value tile
    static constexpr int off_q = 0, off_k = QB * NT * Q, off_v = off_k + STAGES * K;
    static constexpr int off_bar = off_v + STAGES * V;
    // barriers: q_full[2], q_empty[2], kv_full[S], kv_empty[S], then s_full[4], p_full[4], o_full[4],
    // o_free[4] (NT <= 3; one slot of four per query tile), v_full, v_empty (STAGES == 1: K and V move
    // separately -- kv_full / kv_empty then track K alone)
    static constexpr int nbar = 4 + 2 * STAGES + 4 * 4 + 2;
    // [NT tiles][2 key-tile parities][2 halves][128 rows] float exchange of the row maxima (parity double
    // buffer: a thread's write for key tile j+1 never lands in the slot its partner may still be reading
    // for tile j), then [NT][2 halves][128] for the row sums at the end of an item
    static constexpr int off_red = off_bar + nbar * 8 + 16;
    static constexpr int bytes = off_red + NT * 6 * 128 * 4 + 1024;   // + alignment slack
    // TMEM columns (512 allocated)
    // S_t at t*KT, P_t (KT/2 packed columns) at tm_p + t*KT/2, O_t at tm_o + t*64
    static constexpr int tm_o = NT == 3 ? 320 : 256, tm_o_step = NT == 1 ? 0 : 64;
    static constexpr int tm_p = NT == 3 ? 192 : NT == 2 ? 384 : 128, tm_p_step = KT / 2;
};

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x on the FMA pipe (x <= 8 here, lazy maximum): round-to-nearest split x = j + f, f in [-1/2, 1/2], a
// degree-3 fit of 2^f (max relative error 7.5e-5, below the 16-bit rounding of P) and j added
// to the exponent field.  Used for part of every 8-score group so the MUFU ex2 unit (the bound of
// a head_dim-48 softmax: 192 MMA FLOP per exponential) shares the work with the FMA pipe.
#ifndef DVC_ATTN_POLY
#define DVC_ATTN_POLY 2   // scores per 8 computed by ex2_poly2 (even: packed pairs)
#endif
// two lanes at a time with packed fp32x2 adds / FMAs (FADD2 / FFMA2)
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -126.f);
    x.y = fmaxf(x.y, -126.f);
    const float2 mg = make_float2(12582912.f, 12582912.f), nmg = make_float2(-12582912.f, -12582912.f);
    const float2 r = __fadd2_rn(x, mg);
    const float2 j = __fadd2_rn(r, nmg);
    const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
    float2 p = __ffma2_rn(make_float2(0.055172063f, 0.055172063f), f, make_float2(0.24261240f, 0.24261240f));
    p = __ffma2_rn(p, f, make_float2(0.69326103f, 0.69326103f));
    p = __ffma2_rn(p, f, make_float2(0.99992794f, 0.99992794f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(r.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(r.y) << 23)));
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    } else {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
}

template <typename T, int D, int NPOLY, int KT>
__global__ void __launch_bounds__(AttnSmem<D, KT>::THREADS, 1)
    attn_tc_kernel(const T *__restrict__ qp, const T *__restrict__ kp, const T *__restrict__ vp, T *__restrict__ out,
                   int N, int C, int T_, float scale_log2, uint32_t idesc_s, uint32_t idesc_o, int dbg) {
    using L = AttnSmem<D, KT>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(smem);
    const uint32_t bar0 = sb + L::off_bar;
    constexpr int kAttnStages = L::STAGES, NT = L::NT, QB = L::QB;
    const uint32_t q_full = bar0, q_empty = bar0 + 16;   // [QB]
    const uint32_t kv_full = bar0 + 32, kv_empty = kv_full + 8 * kAttnStages;
    const uint32_t s_full = kv_empty + 8 * kAttnStages, p_full = s_full + 32;   // p_full also releases S
    const uint32_t o_full = p_full + 32;   // [t] at o_full + 8 t: O_t final
    const uint32_t o_free = o_full + 32;   // [t]: group t has read O_t (the next item's PV may overwrite it)
    const uint32_t v_full = o_free + 32, v_empty = v_full + 8;   // STAGES == 1 only
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smem + L::off_bar + L::nbar * 8);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int heads = C / D;
    const int ntiles = (N + 127) / 128;                       // 128-token tiles of the packed operands
    const int nqg = (N + 128 * NT - 1) / (128 * NT);           // query-tile groups (one per item)
    const int nitems = nqg * heads * T_;
    const int w_mma = 8 * NT, w_tma = 8 * NT + 1;
    const int nkt = (N + KT - 1) / KT;
    if (tid == 0) {
        uint64_t *b = reinterpret_cast<uint64_t *>(smem + L::off_bar);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&b[i], 1);       // q_full[qb] (expect-tx)
            mbar_init(&b[2 + i], 1);   // q_empty[qb] (tcgen05.commit)
        }
        for (int i = 0; i < kAttnStages; ++i) {
            mbar_init(&b[4 + i], 1);
            mbar_init(&b[4 + kAttnStages + i], 1);
        }
        const int sf = 4 + 2 * kAttnStages;
        for (int i = 0; i < NT; ++i) {
            mbar_init(&b[sf + i], 1);        // s_full[t] (tcgen05.commit)
            mbar_init(&b[sf + 4 + i], 8);    // p_full[t] (8 softmax warps per tile)
            mbar_init(&b[sf + 8 + i], 1);    // o_full[t]
            mbar_init(&b[sf + 12 + i], 8);   // o_free[t] (8 softmax warps per tile)
        }
        mbar_init(&b[sf + 16], 1);   // v_full (expect-tx)
        mbar_init(&b[sf + 17], 1);   // v_empty (tcgen05.commit)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == w_mma) tmem_alloc<1>(smem_u32(tslot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    griddep_wait();

    // The MMA warp and the softmax groups are one latency chain (S -> softmax -> P -> PV, S):
    // they poll without a suspend hint (a suspended try_wait wakes late, measured ~1.6 us per
    // iteration of pure barrier round trips); the TMA producer runs ahead and may sleep.
    // Ring and barrier phases run on per-CTA counters across the work items.
    if (warp == w_tma) {
        // ===================== TMA producer =====================
        if (elect_one()) {
            int jg = 0;
            for (int item = blockIdx.x, it = 0; item < nitems; item += gridDim.x, ++it) {
                const int qg = item % nqg, h = (item / nqg) % heads, t = item / (nqg * heads);
                const size_t base = ((size_t)t * heads + h) * ntiles * (128 * D);   // this (frame, head)
                const int qt = qg * NT, qb = it % QB, use = it / QB;
                const uint32_t nq = (uint32_t)min(NT, ntiles - qt);
                if (use > 0) mbar_wait_addr(q_empty + 8 * qb, (use - 1) & 1);   // the previous user's S MMAs retired
                mbar_arrive_expect_tx_addr(q_full + 8 * qb, nq * L::Q);
                for (uint32_t i = 0; i < nq; ++i)
                    bulk_load(sb + L::off_q + (qb * NT + i) * L::Q, qp + base + (size_t)(qt + i) * 128 * D, L::Q,
                              q_full + 8 * qb);
                for (int j = 0; j < nkt; ++j, ++jg) {
                    const int st = jg % kAttnStages;
                    if constexpr (kAttnStages == 1) {
                        // one buffer each: K(j) lands once S(j-1) has retired (overlapping softmax(j-1) and
                        // PV(j-1)), V(j) once PV(j-1) has (overlapping S(j) and softmax(j))
                        if (jg >= 1) mbar_wait_addr(kv_empty, (jg - 1) & 1);
                        mbar_arrive_expect_tx_addr(kv_full, L::K);
                        bulk_load(sb + L::off_k, kp + base + (size_t)j * KT * D, L::K, kv_full);
                        if (jg >= 1) mbar_wait_addr(v_empty, (jg - 1) & 1);
                        mbar_arrive_expect_tx_addr(v_full, L::V);
                        bulk_load(sb + L::off_v, vp + base + (size_t)j * KT * D, L::V, v_full);
                        continue;
                    }
                    if (jg >= kAttnStages) mbar_wait_addr(kv_empty + 8 * st, ((jg / kAttnStages) - 1) & 1);
                    mbar_arrive_expect_tx_addr(kv_full + 8 * st, L::K + L::V);
                    bulk_load(sb + L::off_k + st * L::K, kp + base + (size_t)j * KT * D, L::K, kv_full + 8 * st);
                    bulk_load(sb + L::off_v + st * L::V, vp + base + (size_t)j * KT * D, L::V, kv_full + 8 * st);
                }
            }
        }
    } else if (warp == w_mma) {
        // ===================== MMA issuer =====================
        if (elect_one()) {
            int jg = 0, cp = 0;   // K/V ring position; P_t(j) handshakes so far
            for (int item = blockIdx.x, it = 0; item < nitems; item += gridDim.x, ++it) {
                const int qb = it % QB;
                mbar_wait_spin_addr(q_full + 8 * qb, (it / QB) & 1);
                tc_fence_after();
                auto issue_s = [&](int tt, int jj) {   // jj: ring position of the key tile
                    const int st = jj % kAttnStages;
                    const uint32_t qa = sb + L::off_q + (qb * NT + tt) * L::Q, ka = sb + L::off_k + st * L::K;
#pragma unroll
                    for (int ks = 0; ks < D / 16; ++ks) {
                        if (dbg & 2) break;   // DVC_ATTN_DEBUG bit 1: no MMAs (pipeline-only timing)
                        const uint64_t ad = ((uint64_t)desc_hi_noswz(128) << 32) | desc_lo(qa + ks * 4096, 2048);
                        const uint64_t bd = ((uint64_t)desc_hi_noswz(128) << 32) | desc_lo(ka + ks * 2 * KT * 16, KT * 16);
                        tc_mma(tmem + tt * KT, ad, bd, idesc_s, ks > 0);
                    }
                    tc_commit_addr(s_full + 8 * tt);
                };
                auto issue_pv = [&](int tt, int jj, bool first) {   // A = P_t from TMEM (8 columns per K step)
                    const int st = jj % kAttnStages;
                    const uint32_t va = sb + L::off_v + st * L::V;
#pragma unroll
                    for (int ks = 0; ks < KT / 16; ++ks) {
                        if (dbg & 2) break;
                        const uint64_t bd = ((uint64_t)desc_hi_noswz(128) << 32) | desc_lo(va + ks * 2 * D * 16, D * 16);
                        tc_mma_ts(tmem + L::tm_o + tt * L::tm_o_step, tmem + L::tm_p + tt * L::tm_p_step + ks * 8, bd,
                                  idesc_o, (!first || ks > 0) ? 1u : 0u);
                    }
                };
                // the first S tiles: S_t columns are free (the previous item's last p_full was awaited)
                mbar_wait_spin_addr(kv_full + 8 * (jg % kAttnStages), (jg / kAttnStages) & 1);
                tc_fence_after();
                for (int tt = 0; tt < NT; ++tt) issue_s(tt, jg);
                if constexpr (kAttnStages == 1) tc_commit_addr(kv_empty);   // K(jg) free once S retires
                for (int j = 0; j < nkt; ++j, ++jg, ++cp) {
                    const bool more = j + 1 < nkt;
                    if constexpr (kAttnStages == 1) {
                        // single K and V buffers, released separately (K after S, V after PV)
                        mbar_wait_spin_addr(p_full, cp & 1);
                        tc_fence_after();
                        if (j == 0 && it > 0) {   // O is overwritten by this item's first PV
                            mbar_wait_spin_addr(o_free, (it - 1) & 1);
                            tc_fence_after();
                        }
                        mbar_wait_spin_addr(v_full, jg & 1);
                        tc_fence_after();
                        issue_pv(0, jg, j == 0);
                        tc_commit_addr(v_empty);
                        if (more) {
                            mbar_wait_spin_addr(kv_full, (jg + 1) & 1);
                            tc_fence_after();
                            issue_s(0, jg + 1);
                            tc_commit_addr(kv_empty);
                        }
                    } else {
                        if (more) {
                            mbar_wait_spin_addr(kv_full + 8 * ((jg + 1) % kAttnStages), ((jg + 1) / kAttnStages) & 1);
                            tc_fence_after();
                        }
                        for (int tt = 0; tt < NT; ++tt) {
                            mbar_wait_spin_addr(p_full + 8 * tt, cp & 1);   // P_t(j) written, S_t(j) released
                            tc_fence_after();
                            if (j == 0 && it > 0) {   // O_t is overwritten by this item's first PV
                                mbar_wait_spin_addr(o_free + 8 * tt, (it - 1) & 1);
                                tc_fence_after();
                            }
                            issue_pv(tt, jg, j == 0);
                            if (more) issue_s(tt, jg + 1);
                        }
                        tc_commit_addr(kv_empty + 8 * (jg % kAttnStages));
                    }
                }
                for (int tt = 0; tt < NT; ++tt) tc_commit_addr(o_full + 8 * tt);   // O_t final
                tc_commit_addr(q_empty + 8 * qb);   // this item's S MMAs (Q readers) have all retired
            }
        }
    } else {
        // ===================== softmax groups =====================
        // tile tt = bit 2 of the warp, lane quarter q4 = bits 0-1, column half = bit 3: each S row is
        // split over two threads (64 keys each) in two warps of the same lane quarter, four softmax
        // warps per SM sub-partition; the row max / sum halves meet through shared memory behind a
        // 64-thread named barrier per warp pair
        const int tt = (warp >> 2) % NT, q4 = warp & 3, half = warp / (4 * NT);
        const int row = q4 * 32 + lane;
        const uint32_t bar_id = 1 + tt * 4 + q4;
        float *red = reinterpret_cast<float *>(smem + L::off_red) + tt * 768;   // [2 parities][2][128] + [2][128]
        const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
        const uint32_t tS = tmem + lane_off + tt * KT + half * (KT / 2);
        const uint32_t tO = tmem + lane_off + L::tm_o + tt * L::tm_o_step;
        const uint32_t tP = tmem + lane_off + L::tm_p + tt * L::tm_p_step + half * (KT / 4);
        auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
        int cs = 0;   // S_t handshakes so far (ring parity of s_full and of the max exchange)
        for (int item = blockIdx.x, it = 0; item < nitems; item += gridDim.x, ++it) {
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < nkt; ++j, ++cs) {
                mbar_wait_spin_addr(s_full + 8 * tt, cs & 1);
                tc_fence_after();
                if (dbg & 1) {   // DVC_ATTN_DEBUG bit 0: no softmax (MMA/TMA pipeline timing)
                    __syncwarp();
                    if (lane == 0) mbar_arrive(p_full + 8 * tt);
                    continue;
                }
                constexpr int HK = KT / 2;   // keys of this thread's half row
                const int kvalid = N - j * KT - half * HK;   // keys >= kvalid of this half are padding
                uint32_t sr[HK];
#pragma unroll
                for (int c = 0; c < HK / 32; ++c)
                    tmem_ld32_nowait(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
#pragma unroll
                for (int c = 0; c < HK / 32; ++c) tmem_wait32(*reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
                if (kvalid < HK) {
#pragma unroll
                    for (int i = 0; i < HK; ++i)
                        if (i >= kvalid) sr[i] = __float_as_uint(-INFINITY);
                }
                float mxp[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) mxp[i] = fmaxf(__uint_as_float(sr[i]), __uint_as_float(sr[8 + i]));
#pragma unroll
                for (int i = 16; i < HK; i += 16)
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mxp[k] = fmaxf(mxp[k], fmaxf(__uint_as_float(sr[i + k]), __uint_as_float(sr[i + 8 + k])));
                float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                                 fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
                float *rj = red + (cs & 1) * 256;
                rj[half * 128 + row] = mx;
                pair_sync();
                mx = fmaxf(mx, rj[(half ^ 1) * 128 + row]);
                const float mt = mx * scale_log2;
                if (j == 0) {
                    m = mt;
                } else {
                    const bool move = mt > m + 8.f;   // lazy maximum: P stays <= 2^8 (same decision in both halves)
                    if (__any_sync(0xffffffffu, move)) {
                        const float alpha = move ? ex2f(m - mt) : 1.f;
#pragma unroll
                        for (int c = 0; c < D / 16; ++c) {
                            if ((c & 1) != half) continue;   // O column chunks split between the halves
                            uint32_t r[16];
                            tmem_ld16(tO + c * 16, r);
#pragma unroll
                            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                            tmem_st16(tO + c * 16, r);
                        }
                        tmem_wait_st();
                        l *= alpha;
                        if (move) m = mt;
                    }
                }
                // packed fp32x2 arithmetic (FFMA2 / FADD2): two scores per instruction
                float2 rsp[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
#pragma unroll
                for (int c = 0; c < HK / 32; ++c) {   // 32 keys -> 16 packed columns of P_t in TMEM
                    uint32_t pk[16];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int e = c * 32 + q * 8 + 2 * i;
                            const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])),
                                                        sc2, nm2);
                            const float2 p = 2 * i < NPOLY ? ex2_poly2(x) : make_float2(ex2f(x.x), ex2f(x.y));
                            rsp[i] = __fadd2_rn(rsp[i], p);   // padding: x = -inf -> ~0
                            pk[q * 4 + i] = pack2<T>(p.x, p.y);
                        }
                    }
                    tmem_st16(tP + c * 16, pk);
                }
                tmem_wait_st();
                l += ((rsp[0].x + rsp[1].x) + (rsp[2].x + rsp[3].x)) + ((rsp[0].y + rsp[1].y) + (rsp[2].y + rsp[3].y));
                tc_fence_before();     // S reads, P stores, O rescale ordered before the release
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + 8 * tt);
            }
            // row sum = both halves' partial sums (same reference max m), through the item's own slots
            float *rl = red + 512;
            rl[half * 128 + row] = l;
            pair_sync();
            l += rl[(half ^ 1) * 128 + row];
            mbar_wait_spin_addr(o_full + 8 * tt, it & 1);
            tc_fence_after();
            const int qg = item % nqg, h = (item / nqg) % heads, t = item / (nqg * heads);
            const int n = qg * 128 * NT + tt * 128 + row;
            const float inv = 1.f / l;
#pragma unroll
            for (int c = 0; c < D / 16; ++c) {
                if ((c & 1) != half) continue;
                uint32_t r[16];
                tmem_ld16(tO + c * 16, r);
                if (n < N) {
                    T *y = out + ((size_t)t * N + n) * C + h * D + c * 16;
                    float f[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[i]) * inv;
                    store8(y, f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[8 + i]) * inv;
                    store8(y + 8, f);
                }
            }
            tc_fence_before();   // O_t read: the next item's first PV may overwrite it
            pair_sync();         // the partner has read rl[] (the next item's exchange may reuse it)
            __syncwarp();
            if (lane == 0) mbar_arrive(o_free + 8 * tt);
        }
    }
    griddep_launch();
    tc_fence_before();
    __syncthreads();
    if (warp == w_mma) tmem_dealloc<1>(tmem, 512);
}

// ----------------------------------------------------------------- host side
static int grid_for(long work, int threads) {
    long b = (work + threads - 1) / threads;
    return (int)(b < 148L * 16 ? (b > 0 ? b : 1) : 148L * 16);
}

PFN_encodeTiled_t get_encode_fn();

static int attn_debug() {   // DVC_ATTN_DEBUG (experiments only): 1 = skip softmax, 2 = skip MMAs
    static int v = -1;
    if (v < 0) {
        const char *e = dvc_knob("DVC_ATTN_DEBUG");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <typename T, int D, int KT = 128>
static dvc_status attn_tc_launch(const void *qkv, void *ws, void *out, int T_, int N, int C, cudaStream_t stream) {
    using L = AttnSmem<D, KT>;
    const int ntiles = (N + 127) / 128;
    const size_t plane = (size_t)T_ * C * ntiles * 128;   // elements of one packed operand
    T *qp = reinterpret_cast<T *>(ws), *kp = qp + plane, *vp = kp + plane;
    DVC_CUDA(launch_pdl(qkv_pack_kernel<T, D, KT>, dim3(ntiles, C / D, T_), dim3(256), 0, stream, 1,
                        reinterpret_cast<const T *>(qkv), qp, kp, vp, N, C));
    ++g_launches;
    ProfSlot slot = prof_begin(stream);
    static int npoly = -1;   // scores per 8 on the FMA pipe (DVC_ATTN_POLY: 0, 2 (default), 4)
    if (npoly < 0) {
        const char *e = dvc_knob("DVC_ATTN_POLY");
        npoly = e ? atoi(e) : DVC_ATTN_POLY;
    }
    auto kfn = npoly == 0 ? attn_tc_kernel<T, D, 0, KT> : npoly == 4 ? attn_tc_kernel<T, D, 4, KT>
             : attn_tc_kernel<T, D, 2, KT>;
    const void *kern = reinterpret_cast<const void *>(kfn);
    {
        dvc_status ss_ = ensure_smem((const void *)kern, (int)(L::bytes));
        if (ss_ != DVC_OK) return ss_;
    }
    const int bf = std::is_same<T, __nv_bfloat16>::value ? 1 : 0;
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const long items = (long)((N + 128 * L::NT - 1) / (128 * L::NT)) * (C / D) * T_;   // persistent: one CTA per SM
    DVC_CUDA(launch_pdl(kfn, dim3((unsigned)(items < nsm ? items : nsm)), dim3(L::THREADS), (size_t)L::bytes, stream, 1,
                        (const T *)qp, (const T *)kp, (const T *)vp, reinterpret_cast<T *>(out), N, C, T_, scale_log2,
                        make_idesc(bf, 128, KT), make_idesc(bf, 128, D), attn_debug()));
    ++g_launches;
    char lab[96];
    snprintf(lab, sizeof(lab), "attn_tc T=%d N=%d C=%d d=%d", T_, N, C, D);
    prof_end_aux(slot, stream, lab, 4.0 * T_ * (double)N * N * C);   // QK^T + PV: 2*N*N*C each
    return DVC_OK;
}

size_t attn_ws_bytes(int T, int N, int C, dvc_dtype dt) {   // packed Q, K, V^T tiles
    return align256(3 * (size_t)T * C * (size_t)((N + 127) / 128 * 128) * dt_size(dt));
}

template <typename T>
static dvc_status attention_t(const void *qkv, int T_, int N, int C, int D, void *ws, void *out, cudaStream_t s) {
    switch (D) {
        case 16: return attn_tc_launch<T, 16>(qkv, ws, out, T_, N, C, s);
        case 32: return attn_tc_launch<T, 32>(qkv, ws, out, T_, N, C, s);
        case 48: return attn_tc_launch<T, 48>(qkv, ws, out, T_, N, C, s);
        case 64: return attn_tc_launch<T, 64>(qkv, ws, out, T_, N, C, s);
        default: return attn_tc_launch<T, 256>(qkv, ws, out, T_, N, C, s);
    }
}

dvc_status attention_run(const void *qkv, int T_, int N, int C, int D, dvc_dtype dt, void *vt, void *out,
                         cudaStream_t s) {
    DVC_CHECK_ARG(T_ >= 1 && T_ < 65536 && N >= 1 && C >= 1, DVC_ERR_ARG, "attention: empty shape");
    DVC_CHECK_ARG(D == 16 || D == 32 || D == 48 || D == 64 || D == 256, DVC_ERR_UNSUPPORTED,
                  "attention: head_dim %d not in {16,32,48,64,256}", D);
    DVC_CHECK_ARG(C % D == 0, DVC_ERR_DIVISIBILITY, "attention: head_dim %d must divide C=%d", D, C);
    if (dt == DVC_F32) {
        const float scale = 1.f / sqrtf((float)D);
        const dim3 g((N + 127) / 128, C / D, T_);
        const float *q = reinterpret_cast<const float *>(qkv);
        float *o = reinterpret_cast<float *>(out);
        switch (D) {
            case 16: attn_simt_kernel<16><<<g, 128, 0, s>>>(q, o, N, C, scale); break;
            case 32: attn_simt_kernel<32><<<g, 128, 0, s>>>(q, o, N, C, scale); break;
            case 48: attn_simt_kernel<48><<<g, 128, 0, s>>>(q, o, N, C, scale); break;
            case 64: attn_simt_kernel<64><<<g, 128, 0, s>>>(q, o, N, C, scale); break;
            default: attn_simt_kernel<256><<<g, 128, 0, s>>>(q, o, N, C, scale); break;
        }
        ++g_launches;
        return check_launch("attn_simt_kernel");
    }
    dvc_status st = dt == DVC_BF16 ? attention_t<__nv_bfloat16>(qkv, T_, N, C, D, vt, out, s)
                                   : attention_t<__half>(qkv, T_, N, C, D, vt, out, s);
    if (st != DVC_OK) return st;
    return check_launch("attn_tc_kernel");
}

// ----------------------------------------------------------------- the block
size_t transformer_ws_bytes(int C, int T, int H, int W, dvc_dtype dt) {
    const size_t px = (size_t)T * H * W, es = dt_size(dt);
    // A, B, E: [px][C]; big: [px][8C] (qkv, then ff1); F: [px][4C]; Vt; coef; box statistics of X
    return 3 * align256(px * C * es) + align256(px * 8 * C * es) + align256(px * 4 * C * es) +
           attn_ws_bytes(T, H * W, C, dt) + align256((size_t)T * C * 8) + box_stats_bytes(T, H, W, C) +
           align256((size_t)8 * C * C * es) + align256((size_t)8 * C * es);
}

dvc_status transformer_validate(const TF &b, int T, int H, int W) {
    DVC_CHECK_ARG(dt_valid(b.dt), DVC_ERR_ARG, "transformer: bad dtype");
    DVC_CHECK_ARG(T >= 1 && T < 256 && H >= 1 && W >= 1, DVC_ERR_ARG, "transformer: empty shape");
    DVC_CHECK_ARG(b.c % 16 == 0 && b.c <= 1024, DVC_ERR_UNSUPPORTED, "transformer: C must be a multiple of 16, <= 1024");
    DVC_CHECK_ARG(b.groups >= 1 && b.c % b.groups == 0, DVC_ERR_DIVISIBILITY, "transformer: G must divide C");
    DVC_CHECK_ARG(b.head_dim == 16 || b.head_dim == 32 || b.head_dim == 48 || b.head_dim == 64, DVC_ERR_UNSUPPORTED,
                  "transformer: head_dim in {16,32,48,64}");
    DVC_CHECK_ARG(b.c % b.head_dim == 0, DVC_ERR_DIVISIBILITY, "transformer: head_dim must divide C");
    DVC_CHECK_ARG(b.gn_w && b.gn_b && b.proj_in_w && b.proj_in_b && b.ln1_w && b.ln1_b && b.qkv_w && b.out_w &&
                      b.out_b && b.ln2_w && b.ln2_b && b.ff1_w && b.ff1_b && b.ff2_w && b.ff2_b && b.proj_out_w &&
                      b.proj_out_b,
                  DVC_ERR_ARG, "transformer: null weight");
    return DVC_OK;
}

template <typename T>
static dvc_status elementwise_launches(int which, const void *a, const void *b, const void *c, void *y, long n,
                                       int C, float eps, int hw, cudaStream_t s) {
    switch (which) {
        case 0:   // GN affine: a = x, b = coef
            DVC_CUDA(launch_pdl(gn_affine_kernel<T>, dim3(grid_for(n * C / 8, 256)), dim3(256), 0, s, 1,
                                reinterpret_cast<const T *>(a), reinterpret_cast<const float2 *>(b),
                                reinterpret_cast<T *>(y), hw, C, n * C / 8));
            break;
        case 1:   // LN: a = x, b = gamma, c = beta, n = pixels
            DVC_CUDA(launch_pdl(layernorm_kernel<T>, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, s, 1,
                                reinterpret_cast<const T *>(a), reinterpret_cast<const T *>(b),
                                reinterpret_cast<const T *>(c), reinterpret_cast<T *>(y), n, C, eps));
            break;
        default:  // GEGLU: a = f [n][2C], C = 4C'
            DVC_CUDA(launch_pdl(geglu_kernel<T>, dim3(grid_for(n * C / 8, 256)), dim3(256), 0, s, 1,
                                reinterpret_cast<const T *>(a), reinterpret_cast<T *>(y), C, n * C / 8));
            break;
    }
    ++g_launches;
    return DVC_OK;
}

static dvc_status ew(int which, dvc_dtype dt, const void *a, const void *b, const void *c, void *y, long n, int C,
                     float eps, cudaStream_t s, int hw = 1) {
    ProfSlot slot = prof_begin(s);
    dvc_status st;
    switch (dt) {
        case DVC_BF16: st = elementwise_launches<__nv_bfloat16>(which, a, b, c, y, n, C, eps, hw, s); break;
        case DVC_F16: st = elementwise_launches<__half>(which, a, b, c, y, n, C, eps, hw, s); break;
        default: st = elementwise_launches<float>(which, a, b, c, y, n, C, eps, hw, s); break;
    }
    prof_end_aux(slot, s, which == 0 ? "tf_gn" : which == 1 ? "tf_ln" : "tf_geglu");
    return st;
}

dvc_status gn_affine_run(const void *x, const void *coef, int T, int HW, int C, dvc_dtype dt, void *y,
                         cudaStream_t s) {
    return ew(0, dt, x, coef, nullptr, y, (long)T * HW, C, 0.f, s, HW);
}

dvc_status interleave_ff1(const TF &b, void *wi, void *bi, cudaStream_t s) {
    const int C4 = 4 * b.c;
    auto one = [&](auto *tag, const void *src, void *dst, int cols) -> dvc_status {
        using E = std::remove_pointer_t<decltype(tag)>;
        const int blocks = (int)std::min<long>((2L * C4 * cols + 255) / 256, 148L * 8);
        DVC_CUDA(launch_pdl(geglu_interleave_kernel<E>, dim3(blocks), dim3(256), 0, s, 1,
                            reinterpret_cast<const E *>(src), reinterpret_cast<E *>(dst), C4, cols));
        ++g_launches;
        return DVC_OK;
    };
    dvc_status st;
    if (b.dt == DVC_BF16) {
        if ((st = one((__nv_bfloat16 *)nullptr, b.ff1_w, wi, b.c)) != DVC_OK) return st;
        return one((__nv_bfloat16 *)nullptr, b.ff1_b, bi, 1);
    }
    if ((st = one((__half *)nullptr, b.ff1_w, wi, b.c)) != DVC_OK) return st;
    return one((__half *)nullptr, b.ff1_b, bi, 1);
}

dvc_status transformer_launch(const TF &b, const void *x, int T, int H, int W, void *y, void *ws, cudaStream_t s,
                              const void *stats_x, void *stats_y) {
    const int C = b.c;
    const size_t px = (size_t)T * H * W, es = dt_size(b.dt);
    uint8_t *p = reinterpret_cast<uint8_t *>(ws);
    auto take = [&](size_t bytes) {
        void *r = p;
        p += align256(bytes);
        return r;
    };
    void *A = take(px * C * es), *B = take(px * C * es), *E = take(px * C * es);
    void *big = take(px * 8 * C * es), *Fb = take(px * 4 * C * es);
    void *vt = take(attn_ws_bytes(T, H * W, C, b.dt));
    float2 *coef = reinterpret_cast<float2 *>(take((size_t)T * C * 8));
    void *bst = take(box_stats_bytes(T, H, W, C));
    void *ff1_wi = take((size_t)8 * C * C * es), *ff1_bi = take((size_t)8 * C * es);
    dvc_status st;
    // a = GN(X): coefficients from box statistics of X (the producer's, or computed here)
    if (!stats_x) {
        if ((st = box_stats_run(x, T, H, W, C, b.dt, reinterpret_cast<float *>(bst), s)) != DVC_OK) return st;
        stats_x = bst;
    }
    NormArgs na{x, nullptr, nullptr, C, 0, 0, T, H * W, b.groups, b.eps_gn, b.gn_w, b.gn_b, coef, nullptr};
    if ((st = gn_coef_box_run(na, BoxStatsIn{stats_x, nullptr, nullptr}, H, W, b.dt, s)) != DVC_OK) return st;
    if ((st = ew(0, b.dt, x, coef, nullptr, A, (long)px, C, 0.f, s, H * W)) != DVC_OK) return st;
    auto lin = [&](const void *src, int cin, const void *w, const void *bias, int cout, const void *res, void *dst,
                   void *stats) {
        ConvDesc d{};
        d.seg[0] = ConvSeg{src, cin, SEG_SAME, H, W, 1, w, cin, 0, cin};
        d.nseg = 1;
        d.T = T;
        d.ho = H;
        d.wo = W;
        d.cout = cout;
        d.bias0 = bias;
        d.residual = res;
        d.out = dst;
        d.stats_out = stats;
        d.dt = b.dt;
        return conv_run(d, s);
    };
    if ((st = lin(A, C, b.proj_in_w, b.proj_in_b, C, nullptr, B, nullptr)) != DVC_OK) return st;          // h0 = B
    if ((st = ew(1, b.dt, B, b.ln1_w, b.ln1_b, A, (long)px, C, b.eps_ln, s)) != DVC_OK) return st;        // l1 = A
    if ((st = lin(A, C, b.qkv_w, nullptr, 3 * C, nullptr, big, nullptr)) != DVC_OK) return st;            // qkv
    if ((st = attention_run(big, T, H * W, C, b.head_dim, b.dt, vt, A, s)) != DVC_OK) return st;          // o = A
    if ((st = lin(A, C, b.out_w, b.out_b, C, B, E, nullptr)) != DVC_OK) return st;                        // h1 = E
    if ((st = ew(1, b.dt, E, b.ln2_w, b.ln2_b, A, (long)px, C, b.eps_ln, s)) != DVC_OK) return st;        // l2 = A
    if (b.dt != DVC_F32 && g_ws_cg != 0) {
        // g = f[:4C] * gelu(f[4C:]) in FF1's epilogue (rows interleaved in 16 + 16 blocks): the 8C-wide
        // FF1 output never reaches HBM
        const void *wi = b.ff1_wi, *bi = b.ff1_bi;
        if (!wi || !bi) {
            if ((st = interleave_ff1(b, ff1_wi, ff1_bi, s)) != DVC_OK) return st;
            wi = ff1_wi, bi = ff1_bi;
        }
        ConvDesc d{};
        d.seg[0] = ConvSeg{A, C, SEG_SAME, H, W, 1, wi, C, 0, C};
        d.nseg = 1, d.T = T, d.ho = H, d.wo = W, d.cout = 8 * C, d.bias0 = bi, d.out = Fb, d.dt = b.dt;
        d.geglu = 1;
        if ((st = conv_run(d, s)) != DVC_OK) return st;                                                    // g
    } else {
        if ((st = lin(A, C, b.ff1_w, b.ff1_b, 8 * C, nullptr, big, nullptr)) != DVC_OK) return st;        // f
        if ((st = ew(2, b.dt, big, nullptr, nullptr, Fb, (long)px, 4 * C, 0.f, s)) != DVC_OK) return st;  // g
    }
    if ((st = lin(Fb, 4 * C, b.ff2_w, b.ff2_b, C, E, B, nullptr)) != DVC_OK) return st;                   // h2 = B
    return lin(B, C, b.proj_out_w, b.proj_out_b, C, x, y, stats_y);                                       // Y
}

}  // namespace dvc

// ----------------------------------------------------------------- C-ABI (include/dvc.h, f1)
using namespace dvc;

static TF tf_from_abi(const dvc_transformer *b) {
    return TF{b->c,     b->groups,  b->head_dim,  b->eps_gn, b->eps_ln, b->dt,    b->gn_w,       b->gn_b,
              b->proj_in_w, b->proj_in_b, b->ln1_w, b->ln1_b, b->qkv_w, b->out_w, b->out_b, b->ln2_w,
              b->ln2_b, b->ff1_w, b->ff1_b, b->ff2_w, b->ff2_b, b->proj_out_w, b->proj_out_b};
}

extern "C" {

dvc_status dvc_transformer_workspace_size(const dvc_transformer *b, int T, int H, int W, size_t *bytes) {
    DVC_CHECK_ARG(b && bytes, DVC_ERR_ARG, "null argument");
    const TF t = tf_from_abi(b);
    dvc_status st = transformer_validate(t, T, H, W);
    if (st != DVC_OK) return st;
    *bytes = transformer_ws_bytes(t.c, T, H, W, t.dt);
    return DVC_OK;
}

dvc_status dvc_transformer_forward(const dvc_transformer *b, const void *x, int T, int H, int W, void *y,
                                   void *workspace, size_t ws_bytes, void *stream) {
    NvtxRange nv("dvc_transformer_forward T=%d %dx%d", T, H, W);
    DVC_CHECK_ARG(b && x && y && workspace, DVC_ERR_ARG, "null argument");
    const TF t = tf_from_abi(b);
    dvc_status st = transformer_validate(t, T, H, W);
    if (st != DVC_OK) return st;
    DVC_CHECK_ARG(ws_bytes >= transformer_ws_bytes(t.c, T, H, W, t.dt), DVC_ERR_WORKSPACE, "workspace too small");
    DVC_CHECK_ARG(((uintptr_t)workspace & 255) == 0, DVC_ERR_ARG, "workspace must be 256-byte aligned");
    if ((st = check_device()) != DVC_OK) return st;
    return transformer_launch(t, x, T, H, W, y, workspace, reinterpret_cast<cudaStream_t>(stream));
}

dvc_status dvc_attention_workspace_size(int T, int N, int C, dvc_dtype dt, size_t *bytes) {
    DVC_CHECK_ARG(bytes && T >= 1 && N >= 1 && C >= 1 && dt_valid(dt), DVC_ERR_ARG, "bad arguments");
    *bytes = dt == DVC_F32 ? 0 : attn_ws_bytes(T, N, C, dt);
    return DVC_OK;
}

dvc_status dvc_attention_forward(const void *qkv, int T, int N, int C, int head_dim, dvc_dtype dt, void *out,
                                 void *workspace, size_t ws_bytes, void *stream) {
    DVC_CHECK_ARG(qkv && out && dt_valid(dt), DVC_ERR_ARG, "null argument / bad dtype");
    DVC_CHECK_ARG(C % 8 == 0, DVC_ERR_UNSUPPORTED, "attention: C must be a multiple of 8");
    if (dt != DVC_F32) {
        DVC_CHECK_ARG(workspace && ws_bytes >= attn_ws_bytes(T, N, C, dt), DVC_ERR_WORKSPACE, "workspace too small");
        DVC_CHECK_ARG(((uintptr_t)workspace & 255) == 0 && ((uintptr_t)qkv & 15) == 0 && ((uintptr_t)out & 15) == 0,
                      DVC_ERR_ARG, "workspace 256-byte, qkv/out 16-byte aligned");
    }
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    return attention_run(qkv, T, N, C, head_dim, dt, workspace, out, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
