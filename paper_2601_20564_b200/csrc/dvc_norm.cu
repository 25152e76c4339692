// dvc_norm.cu -- GroupNorm statistics and the fused GN-apply + SiLU operand
// producer (reading R2-R4), with the Batch-dimension temporal
// shift folded into the element addressing (a3).
//
// HBM-bound.  Every thread owns one 8-channel vector of the pixel row and
// walks pixels with a fixed stride, so (a) the shift / concat / carry source
// of its vector is resolved once, outside the pixel loop, (b) a warp reads
// 32 consecutive 16-byte vectors (coalesced), (c) the per-channel GN
// coefficients live in registers.
//
// Statistics are deterministic and independent of batching (H4): frame t's
// (mean, rstd) per group come only from frame t's shifted input, reduced in a
// fixed order (per-thread fp64 sums over a fixed pixel stride, fixed-order
// smem merge per 256-pixel chunk, fixed-order merge over chunks).
#include <cstdio>
#include "dvc_norm.cuh"
#include "dvc_boxstats.cuh"
#include "dvc_conv.cuh"

namespace dvc {

constexpr int kPixPerThread = 32;   // pixels per thread per statistics / apply block

// pixels per block: every thread owns one 8-channel vector and kPixPerThread pixels
__host__ __device__ __forceinline__ int chunk_pix(int C) { return (256 / (C >> 3)) * kPixPerThread; }

// Source of one thread's 8-channel vector of the (shifted, concatenated) operand
// for frame t.  mode: 0 = zeros, 1 = vector load, 2 = per-element carry,
// 3 = straddle with zeros / carry (frame 0), 4 = straddle with frame t-1 (vector loads).
template <typename T>
struct VecSrc {
    const T *cur;      // unshifted row base for this vector (frame t), stride `ld`
    const T *prev;     // shifted-slice source: frame t-1 row base (stride ld) or carry (stride cs)
    int ld, pstride, c, cs, mode;

    __device__ __forceinline__ void load(int p, float (&f)[8]) const {
        if (mode == 1) {
            load8(cur + (size_t)p * ld, f);
        } else if (mode == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = 0.f;
        } else if (mode == 2) {   // all 8 channels from the carry [HW][cs] (element loads)
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = Elem<T>::to_f(prev[(size_t)p * pstride + i]);
        } else {                  // modes 3/4: straddles the slice boundary, element-wise select
            float g[8];
            load8(cur + (size_t)p * ld, f);
            if (prev == nullptr) {
#pragma unroll
                for (int i = 0; i < 8; ++i) g[i] = 0.f;
            } else if (pstride == ld) {
                load8(prev + (size_t)p * ld, g);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    g[i] = (c + i < cs) ? Elem<T>::to_f(prev[(size_t)p * pstride + i]) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (c + i < cs) f[i] = g[i];
        }
    }
};

// raw 16-byte vector (8 x 16-bit, or the first half of 8 x fp32 when T is float)
template <typename T>
__device__ __forceinline__ void cvt8(const uint4 (&u)[sizeof(T) / 2], float (&f)[8]) {
    const T *e = reinterpret_cast<const T *>(u);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = Elem<T>::to_f(e[i]);
}
template <typename T>
__device__ __forceinline__ void ldraw8(const T *p, uint4 (&u)[sizeof(T) / 2]) {
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 2); ++k) u[k] = __ldg(reinterpret_cast<const uint4 *>(p) + k);
}

// Fast path for modes 1 and 4: issue the raw loads of NP pixels first, convert after.
template <typename T, int NP, bool STRADDLE>
__device__ __forceinline__ void load_fast(const VecSrc<T> &src, int p, int step, float (&f)[NP][8]) {
    constexpr int NU = sizeof(T) / 2;
    uint4 u[NP][NU];
#pragma unroll
    for (int j = 0; j < NP; ++j) ldraw8(src.cur + (size_t)(p + j * step) * src.ld, u[j]);
    if constexpr (STRADDLE) {
        uint4 w[NP][NU];
#pragma unroll
        for (int j = 0; j < NP; ++j) ldraw8(src.prev + (size_t)(p + j * step) * src.ld, w[j]);
#pragma unroll
        for (int j = 0; j < NP; ++j) cvt8<T>(u[j], f[j]);
        const int k = src.cs - src.c;   // first k channels come from frame t-1
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            float g[8];
            cvt8<T>(w[j], g);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < k) f[j][i] = g[i];
        }
    } else {
#pragma unroll
        for (int j = 0; j < NP; ++j) cvt8<T>(u[j], f[j]);
    }
}

// Resolve the source of vector `v` (channels 8v..8v+7) of frame t.
template <typename T>
__device__ __forceinline__ VecSrc<T> vec_src(const ShiftSrc<T> &X, int t, int v) {
    VecSrc<T> s;
    const int c = 8 * v;
    const bool in_a = c < X.ca;
    const T *base = in_a ? X.xa : X.xb;
    const int ld = in_a ? X.ca : X.cb;
    const int cc = in_a ? c : c - X.ca;
    s.ld = ld;
    s.c = c;
    s.cs = X.cs;
    s.cur = base + (size_t)t * X.HW * ld + cc;
    s.prev = nullptr;
    s.pstride = ld;
    if (c >= X.cs) {
        s.mode = 1;
        return s;
    }
    // (part of) the shifted slice: frame t-1, or the carry at t == 0 (zeros if none)
    if (t > 0) {
        s.prev = base + (size_t)(t - 1) * X.HW * ld + cc;
        if (c + 8 <= X.cs) {
            s.cur = s.prev;
            s.mode = 1;
        } else {
            s.mode = 4;
        }
    } else if (X.carry == nullptr) {
        s.mode = c + 8 <= X.cs ? 0 : 3;
    } else {
        s.prev = X.carry + c;
        s.pstride = X.cs;
        s.mode = c + 8 <= X.cs ? 2 : 3;
    }
    return s;
}

// Partial sums per (frame, chunk, group): grid (nchunk, T), 256 threads.
template <typename T>
__global__ void __launch_bounds__(256, 3) gn_partial_kernel(const ShiftSrc<T> X, int G, double2 *__restrict__ partial,
                                                         int nchunk) {
    griddep_wait();
    __shared__ double s_sum[2048];
    __shared__ double s_sq[2048];
    const int t = blockIdx.y, chunk = blockIdx.x;
    const int C = X.C(), nv = C >> 3, npl = 256 / nv;
    const int tid = threadIdx.x, v = tid % nv, pl = tid / nv;
    const int cp = chunk_pix(C);
    const int p0 = chunk * cp, p1 = min(X.HW, p0 + cp);
    if (pl < npl) {
        const VecSrc<T> src = vec_src(X, t, v);
        // fp32 partial over <= kPixPerThread values per channel; fp64 from the block merge on
        float s[8], q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = q[i] = 0.f;
        // identical arithmetic for every source mode and every T (bit-exact batch == online, H4):
        // pixels are accumulated one at a time in increasing p.
        constexpr int NU = sizeof(T) / 2;
        int p = p0 + pl;
        if (src.mode == 1) {   // hot path: raw loads of 4 pixels in flight before any use
            for (; p + 3 * npl < p1; p += 4 * npl) {
                uint4 u[4][NU];
#pragma unroll
                for (int j = 0; j < 4; ++j) ldraw8(src.cur + (size_t)(p + j * npl) * src.ld, u[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float f[8];
                    cvt8<T>(u[j], f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        s[i] += f[i];
                        q[i] = fmaf(f[i], f[i], q[i]);
                    }
                }
            }
        }
        for (; p < p1; p += npl) {
            float f[8];
            src.load(p, f);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                s[i] += f[i];
                q[i] = fmaf(f[i], f[i], q[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s_sum[pl * C + v * 8 + i] = (double)s[i];
            s_sq[pl * C + v * 8 + i] = (double)q[i];
        }
    }
    __syncthreads();
    const int cg = C / G;
    for (int g = tid; g < G; g += blockDim.x) {
        double S = 0.0, Q = 0.0;
        for (int l = 0; l < npl; ++l)
            for (int c = g * cg; c < (g + 1) * cg; ++c) {
                S += s_sum[l * C + c];
                Q += s_sq[l * C + c];
            }
        partial[((size_t)t * nchunk + chunk) * G + g] = make_double2(S, Q);
    }
}

// coef[t][c] = (mean of c's group, rstd * gamma[c]): grid (T), 256 threads.
// One warp per group: lanes take chunks l, l+32, ... and a fixed xor-shuffle
// tree merges them (deterministic for a given nchunk).
template <typename T>
__global__ void __launch_bounds__(256) gn_finalize_kernel(const double2 *__restrict__ partial, int nchunk, int G,
                                                          int C, double n, double eps, const T *__restrict__ gamma,
                                                          float2 *__restrict__ coef) {
    griddep_wait();
    __shared__ float s_mu[256], s_rs[256];
    const int t = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = warp; g < G; g += blockDim.x >> 5) {
        double S = 0.0, Q = 0.0;
        for (int c = lane; c < nchunk; c += 32) {
            const double2 v = partial[((size_t)t * nchunk + c) * G + g];
            S += v.x;
            Q += v.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            S += __shfl_xor_sync(0xffffffffu, S, o);
            Q += __shfl_xor_sync(0xffffffffu, Q, o);
        }
        if (lane == 0) {
            const double mu = S / n;
            double var = Q / n - mu * mu;   // biased variance (R4)
            if (var < 0.0) var = 0.0;
            s_mu[g] = (float)mu;
            s_rs[g] = (float)(1.0 / sqrt(var + eps));
        }
    }
    __syncthreads();
    const int cg = C / G;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        const int g = c / cg;
        coef[(size_t)t * C + c] = make_float2(s_mu[g], s_rs[g] * Elem<T>::to_f(gamma[c]));
    }
}

// SiLU(z) = z / (1 + e^-z).  16-bit outputs: one MUFU (ex2) per element and a
// Newton reciprocal on the FMA pipe (rel. error < 1e-6, far below the 16-bit
// rounding of the result); the MUFU pipe would otherwise bound this HBM kernel.
template <typename T>
__device__ __forceinline__ float silu_t(float z) {
    if constexpr (sizeof(T) == 4) {
        return z / (1.0f + expf(-z));   // validation mode: accurate
    } else {   // z holds hz = z / 2 (the affine is pre-scaled): SiLU = hz + hz tanh(hz), ONE MUFU op (R23)
        return fmaf(z, tanh_fast(z), z);
    }
}

// out[t][p][c] = SiLU((Xs[t][p][c] - mu) * (rstd*gamma[c]) + beta[c]): grid (nchunk, T).
template <typename T>
__global__ void __launch_bounds__(256) gn_silu_kernel(const ShiftSrc<T> X, const float2 *__restrict__ coef,
                                                      const T *__restrict__ beta, T *__restrict__ out, int cp) {
    griddep_wait();
    const int t = blockIdx.y, chunk = blockIdx.x;
    const int C = X.C(), nv = C >> 3, npl = 256 / nv;
    const int tid = threadIdx.x, v = tid % nv, pl = tid / nv;
    if (pl >= npl) return;
    const int p0 = chunk * cp, p1 = min(X.HW, p0 + cp);
    const VecSrc<T> src = vec_src(X, t, v);
    float mu[8], sc[8], be[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float2 cf = coef[(size_t)t * C + 8 * v + i];
        sc[i] = cf.y;
        mu[i] = cf.x;
        be[i] = Elem<T>::to_f(beta[8 * v + i]);
        if (sizeof(T) == 2) {   // 16-bit outputs: hz = f*sc/2 + (beta - mu*sc)/2, one FMA per element
            be[i] = 0.5f * (be[i] - mu[i] * sc[i]);
            sc[i] *= 0.5f;
            mu[i] = 0.f;
        }
    }
    T *o = out + (size_t)t * X.HW * C + 8 * v;
    int p = p0 + pl;
    if (src.mode == 1) {   // hot path: 8 pixels' raw loads in flight, then compute + store
        for (; p + 7 * npl < p1; p += 8 * npl) {
            float f[8][8];
            load_fast<T, 8, false>(src, p, npl, f);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
#pragma unroll
                for (int i = 0; i < 8; ++i) f[j][i] = silu_t<T>(sizeof(T) == 2 ? fmaf(f[j][i], sc[i], be[i]) : (f[j][i] - mu[i]) * sc[i] + be[i]);
                store8(o + (size_t)(p + j * npl) * C, f[j]);
            }
        }
    } else if (src.mode == 4) {   // vector straddling the shifted slice: two sources, 2 pixels in flight
        for (; p + npl < p1; p += 2 * npl) {
            float f[2][8];
            load_fast<T, 2, true>(src, p, npl, f);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
#pragma unroll
                for (int i = 0; i < 8; ++i) f[j][i] = silu_t<T>(sizeof(T) == 2 ? fmaf(f[j][i], sc[i], be[i]) : (f[j][i] - mu[i]) * sc[i] + be[i]);
                store8(o + (size_t)(p + j * npl) * C, f[j]);
            }
        }
    }
    for (; p < p1; p += npl) {
        float f[8];
        src.load(p, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = silu_t<T>(sizeof(T) == 2 ? fmaf(f[i], sc[i], be[i]) : (f[i] - mu[i]) * sc[i] + be[i]);
        store8(o + (size_t)p * C, f);
    }
}

// Test-only: materialise Xs with the same addressing (dvc_debug_shift_gather).
template <typename T>
__global__ void __launch_bounds__(256) shift_gather_kernel(const ShiftSrc<T> X, T *__restrict__ out) {
    griddep_wait();
    const int t = blockIdx.y, chunk = blockIdx.x;
    const int C = X.C(), nv = C >> 3, npl = 256 / nv;
    const int tid = threadIdx.x, v = tid % nv, pl = tid / nv;
    if (pl >= npl) return;
    const int cp = chunk_pix(C);
    const int p0 = chunk * cp, p1 = min(X.HW, p0 + cp);
    const VecSrc<T> src = vec_src(X, t, v);
    for (int p = p0 + pl; p < p1; p += npl) {
        float f[8];
        src.load(p, f);
        store8(out + ((size_t)t * X.HW + p) * C + 8 * v, f);   // exact: 16-bit -> fp32 -> 16-bit is the identity
    }
}

size_t gn_workspace_bytes(int T, int HW, int G, int C) {
    const int nchunk = (HW + chunk_pix(C) - 1) / chunk_pix(C);
    return align256((size_t)T * nchunk * G * sizeof(double2)) + align256((size_t)T * C * sizeof(float2));
}

template <typename T>
static dvc_status gn_silu_t(const NormArgs &a, cudaStream_t stream) {
    ShiftSrc<T> X{reinterpret_cast<const T *>(a.xa), reinterpret_cast<const T *>(a.xb),
                  reinterpret_cast<const T *>(a.carry), a.ca, a.cb, a.cs, a.HW};
    const int C = a.ca + a.cb;
    const int nchunk = (a.HW + chunk_pix(C) - 1) / chunk_pix(C);
    double2 *partial = reinterpret_cast<double2 *>(a.ws);
    float2 *coef = reinterpret_cast<float2 *>(reinterpret_cast<uint8_t *>(a.ws) +
                                              align256((size_t)a.T * nchunk * a.G * sizeof(double2)));
    DVC_CUDA(launch_pdl(gn_partial_kernel<T>, dim3(dim3(nchunk, a.T)), dim3(256), 0, stream, 1, X, a.G, partial, nchunk));
    ++g_launches;
    DVC_CUDA(launch_pdl(gn_finalize_kernel<T>, dim3(a.T), dim3(256), 0, stream, 1, partial, nchunk, a.G, C, (double)(C / a.G) * a.HW, (double)a.eps,
                                                   reinterpret_cast<const T *>(a.gamma), coef));
    ++g_launches;
    DVC_CUDA(launch_pdl(gn_silu_kernel<T>, dim3(dim3(nchunk, a.T)), dim3(256), 0, stream, 1, X, coef, reinterpret_cast<const T *>(a.beta),
                                                             reinterpret_cast<T *>(a.out), chunk_pix(C)));
    ++g_launches;
    return check_launch("gn_silu");
}

dvc_status gn_silu_run(const NormArgs &a, dvc_dtype dt, cudaStream_t stream) {
    const int C = a.ca + a.cb;
    DVC_CHECK_ARG(a.ca % 8 == 0 && a.cb % 8 == 0 && C / 8 <= 256, DVC_ERR_UNSUPPORTED,
                  "GN: channel counts must be multiples of 8 and at most 2048");
    DVC_CHECK_ARG(a.G >= 1 && a.G <= 256 && C % a.G == 0, DVC_ERR_DIVISIBILITY, "GN: G=%d must divide C=%d", a.G, C);
    DVC_CHECK_ARG(a.cs <= a.ca, DVC_ERR_UNSUPPORTED, "shift slice must lie in the first source");
    switch (dt) {
        case DVC_BF16: return gn_silu_t<__nv_bfloat16>(a, stream);
        case DVC_F16: return gn_silu_t<__half>(a, stream);
        default: return gn_silu_t<float>(a, stream);
    }
}

template <typename T>
static dvc_status gather_t(const NormArgs &a, cudaStream_t stream) {
    ShiftSrc<T> X{reinterpret_cast<const T *>(a.xa), reinterpret_cast<const T *>(a.xb),
                  reinterpret_cast<const T *>(a.carry), a.ca, a.cb, a.cs, a.HW};
    const int nchunk = (a.HW + chunk_pix(a.ca + a.cb) - 1) / chunk_pix(a.ca + a.cb);
    DVC_CUDA(launch_pdl(shift_gather_kernel<T>, dim3(dim3(nchunk, a.T)), dim3(256), 0, stream, 1, X, reinterpret_cast<T *>(a.out)));
    ++g_launches;
    return check_launch("shift_gather");
}

dvc_status shift_gather_run(const NormArgs &a, dvc_dtype dt, cudaStream_t stream) {
    DVC_CHECK_ARG(a.ca % 8 == 0 && a.cb % 8 == 0 && (a.ca + a.cb) / 8 <= 256, DVC_ERR_UNSUPPORTED,
                  "gather: channels must be multiples of 8, at most 2048");
    DVC_CHECK_ARG(a.cs <= a.ca, DVC_ERR_UNSUPPORTED, "shift slice must lie in the first source");
    switch (dt) {
        case DVC_BF16: return gather_t<__nv_bfloat16>(a, stream);
        case DVC_F16: return gather_t<__half>(a, stream);
        default: return gather_t<float>(a, stream);
    }
}

// ----------------------------------------------------------------- nearest resize (R11)
// U[t][y][x][c] = V[t][floor(y*hi/ho)][floor(x*wi/wo)][c]: materialises the
// up-sampler's operand so its 3x3 conv runs on the TMA engine.  Exact copy.
__global__ void __launch_bounds__(256) nearest_kernel(const uint4 *__restrict__ V, uint4 *__restrict__ U, int hi,
                                                      int wi, int ho, int wo, int nvec) {
    griddep_wait();
    const int y = blockIdx.y, t = blockIdx.z;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;   // x * nvec + v within the output row
    if (i >= wo * nvec) return;
    const int x = i / nvec, v = i - x * nvec;
    const int sy = (int)(((long)y * hi) / ho), sx = (int)(((long)x * wi) / wo);
    U[(((size_t)t * ho + y) * wo) * nvec + i] = __ldg(V + (((size_t)t * hi + sy) * wi + sx) * nvec + v);
}

dvc_status nearest_run(const void *src, void *dst, int T, int hi, int wi, int ho, int wo, int C, dvc_dtype dt,
                       cudaStream_t stream) {
    DVC_CHECK_ARG((C * dt_size(dt)) % 16 == 0, DVC_ERR_UNSUPPORTED, "nearest: rows must be 16-byte multiples");
    const int nvec = (int)(C * dt_size(dt) / 16);
    dim3 grid((wo * nvec + 255) / 256, ho, T);
    ProfSlot s0 = prof_begin(stream);
    DVC_CUDA(launch_pdl(nearest_kernel, dim3(grid), dim3(256), 0, stream, 1, reinterpret_cast<const uint4 *>(src), reinterpret_cast<uint4 *>(dst), hi, wi,
                                             ho, wo, nvec));
    ++g_launches;
    if (s0.idx >= 0) {
        char lab[96];
        snprintf(lab, sizeof(lab), "nearest T=%d %dx%d->%dx%d C=%d", T, hi, wi, ho, wo, C);
        prof_end_aux(s0, stream, lab);
    }
    return check_launch("nearest");
}

// ----------------------------------------------------------------- box statistics (standalone)
// Same partials, same bits as the TMA engine's epilogue (dvc_boxstats.cuh).  grid (nbox, T), 128 threads.
template <typename T>
__global__ void __launch_bounds__(128) box_stats_kernel(const T *__restrict__ x, int H, int W, int C, int BX, int BY,
                                                        int tiles_x, int vec_ok, float *__restrict__ stats) {
    griddep_wait();
    __shared__ float red[2][4][32];
    const int b = blockIdx.x, t = blockIdx.y, per = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = threadIdx.x;
    const int y = (b / tiles_x) * BY + r / BX, xx = (b % tiles_x) * BX + r % BX;
    const bool valid = r < BX * BY && y < H && xx < W;
    const T *row = x + (((size_t)t * H + (valid ? y : 0)) * W + (valid ? xx : 0)) * C;
    for (int c0 = 0, par = 0; c0 < C; c0 += 16, par ^= 1) {
        float v[16];
        if (vec_ok) {   // 16-byte aligned rows: vector loads
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float e[8];
                if (valid && c0 + 8 * h < C) load8(row + c0 + 8 * h, e);
                else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) e[i] = 0.f;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) v[8 * h + i] = e[i];
            }
        } else {              // e.g. a carry slice of C_in/P = 30 channels: element loads
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = (valid && c0 + i < C) ? Elem<T>::to_f(row[c0 + i]) : 0.f;
        }
        float xs[32];
        box_row_values(v, valid, xs);
        red[par][warp][lane] = box_reduce_scatter32(xs, lane);
        __syncthreads();
        if (warp == 0 && c0 + (lane & 15) < C)
            stats[(((size_t)t * per + b) * C + c0 + (lane & 15)) * 2 + (lane >> 4)] = box_combine4(&red[par][0][0], lane);
    }
}

dvc_status box_stats_run(const void *x, int T, int H, int W, int C, dvc_dtype dt, float *stats, cudaStream_t stream) {
    DVC_CHECK_ARG(C >= 1, DVC_ERR_ARG, "box statistics: C must be >= 1");
    int BX = 1, BY = 1;
    choose_box(H, W, &BX, &BY);
    const int tx = (W + BX - 1) / BX, ty = (H + BY - 1) / BY;
    dim3 grid(tx * ty, T);
    // e.g. a packed carry slice may start at any element offset: vector loads only when aligned
    const int vec_ok = (C % 8 == 0) && ((uintptr_t)x % 16 == 0) && ((C * dt_size(dt)) % 16 == 0);
    ProfSlot s0 = prof_begin(stream);
    switch (dt) {
        case DVC_BF16:
            DVC_CUDA(launch_pdl(box_stats_kernel<__nv_bfloat16>, dim3(grid), dim3(128), 0, stream, 1, reinterpret_cast<const __nv_bfloat16 *>(x), H, W,
                                                                      C, BX, BY, tx, vec_ok, stats));
            break;
        case DVC_F16:
            DVC_CUDA(launch_pdl(box_stats_kernel<__half>, dim3(grid), dim3(128), 0, stream, 1, reinterpret_cast<const __half *>(x), H, W, C, BX, BY, tx,
                                                               vec_ok, stats));
            break;
        default:
            DVC_CUDA(launch_pdl(box_stats_kernel<float>, dim3(grid), dim3(128), 0, stream, 1, reinterpret_cast<const float *>(x), H, W, C, BX, BY, tx,
                                                              vec_ok, stats));
    }
    ++g_launches;
    prof_end_aux(s0, stream, "box_stats");
    return check_launch("box_stats");
}

// GN coefficients of the (shifted, concatenated) operand from box statistics:
// group g of frame t takes frame t-1's statistics when its channels lie in the
// shifted slice [0, cs) (carry statistics at t = 0, zeros without a carry),
// else frame t's.  Requires cs % (C/G) == 0.  grid (T), 256 threads, warp per
// group, lanes stride over boxes, fixed xor tree (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) gn_finalize_box_kernel(const float2 *__restrict__ pa, int ca,
                                                              const float2 *__restrict__ pb, int cb,
                                                              const float2 *__restrict__ pk, int cs, int nbox, int G,
                                                              double n, double eps, const T *__restrict__ gamma,
                                                              const T *__restrict__ beta, float2 *__restrict__ coef) {
    griddep_wait();
    __shared__ double s_S[8], s_Q[8];
    __shared__ float s_mu, s_rs;
    const int g = blockIdx.x, t = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = ca + cb, cg = C / G;
    const bool shifted = (g + 1) * cg <= cs;
    const int tf = shifted ? t - 1 : t;
    double S = 0.0, Q = 0.0;
    if (tf >= 0 || pk != nullptr) {
        // the 256 threads stride over the group's (box, channel) items: a fixed order per thread
        const int n_items = nbox * cg;
        for (int i = threadIdx.x; i < n_items; i += blockDim.x) {
            const int b = i / cg, c = g * cg + (i - b * cg);
            float2 v;
            if (tf < 0) v = pk[(size_t)b * cs + c];
            else if (c < ca) v = pa[((size_t)tf * nbox + b) * ca + c];
            else v = pb[((size_t)tf * nbox + b) * cb + (c - ca)];
            S += (double)v.x;
            Q += (double)v.y;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    if (lane == 0) {
        s_S[warp] = S;
        s_Q[warp] = Q;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double SS = 0.0, QQ = 0.0;
        for (int w = 0; w < 8; ++w) {
            SS += s_S[w];
            QQ += s_Q[w];
        }
        const double mu = SS / n;
        double var = QQ / n - mu * mu;   // biased variance (R4)
        if (var < 0.0) var = 0.0;
        s_mu = (float)mu;
        s_rs = (float)(1.0 / sqrt(var + eps));
    }
    __syncthreads();
    for (int c = g * cg + threadIdx.x; c < (g + 1) * cg; c += blockDim.x) {
        const float sc = s_rs * Elem<T>::to_f(gamma[c]);
        // beta == null: (mean, scale) for gn_silu; else the folded affine (scale, beta - mean * scale)
        coef[(size_t)t * C + c] = beta ? make_float2(sc, Elem<T>::to_f(beta[c]) - s_mu * sc) : make_float2(s_mu, sc);
    }
}

size_t box_stats_bytes(int T, int H, int W, int C) { return align256((size_t)T * boxes_per_frame(H, W) * C * 8); }

template <typename T>
static dvc_status gn_silu_box_t(const NormArgs &a, const BoxStatsIn &bs, int H, int W, cudaStream_t stream) {
    ShiftSrc<T> X{reinterpret_cast<const T *>(a.xa), reinterpret_cast<const T *>(a.xb),
                  reinterpret_cast<const T *>(a.carry), a.ca, a.cb, a.cs, a.HW};
    const int C = a.ca + a.cb;
    // one pass of 8 pixels in flight per thread: many short CTAs, no dependent load chains
    const int cp = (256 / (C / 8)) * 8;
    const int nchunk = (a.HW + cp - 1) / cp;
    float2 *coef = reinterpret_cast<float2 *>(a.ws);
    ProfSlot s0 = prof_begin(stream);
    DVC_CUDA(launch_pdl(gn_finalize_box_kernel<T>, dim3(dim3(a.G, a.T)), dim3(256), 0, stream, 1, 
        reinterpret_cast<const float2 *>(bs.a), a.ca, reinterpret_cast<const float2 *>(bs.b), a.cb,
        reinterpret_cast<const float2 *>(bs.carry), a.cs, boxes_per_frame(H, W), a.G, (double)(C / a.G) * a.HW,
        (double)a.eps, reinterpret_cast<const T *>(a.gamma), nullptr, coef));
    ++g_launches;
    if (s0.idx >= 0) {
        char lab[96];
        snprintf(lab, sizeof(lab), "gn_finalize T=%d G=%d C=%d nbox=%d", a.T, a.G, C, boxes_per_frame(H, W));
        prof_end_aux(s0, stream, lab);
    }
    ProfSlot s1 = prof_begin(stream);
    DVC_CUDA(launch_pdl(gn_silu_kernel<T>, dim3(dim3(nchunk, a.T)), dim3(256), 0, stream, 1, X, coef, reinterpret_cast<const T *>(a.beta),
                                                             reinterpret_cast<T *>(a.out), cp));
    ++g_launches;
    if (s1.idx >= 0) {
        char lab[96];
        snprintf(lab, sizeof(lab), "gn_silu T=%d HW=%d C=%d cs=%d", a.T, a.HW, C, a.cs);
        prof_end_aux(s1, stream, lab);
    }
    return check_launch("gn_silu_box");
}

template <typename T>
static dvc_status gn_coef_t(const NormArgs &a, const BoxStatsIn &bs, int H, int W, cudaStream_t stream) {
    const int C = a.ca + a.cb;
    ProfSlot s0 = prof_begin(stream);
    DVC_CUDA(launch_pdl(gn_finalize_box_kernel<T>, dim3(dim3(a.G, a.T)), dim3(256), 0, stream, 1, 
        reinterpret_cast<const float2 *>(bs.a), a.ca, reinterpret_cast<const float2 *>(bs.b), a.cb,
        reinterpret_cast<const float2 *>(bs.carry), a.cs, boxes_per_frame(H, W), a.G, (double)(C / a.G) * a.HW,
        (double)a.eps, reinterpret_cast<const T *>(a.gamma), reinterpret_cast<const T *>(a.beta),
        reinterpret_cast<float2 *>(a.out)));
    ++g_launches;
    if (s0.idx >= 0) {
        char lab[96];
        snprintf(lab, sizeof(lab), "gn_coef T=%d G=%d C=%d nbox=%d", a.T, a.G, C, boxes_per_frame(H, W));
        prof_end_aux(s0, stream, lab);
    }
    return check_launch("gn_coef");
}

dvc_status gn_coef_box_run(const NormArgs &a, const BoxStatsIn &bs, int H, int W, dvc_dtype dt, cudaStream_t stream) {
    const int C = a.ca + a.cb;
    DVC_CHECK_ARG(a.G >= 1 && C % a.G == 0 && a.cs % (C / a.G) == 0, DVC_ERR_UNSUPPORTED, "GN coef: bad groups");
    switch (dt) {
        case DVC_BF16: return gn_coef_t<__nv_bfloat16>(a, bs, H, W, stream);
        case DVC_F16: return gn_coef_t<__half>(a, bs, H, W, stream);
        default: return gn_coef_t<float>(a, bs, H, W, stream);
    }
}

dvc_status gn_silu_box_run(const NormArgs &a, const BoxStatsIn &bs, int H, int W, dvc_dtype dt, cudaStream_t stream) {
    const int C = a.ca + a.cb;
    DVC_CHECK_ARG(a.ca % 8 == 0 && a.cb % 8 == 0 && C / 8 <= 256, DVC_ERR_UNSUPPORTED,
                  "GN: channel counts must be multiples of 8 and at most 2048");
    DVC_CHECK_ARG(a.G >= 1 && a.G <= 256 && C % a.G == 0, DVC_ERR_DIVISIBILITY, "GN: G=%d must divide C=%d", a.G, C);
    DVC_CHECK_ARG(a.cs <= a.ca && a.cs % (C / a.G) == 0, DVC_ERR_UNSUPPORTED, "box GN: slice must be whole groups");
    switch (dt) {
        case DVC_BF16: return gn_silu_box_t<__nv_bfloat16>(a, bs, H, W, stream);
        case DVC_F16: return gn_silu_box_t<__half>(a, bs, H, W, stream);
        default: return gn_silu_box_t<float>(a, bs, H, W, stream);
    }
}

}  // namespace dvc
