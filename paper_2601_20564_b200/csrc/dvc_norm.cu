// dvc_norm.cu -- GroupNorm statistics and the fused GN-apply + SiLU operand
// producer (reading R2-R4), with the Batch-dimension temporal
// shift folded into the element addressing (a3).
//
// Statistics are deterministic and independent of batching (H4): frame t's
// (mean, rstd) per group come only from frame t's shifted input, reduced in a
// fixed order (per-thread fp64 sums over a fixed pixel stride, fixed-order
// merge over 128-pixel chunks).  HBM-bound: one read of the operand.
#include "dvc_norm.cuh"

namespace dvc {

constexpr int kStatPix = 128;   // pixels per partial-statistics chunk

template <typename T>
__global__ void __launch_bounds__(256) gn_partial_kernel(const ShiftSrc<T> X, int G, double2 *__restrict__ partial,
                                                         int nchunk) {
    __shared__ double s_sum[2048];
    __shared__ double s_sq[2048];
    const int t = blockIdx.y, chunk = blockIdx.x;
    const int C = X.C(), nv = C >> 3, npl = 256 / nv;
    const int tid = threadIdx.x, v = tid % nv, pl = tid / nv;
    const int p0 = chunk * kStatPix, p1 = min(X.HW, p0 + kStatPix);
    if (pl < npl) {
        double s[8], q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = q[i] = 0.0;
        for (int p = p0 + pl; p < p1; p += npl) {
            float f[8];
            X.shifted8(t, p, v * 8, f);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                s[i] += (double)f[i];
                q[i] = fma((double)f[i], (double)f[i], q[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s_sum[pl * C + v * 8 + i] = s[i];
            s_sq[pl * C + v * 8 + i] = q[i];
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

__global__ void gn_finalize_kernel(const double2 *__restrict__ partial, int nchunk, int G, int T, double n, double eps,
                                   float2 *__restrict__ stats) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * G) return;
    const int t = i / G, g = i % G;
    double S = 0.0, Q = 0.0;
    for (int c = 0; c < nchunk; ++c) {
        double2 v = partial[((size_t)t * nchunk + c) * G + g];
        S += v.x;
        Q += v.y;
    }
    const double mu = S / n;
    double var = Q / n - mu * mu;   // biased variance (R4)
    if (var < 0.0) var = 0.0;
    stats[i] = make_float2((float)mu, (float)(1.0 / sqrt(var + eps)));
}

// out[t][p][c] = SiLU((Xs[t][p][c] - mu[t,g]) * rstd[t,g] * gamma[c] + beta[c])
template <typename T>
__global__ void __launch_bounds__(256) gn_silu_kernel(const ShiftSrc<T> X, const float2 *__restrict__ stats, int G,
                                                      const T *__restrict__ gamma, const T *__restrict__ beta,
                                                      T *__restrict__ out, long nvec) {
    const int C = X.C(), nv = C >> 3, cg = C / G;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % nv);
        const long pix = i / nv;
        const int t = (int)(pix / X.HW), p = (int)(pix % X.HW);
        float f[8];
        X.shifted8(t, p, v * 8, f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int c = v * 8 + k;
            const float2 st = stats[t * G + c / cg];
            const float z = (f[k] - st.x) * st.y * Elem<T>::to_f(gamma[c]) + Elem<T>::to_f(beta[c]);
            f[k] = silu_f(z);
        }
        store8(out + pix * C + v * 8, f);
    }
}

// Test-only: materialise Xs with the same addressing (dvc_debug_shift_gather).
template <typename T>
__global__ void shift_gather_kernel(const ShiftSrc<T> X, T *__restrict__ out, long nvec) {
    const int C = X.C(), nv = C >> 3;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % nv);
        const long pix = i / nv;
        float f[8];
        X.shifted8((int)(pix / X.HW), (int)(pix % X.HW), v * 8, f);
        store8(out + pix * C + v * 8, f);   // exact: 16-bit -> fp32 -> 16-bit round trip is the identity
    }
}

size_t gn_workspace_bytes(int T, int HW, int G) {
    const int nchunk = (HW + kStatPix - 1) / kStatPix;
    return align256((size_t)T * nchunk * G * sizeof(double2)) + align256((size_t)T * G * sizeof(float2));
}

static int grid_for(long nvec) {
    long b = (nvec + 255) / 256;
    return (int)(b < 148L * 16 ? b : 148L * 16);
}

template <typename T>
static dvc_status gn_silu_t(const NormArgs &a, cudaStream_t stream) {
    ShiftSrc<T> X{reinterpret_cast<const T *>(a.xa), reinterpret_cast<const T *>(a.xb),
                  reinterpret_cast<const T *>(a.carry), a.ca, a.cb, a.cs, a.HW};
    const int C = a.ca + a.cb;
    const int nchunk = (a.HW + kStatPix - 1) / kStatPix;
    double2 *partial = reinterpret_cast<double2 *>(a.ws);
    float2 *stats = reinterpret_cast<float2 *>(reinterpret_cast<uint8_t *>(a.ws) +
                                               align256((size_t)a.T * nchunk * a.G * sizeof(double2)));
    gn_partial_kernel<T><<<dim3(nchunk, a.T), 256, 0, stream>>>(X, a.G, partial, nchunk);
    ++g_launches;
    gn_finalize_kernel<<<(a.T * a.G + 127) / 128, 128, 0, stream>>>(partial, nchunk, a.G, a.T,
                                                                    (double)(C / a.G) * a.HW, (double)a.eps, stats);
    ++g_launches;
    const long nvec = (long)a.T * a.HW * (C / 8);
    gn_silu_kernel<T><<<grid_for(nvec), 256, 0, stream>>>(X, stats, a.G, reinterpret_cast<const T *>(a.gamma),
                                                          reinterpret_cast<const T *>(a.beta),
                                                          reinterpret_cast<T *>(a.out), nvec);
    ++g_launches;
    return check_launch("gn_silu");
}

dvc_status gn_silu_run(const NormArgs &a, dvc_dtype dt, cudaStream_t stream) {
    const int C = a.ca + a.cb;
    DVC_CHECK_ARG(a.ca % 8 == 0 && a.cb % 8 == 0 && C / 8 <= 256, DVC_ERR_UNSUPPORTED,
                  "GN: channel counts must be multiples of 8 and at most 2048");
    DVC_CHECK_ARG(a.G >= 1 && C % a.G == 0, DVC_ERR_DIVISIBILITY, "GN: G=%d must divide C=%d", a.G, C);
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
    const long nvec = (long)a.T * a.HW * ((a.ca + a.cb) / 8);
    shift_gather_kernel<T><<<grid_for(nvec), 256, 0, stream>>>(X, reinterpret_cast<T *>(a.out), nvec);
    ++g_launches;
    return check_launch("shift_gather");
}

dvc_status shift_gather_run(const NormArgs &a, dvc_dtype dt, cudaStream_t stream) {
    DVC_CHECK_ARG(a.ca % 8 == 0 && a.cb % 8 == 0, DVC_ERR_UNSUPPORTED, "gather: channels must be multiples of 8");
    DVC_CHECK_ARG(a.cs <= a.ca, DVC_ERR_UNSUPPORTED, "shift slice must lie in the first source");
    switch (dt) {
        case DVC_BF16: return gather_t<__nv_bfloat16>(a, stream);
        case DVC_F16: return gather_t<__half>(a, stream);
        default: return gather_t<float>(a, stream);
    }
}

}  // namespace dvc
