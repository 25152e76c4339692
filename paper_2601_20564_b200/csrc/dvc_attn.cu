// dvc_attn.cu -- f1: the self-attention Transformer2D blocks of the full pruned U-Net
// ("U-Net" of SD-2.1 via AdcSR, P:525 parameter count; readings R21-R24).
//
// One block over X [T][H][W][C] (frames independent, no temporal shift):
//   a  = GN(X)                      gn_affine_kernel  (coefficients from box statistics)
//   h0 = proj_in(a)                 1x1 tensor-core conv (conv_run)
//   l1 = LN1(h0)                    layernorm_kernel  (one warp per pixel)
//   qkv = l1 W_qkv^T                1x1 conv, no bias, [T][N][3C]
//   Vt = transpose(v)               vt_kernel: [T][C][Npad] so V is a K-major UMMA operand
//   o  = attention(q, k, v)         attn_tc_kernel (tcgen05, S and PV in TMEM)
//   h1 = out(o) + h0                1x1 conv with residual
//   l2 = LN2(h1)
//   f  = ff1(l2)                    1x1 conv C -> 8C
//   g  = f[:4C] * gelu(f[4C:])      geglu_kernel
//   h2 = ff2(g) + h1                1x1 conv 4C -> C with residual
//   Y  = proj_out(h2) + X           1x1 conv with residual (+ box statistics of Y for the next GN)
//
// attn_tc_kernel: one CTA = 128 queries of one (frame, head); 4 warps, thread r owns query
// row r = TMEM lane r.  Per 128-key tile j:
//   S = Q K_j^T          tcgen05.mma kind::f16 M=128 N=128 K=D (D/16 instructions), S in TMEM
//   softmax              tcgen05.ld of the row, running max m / sum l (exp2 domain), P = 16-bit
//                        probabilities written to shared memory in the UMMA K-major layout
//   PV = P V_j           tcgen05.mma M=128 N=D K=128 into a second TMEM region
//   O = O * alpha + PV   in registers (online softmax, no TMEM read-modify-write)
// K/V tiles are double-buffered with cp.async (zero-filled past N; masked keys get p = 0).
// All operands use the no-swizzle canonical layout: 8-row x 16-byte core matrices, core
// matrices adjacent in K 128 B apart (LBO), 8-row groups SBO apart.
#include <cuda.h>
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
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total8; i += (long)gridDim.x * blockDim.x) {
        const long pix = i / c8;
        const int c = (int)(i - pix * c8) * 8;
        const int t = (int)(pix / HW);
        float f[8];
        load8(x + pix * C + c, f);
        const float2 *cf = coef + (size_t)t * C + c;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float2 s = cf[k];
            f[k] = fmaf(f[k], s.x, s.y);
        }
        store8(y + pix * C + c, f);
    }
    griddep_launch();
}

// LayerNorm over the C channels of each pixel (R21): one warp per pixel, fp32 two-pass
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

// GEGLU (R21): g[m][j] = f[m][j] * gelu(f[m][C4 + j]), exact erf GELU.
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

// V part of qkv [T][N][3C] -> Vt [T][C][Npad] (zero for n >= N): 32x32 tiles through smem.
template <typename T>
__global__ void __launch_bounds__(256) vt_kernel(const T *__restrict__ qkv, T *__restrict__ vt, int N, int Npad,
                                                 int C) {
    griddep_wait();
    __shared__ T tile[32][33];
    const int t = blockIdx.z;
    const int n0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) {
        const int n = n0 + r, c = c0 + tx;
        T v = Elem<T>::from_f(0.f);
        if (n < N && c < C) v = qkv[((size_t)t * N + n) * 3 * C + 2 * C + c];
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int c = c0 + r, n = n0 + tx;
        if (c < C && n < Npad) vt[((size_t)t * C + c) * Npad + n] = tile[tx][r];
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
constexpr int kAttnThreads = 128;
template <int D>
struct AttnSmem {
    static constexpr int Q = 128 * D * 2;        // [128 q][D]      SBO = D*16
    static constexpr int K = 128 * D * 2;        // [128 keys][D]   SBO = D*16
    static constexpr int V = D * 128 * 2;        // [D][128 keys]   SBO = 2048
    static constexpr int P = 128 * 128 * 2;      // [128 q][128 keys] SBO = 2048
    static constexpr int off_q = 0, off_k = Q, off_v = off_k + 2 * K, off_p = off_v + 2 * V;
    static constexpr int off_bar = off_p + P;
    static constexpr int bytes = off_bar + 64;
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
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

template <typename T, int D>
__global__ void __launch_bounds__(kAttnThreads, 1) attn_tc_kernel(const T *__restrict__ qkv, const T *__restrict__ vt,
                                                                  T *__restrict__ out, int N, int Npad, int C,
                                                                  float scale_log2, uint32_t idesc_s,
                                                                  uint32_t idesc_o) {
    using L = AttnSmem<D>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = smem_u32(smem);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::off_bar);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smem + L::off_bar + 16);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int t = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * 128;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc<1>(smem_u32(tslot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t tS = tmem, tO = tmem + 128;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    griddep_wait();

    const size_t ld = 3 * (size_t)C;
    const T *qbase = qkv + (size_t)t * N * ld + h * D;
    const T *kbase = qbase + C;
    const T *vbase = vt + ((size_t)t * C + h * D) * Npad;
    constexpr int DC = D / 8;   // 16-byte chunks per Q/K row
    // Q tile
    for (int i = tid; i < 128 * DC; i += kAttnThreads) {
        const int r = i / DC, kc = i - r * DC;
        const int n = q0 + r;
        const T *src = qbase + (size_t)(n < N ? n : 0) * ld + kc * 8;
        cp_async_16(sb + L::off_q + (r >> 3) * (D * 16) + kc * 128 + (r & 7) * 16, src, n < N ? 16u : 0u);
    }
    auto load_kv = [&](int j, int buf) {
        const int k0 = j * 128;
        for (int i = tid; i < 128 * DC; i += kAttnThreads) {
            const int r = i / DC, kc = i - r * DC;
            const int n = k0 + r;
            const T *src = kbase + (size_t)(n < N ? n : 0) * ld + kc * 8;
            cp_async_16(sb + L::off_k + buf * L::K + (r >> 3) * (D * 16) + kc * 128 + (r & 7) * 16, src,
                        n < N ? 16u : 0u);
        }
        for (int i = tid; i < D * 16; i += kAttnThreads) {
            const int r = i >> 4, kc = i & 15;
            const T *src = vbase + (size_t)r * Npad + k0 + kc * 8;
            cp_async_16(sb + L::off_v + buf * L::V + (r >> 3) * 2048 + kc * 128 + (r & 7) * 16, src, 16u);
        }
    };
    load_kv(0, 0);
    cp_async_commit();

    const int nkt = (N + 127) / 128;
    float o[D];
#pragma unroll
    for (int i = 0; i < D; ++i) o[i] = 0.f;
    float m = -INFINITY, l = 0.f;
    uint32_t ph_s = 0, ph_o = 0;
    const int row = tid;
    const uint32_t p_row = sb + L::off_p + (row >> 3) * 2048 + (row & 7) * 16;

    for (int j = 0; j < nkt; ++j) {
        const int buf = j & 1;
        if (j + 1 < nkt) {
            load_kv(j + 1, buf ^ 1);
            cp_async_commit();
            cp_async_wait_1();
        } else {
            cp_async_wait_all();
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t qa = sb + L::off_q, ka = sb + L::off_k + buf * L::K;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const uint64_t ad = ((uint64_t)desc_hi_noswz(D * 16) << 32) | desc_lo(qa + ks * 256, 128);
                const uint64_t bd = ((uint64_t)desc_hi_noswz(D * 16) << 32) | desc_lo(ka + ks * 256, 128);
                tc_mma(tS, ad, bd, idesc_s, ks > 0);
            }
            tc_commit(&bars[0]);
        }
        mbar_wait(&bars[0], ph_s);
        ph_s ^= 1;
        tc_fence_after();
        // ---- softmax of row `row` over this key tile
        const int kvalid = N - j * 128;   // keys >= kvalid are padding
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint32_t r[16];
            tmem_ld16(tS + lane_off + c * 16, r);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float s = __uint_as_float(r[i]);
                mx = (c * 16 + i < kvalid) ? fmaxf(mx, s) : mx;
            }
        }
        const float m_new = fmaxf(m, mx * scale_log2);
        const float alpha = ex2f(m - m_new);
        float rs = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint32_t r[16];
            tmem_ld16(tS + lane_off + c * 16, r);
            float p[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float e = ex2f(fmaf(__uint_as_float(r[i]), scale_log2, -m_new));
                p[i] = (c * 16 + i < kvalid) ? e : 0.f;
                rs += p[i];
            }
            st_shared_v4(p_row + (2 * c) * 128, pack2<T>(p[0], p[1]), pack2<T>(p[2], p[3]), pack2<T>(p[4], p[5]),
                         pack2<T>(p[6], p[7]));
            st_shared_v4(p_row + (2 * c + 1) * 128, pack2<T>(p[8], p[9]), pack2<T>(p[10], p[11]),
                         pack2<T>(p[12], p[13]), pack2<T>(p[14], p[15]));
        }
        l = l * alpha + rs;
        m = m_new;
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t pa = sb + L::off_p, va = sb + L::off_v + buf * L::V;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint64_t ad = ((uint64_t)desc_hi_noswz(2048) << 32) | desc_lo(pa + ks * 256, 128);
                const uint64_t bd = ((uint64_t)desc_hi_noswz(2048) << 32) | desc_lo(va + ks * 256, 128);
                tc_mma(tO, ad, bd, idesc_o, ks > 0);
            }
            tc_commit(&bars[1]);
        }
        mbar_wait(&bars[1], ph_o);
        ph_o ^= 1;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(tO + lane_off + c * 16, r);
#pragma unroll
            for (int i = 0; i < 16; ++i) o[c * 16 + i] = fmaf(o[c * 16 + i], alpha, __uint_as_float(r[i]));
        }
        tc_fence_before();
    }
    // ---- epilogue: O / l, 16-bit store of this row's D channels
    const int n = q0 + row;
    if (n < N) {
        const float inv = 1.f / l;
        T *y = out + ((size_t)t * N + n) * C + h * D;
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
            float f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = o[c * 8 + i] * inv;
            store8(y + c * 8, f);
        }
    }
    griddep_launch();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<1>(tmem, 256);
}

// ----------------------------------------------------------------- host side
static int grid_for(long work, int threads) {
    long b = (work + threads - 1) / threads;
    return (int)(b < 148L * 16 ? (b > 0 ? b : 1) : 148L * 16);
}

template <typename T, int D>
static dvc_status attn_tc_launch(const void *qkv, const void *vt, void *out, int T_, int N, int Npad, int C,
                                 cudaStream_t stream) {
    using L = AttnSmem<D>;
    const void *kern = reinterpret_cast<const void *>(attn_tc_kernel<T, D>);
    if (!smem_attr_ok(kern, L::bytes))
        DVC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::bytes));
    const int bf = std::is_same<T, __nv_bfloat16>::value ? 1 : 0;
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
    DVC_CUDA(launch_pdl(attn_tc_kernel<T, D>, dim3((N + 127) / 128, C / D, T_), dim3(kAttnThreads), (size_t)L::bytes,
                        stream, 1, reinterpret_cast<const T *>(qkv), reinterpret_cast<const T *>(vt),
                        reinterpret_cast<T *>(out), N, Npad, C, scale_log2, make_idesc(bf, 128, 128),
                        make_idesc(bf, 128, D)));
    ++g_launches;
    return DVC_OK;
}

size_t attn_vt_bytes(int T, int N, int C, dvc_dtype dt) {
    return align256((size_t)T * C * (size_t)((N + 127) / 128 * 128) * dt_size(dt));
}

template <typename T>
static dvc_status attention_t(const void *qkv, int T_, int N, int C, int D, void *vt, void *out, cudaStream_t s) {
    const int Npad = (N + 127) / 128 * 128;
    DVC_CUDA(launch_pdl(vt_kernel<T>, dim3(Npad / 32, (C + 31) / 32, T_), dim3(256), 0, s, 1,
                        reinterpret_cast<const T *>(qkv), reinterpret_cast<T *>(vt), N, Npad, C));
    ++g_launches;
    ProfSlot slot = prof_begin(s);
    dvc_status st;
    switch (D) {
        case 16: st = attn_tc_launch<T, 16>(qkv, vt, out, T_, N, Npad, C, s); break;
        case 32: st = attn_tc_launch<T, 32>(qkv, vt, out, T_, N, Npad, C, s); break;
        case 48: st = attn_tc_launch<T, 48>(qkv, vt, out, T_, N, Npad, C, s); break;
        default: st = attn_tc_launch<T, 64>(qkv, vt, out, T_, N, Npad, C, s); break;
    }
    prof_end_aux(slot, s, "attn_tc");
    return st;
}

dvc_status attention_run(const void *qkv, int T_, int N, int C, int D, dvc_dtype dt, void *vt, void *out,
                         cudaStream_t s) {
    DVC_CHECK_ARG(T_ >= 1 && T_ < 65536 && N >= 1 && C >= 1, DVC_ERR_ARG, "attention: empty shape");
    DVC_CHECK_ARG(D == 16 || D == 32 || D == 48 || D == 64, DVC_ERR_UNSUPPORTED, "attention: head_dim %d not in {16,32,48,64}",
                  D);
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
            default: attn_simt_kernel<64><<<g, 128, 0, s>>>(q, o, N, C, scale); break;
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
           attn_vt_bytes(T, H * W, C, dt) + align256((size_t)T * C * 8) + box_stats_bytes(T, H, W, C);
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
    void *vt = take(attn_vt_bytes(T, H * W, C, b.dt));
    float2 *coef = reinterpret_cast<float2 *>(take((size_t)T * C * 8));
    void *bst = take(box_stats_bytes(T, H, W, C));
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
    if ((st = lin(A, C, b.ff1_w, b.ff1_b, 8 * C, nullptr, big, nullptr)) != DVC_OK) return st;            // f
    if ((st = ew(2, b.dt, big, nullptr, nullptr, Fb, (long)px, 4 * C, 0.f, s)) != DVC_OK) return st;      // g
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
    *bytes = dt == DVC_F32 ? 0 : attn_vt_bytes(T, N, C, dt);
    return DVC_OK;
}

dvc_status dvc_attention_forward(const void *qkv, int T, int N, int C, int head_dim, dvc_dtype dt, void *out,
                                 void *workspace, size_t ws_bytes, void *stream) {
    DVC_CHECK_ARG(qkv && out && dt_valid(dt), DVC_ERR_ARG, "null argument / bad dtype");
    DVC_CHECK_ARG(C % 8 == 0, DVC_ERR_UNSUPPORTED, "attention: C must be a multiple of 8");
    if (dt != DVC_F32) {
        DVC_CHECK_ARG(workspace && ws_bytes >= attn_vt_bytes(T, N, C, dt), DVC_ERR_WORKSPACE, "workspace too small");
        DVC_CHECK_ARG(((uintptr_t)workspace & 255) == 0 && ((uintptr_t)qkv & 15) == 0 && ((uintptr_t)out & 15) == 0,
                      DVC_ERR_ARG, "workspace 256-byte, qkv/out 16-byte aligned");
    }
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    return attention_run(qkv, T, N, C, head_dim, dt, workspace, out, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
