// dvc_common.cuh -- shared device/host helpers of libdvc (product path only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstddef>
#include <utility>
#include <type_traits>
#include <cstdlib>
#include "../../include/dvc.h"

namespace dvc {

// Experiment knobs (A/B timing, work-skipping debug switches) are read from the environment only
// in builds compiled with -DDVC_EXPERIMENTS (tools/ab.sh); the product library ignores every DVC_*
// variable, so no environment can make it skip work or change its arithmetic.
inline const char *dvc_knob(const char *name) {
#ifdef DVC_EXPERIMENTS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

// ----------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
extern int g_launches;   // kernels launched through launch helpers (bookkeeping for bench)

#define DVC_CHECK_ARG(cond, code, ...)        \
    do {                                      \
        if (!(cond)) {                        \
            ::dvc::set_error(__VA_ARGS__);    \
            return code;                      \
        }                                     \
    } while (0)

#define DVC_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            ::dvc::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                             cudaGetErrorString(e_));                               \
            return DVC_ERR_CUDA;                                                    \
        }                                                                           \
    } while (0)

// Returns DVC_ERR_CUDA if a previous asynchronous launch failed (sticky or not).
dvc_status check_launch(const char *what);
dvc_status check_device();   // cached: current device must be sm_100

inline size_t dt_size(dvc_dtype dt) { return dt == DVC_F32 ? 4 : 2; }
inline bool dt_valid(dvc_dtype dt) { return dt == DVC_BF16 || dt == DVC_F16 || dt == DVC_F32; }

// ----------------------------------------------------------------- element conversion
template <typename T> struct Elem;
template <> struct Elem<float> {
    static __device__ __forceinline__ float to_f(float v) { return v; }
    static __device__ __forceinline__ float from_f(float v) { return v; }
};
template <> struct Elem<__half> {
    static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
    static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
};
template <> struct Elem<__nv_bfloat16> {
    static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

// 8 consecutive elements as one vector unit (16 B for 16-bit types, 32 B for fp32).
template <typename T>
struct alignas(16) Vec8 {
    T v[8];
};

template <typename T>
__device__ __forceinline__ void load8(const T *p, float (&f)[8]) {
    Vec8<T> u;
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4 *>(&u) = __ldg(reinterpret_cast<const uint4 *>(p));
    } else {
        reinterpret_cast<float4 *>(&u)[0] = __ldg(reinterpret_cast<const float4 *>(p));
        reinterpret_cast<float4 *>(&u)[1] = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = Elem<T>::to_f(u.v[i]);
}

template <typename T>
__device__ __forceinline__ void store8(T *p, const float (&f)[8]) {
    Vec8<T> u;
#pragma unroll
    for (int i = 0; i < 8; ++i) u.v[i] = Elem<T>::from_f(f[i]);
    if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4 *>(p) = *reinterpret_cast<uint4 *>(&u);
    } else {
        reinterpret_cast<float4 *>(p)[0] = reinterpret_cast<float4 *>(&u)[0];
        reinterpret_cast<float4 *>(p)[1] = reinterpret_cast<float4 *>(&u)[1];
    }
}

// Round 16 fp32 values to the 16-bit storage type with packed conversions (one cvt per pair)
// into two 8-element vectors, and replace f[] by the stored values (the box statistics use the
// stored values, R17).  Same rounding as Elem<T>::from_f element by element.
template <typename T>
__device__ __forceinline__ void round_store16(float (&f)[16], Vec8<T> &lo, Vec8<T> &hi) {
    if constexpr (sizeof(T) == 2) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (std::is_same<T, __nv_bfloat16>::value) {
                __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
                w[i] = *reinterpret_cast<uint32_t *>(&h);
                f[2 * i] = __uint_as_float(w[i] << 16);
                f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
            } else {
                __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
                w[i] = *reinterpret_cast<uint32_t *>(&h);
                const float2 b = __half22float2(h);
                f[2 * i] = b.x;
                f[2 * i + 1] = b.y;
            }
        }
        *reinterpret_cast<uint4 *>(&lo) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4 *>(&hi) = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            lo.v[i] = Elem<T>::from_f(f[i]);
            hi.v[i] = Elem<T>::from_f(f[8 + i]);
        }
    }
}

__device__ __forceinline__ float silu_f(float z) { return z / (1.0f + __expf(-z)); }

// SiLU(z) = z / (1 + e^-z) for 16-bit outputs: two MUFU ops (ex2.approx, rcp.approx,
// each <= 2 ulp in fp32), far below the 16-bit rounding of the result.
__device__ __forceinline__ float tanh_fast(float x) {   // tanh.approx.f32: max rel. error 2^-11
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

inline int ceil_div(long a, long b) { return (int)((a + b - 1) / b); }

// NVTX ranges (header-only NVTX v3: a no-op branch unless a tool such as ncu / nsys injects itself):
// one per C-ABI call and one per U-Net block, so profiles can be filtered by block
// (ncu --nvtx --nvtx-include "regex:block 05 .*/").
struct NvtxRange {
    explicit NvtxRange(const char *fmt, ...) __attribute__((format(printf, 2, 3)));
    ~NvtxRange();
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// true if `kern` already allows >= smem bytes of dynamic shared memory (records the new size otherwise)
dvc_status ensure_smem(const void *kern, int smem);   // cudaFuncSetAttribute, cached

// Programmatic dependent launch (PDL): kernels of the decode chain are launched with
// programmatic stream serialisation, so a kernel's CTAs may start (prologue: barriers, TMEM,
// tensor-map prefetch, weight-side loads) while its predecessor drains.  griddep_wait() blocks
// until the predecessor grid has completed and its memory is visible -- every kernel calls it
// before its first access to activation data; without the launch attribute it is a no-op.
// griddep_launch() lets the successor grid be scheduled (correctness never depends on it).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// PDL (programmatic dependent launch) for the decode chain; DVC_PDL=0 disables it
bool pdl_enabled();
// launch `kern` with programmatic stream serialisation (+ an optional cluster dimension)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, int cluster,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (cluster > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------- shifted-operand addressing (a3)
// One ResBlock input X = concat(xa[ca], xb[cb]) over frames [T][HW].  The
// Batch-dimension temporal shift is pure addressing:
//   Xs[t][p][c] = c < cs ? (t > 0 ? X[t-1][p][c] : carry[p][c] (0 if null)) : X[t][p][c]
// used identically by the GN statistics, the GN/SiLU operand producer and the
// test-only gather.
template <typename T>
struct ShiftSrc {
    const T *xa, *xb, *carry;
    int ca, cb, cs;   // cs = C_in / P (0 = no shift)
    int HW;

    __device__ __forceinline__ int C() const { return ca + cb; }

    // raw (unshifted) 8-vector X[t][p][c..c+7]; c % 8 == 0 and ca % 8 == 0
    __device__ __forceinline__ void raw8(int t, int p, int c, float (&f)[8]) const {
        if (c < ca) load8(xa + ((size_t)t * HW + p) * ca + c, f);
        else load8(xb + ((size_t)t * HW + p) * cb + (c - ca), f);
    }
    // shifted-slice source for the same channels: frame t-1 or the carry
    __device__ __forceinline__ void prev8(int t, int p, int c, float (&f)[8]) const {
        if (t > 0) { raw8(t - 1, p, c, f); return; }
        if (carry == nullptr) {
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = 0.f;
            return;
        }
        // carry is [HW][cs]; cs may not be a multiple of 8: per element
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            int cc = c + i;
            f[i] = cc < cs ? Elem<T>::to_f(carry[(size_t)p * cs + cc]) : 0.f;
        }
    }
    __device__ __forceinline__ void shifted8(int t, int p, int c, float (&f)[8]) const {
        if (c + 8 <= cs) { prev8(t, p, c, f); return; }
        raw8(t, p, c, f);
        if (c < cs) {   // vector straddles the slice boundary
            float g[8];
            prev8(t, p, c, g);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (c + i < cs) f[i] = g[i];
        }
    }
};

}  // namespace dvc
