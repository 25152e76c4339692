// dvc_fp8.cu -- f4 variant: fp8 (E4M3) convolutions on the TMA engine (kind::f8f6f4).
//
// dvc_quantize_e4m3: q = sat_E4M3(RNE(x / scale)) element by element (fp32 quotient, IEEE).
// dvc_conv_fp8: y = (s_x * s_w) * conv(q_x, q_w) + b, fp32 accumulate, 16-bit output -- the
// dequantisation scales fold into the epilogue; the operands move as bytes (half the HBM / SMEM
// traffic of 16-bit) and the tensor core runs its fp8 rate (2x the 16-bit dense peak).
#include <cuda_fp8.h>
#include "dvc_conv.cuh"

using namespace dvc;

namespace {
template <typename T>
__global__ void __launch_bounds__(256) quant_e4m3_kernel(const T *__restrict__ x, uint8_t *__restrict__ q, long n8,
                                                         float scale) {
    griddep_wait();
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n8; i += (long)gridDim.x * blockDim.x) {
        float f[8];
        load8(x + i * 8, f);
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t b = (uint32_t)__nv_cvt_float_to_fp8(f[k] / scale, __NV_SATFINITE, __NV_E4M3);
            if (k < 4) lo |= b << (8 * k);
            else hi |= b << (8 * (k - 4));
        }
        *reinterpret_cast<uint2 *>(q + i * 8) = make_uint2(lo, hi);
    }
    griddep_launch();
}
}  // namespace

extern "C" {

dvc_status dvc_quantize_e4m3(const void *x, dvc_dtype dt, size_t n, float scale, void *q, void *stream) {
    DVC_CHECK_ARG(x && q && dt_valid(dt) && n % 8 == 0 && scale > 0.f, DVC_ERR_ARG,
                  "bad arguments (n multiple of 8, scale > 0)");
    DVC_CHECK_ARG(((uintptr_t)x & 15) == 0 && ((uintptr_t)q & 7) == 0, DVC_ERR_ARG, "alignment");
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const long n8 = (long)(n / 8);
    const int blocks = (int)std::min<long>((n8 + 255) / 256, 148L * 16);
    if (n8 == 0) return DVC_OK;
    if (dt == DVC_BF16)
        DVC_CUDA(launch_pdl(quant_e4m3_kernel<__nv_bfloat16>, dim3(blocks), dim3(256), 0, s, 1,
                            reinterpret_cast<const __nv_bfloat16 *>(x), reinterpret_cast<uint8_t *>(q), n8, scale));
    else if (dt == DVC_F16)
        DVC_CUDA(launch_pdl(quant_e4m3_kernel<__half>, dim3(blocks), dim3(256), 0, s, 1,
                            reinterpret_cast<const __half *>(x), reinterpret_cast<uint8_t *>(q), n8, scale));
    else
        DVC_CUDA(launch_pdl(quant_e4m3_kernel<float>, dim3(blocks), dim3(256), 0, s, 1,
                            reinterpret_cast<const float *>(x), reinterpret_cast<uint8_t *>(q), n8, scale));
    ++g_launches;
    return check_launch("quant_e4m3_kernel");
}

dvc_status dvc_conv_fp8(const void *x8, float sx, const void *w8, float sw, const void *bias, int T, int H, int W,
                        int cin, int cout, int taps, dvc_dtype out_dt, void *y, void *stream) {
    DVC_CHECK_ARG(x8 && w8 && y && (taps == 1 || taps == 9) && (out_dt == DVC_BF16 || out_dt == DVC_F16),
                  DVC_ERR_ARG, "bad arguments (taps 1 or 9, 16-bit output)");
    DVC_CHECK_ARG(cin % 32 == 0 && cout % 16 == 0, DVC_ERR_UNSUPPORTED, "fp8 conv: C_in % 32, C_out % 16");
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    ConvDesc d{};
    d.seg[0] = ConvSeg{x8, cin, SEG_SAME, H, W, taps, w8, taps * cin, 0, cin};
    d.nseg = 1;
    d.T = T;
    d.ho = H;
    d.wo = W;
    d.cout = cout;
    d.bias0 = bias;
    d.out = y;
    d.dt = out_dt;
    d.fp8 = 1;
    d.out_scale = sx * sw;
    DVC_CHECK_ARG(g_ws_cg != 0 && conv_ws_applicable(d), DVC_ERR_UNSUPPORTED, "fp8 conv needs the TMA engine");
    ProfSlot slot = prof_begin(reinterpret_cast<cudaStream_t>(stream));
    st = conv_ws_run(d, reinterpret_cast<cudaStream_t>(stream));
    prof_end(slot, reinterpret_cast<cudaStream_t>(stream), conv_flops(d), "ws_fp8", d);
    return st;
}

dvc_status dvc_conv(const void *x, const void *w, const void *bias, int T, int H, int W, int cin, int cout, int taps,
                    dvc_dtype dt, void *y, void *stream) {
    DVC_CHECK_ARG(x && w && y && (taps == 1 || taps == 9) && dt_valid(dt), DVC_ERR_ARG, "bad arguments");
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    ConvDesc d{};
    d.seg[0] = ConvSeg{x, cin, SEG_SAME, H, W, taps, w, taps * cin, 0, cin};
    d.nseg = 1;
    d.T = T;
    d.ho = H;
    d.wo = W;
    d.cout = cout;
    d.bias0 = bias;
    d.out = y;
    d.dt = dt;
    return conv_run(d, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
