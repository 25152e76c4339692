// dvc_pack.cu -- weight packing for the TMA conv engines: each (tap, 64-channel
// chunk) B tile of BN output channels becomes one contiguous block of BN x 128 B, so
// a weight-tile TMA reads sequential memory instead of BN rows 9*C_in*2 bytes apart.
#include "dvc_conv.cuh"

namespace dvc {

size_t packed_elems(int cout, int taps, int cs) { return (size_t)taps * ((cs + 63) / 64) * cout * 64; }

template <typename T>
__global__ void pack_kernel(const T *__restrict__ W, int cout, int taps, int cin_total, int off, int cs, int nch,
                            T *__restrict__ out, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % 64);
        size_t r = i / 64;
        const int o = (int)(r % cout);
        r /= cout;
        const int ch = (int)(r % nch);
        const int tap = (int)(r / nch);
        const int c = ch * 64 + k;
        out[i] = c < cs ? W[((size_t)o * taps + tap) * cin_total + off + c] : T(0.f);
    }
}

dvc_status pack_weights_run(const void *W, dvc_dtype dt, int cout, int taps, int cin_total, int off, int cs, void *out,
                            cudaStream_t stream) {
    DVC_CHECK_ARG(dt != DVC_F32, DVC_ERR_ARG, "packing is for the 16-bit tensor-core engines");
    const size_t n = packed_elems(cout, taps, cs);
    const int nch = (cs + 63) / 64;
    const int blocks = (int)((n + 255) / 256 < 148 * 64 ? (n + 255) / 256 : 148 * 64);
    if (dt == DVC_BF16)
        pack_kernel<__nv_bfloat16><<<blocks, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16 *>(W), cout, taps,
                                                               cin_total, off, cs, nch,
                                                               reinterpret_cast<__nv_bfloat16 *>(out), n);
    else
        pack_kernel<__half><<<blocks, 256, 0, stream>>>(reinterpret_cast<const __half *>(W), cout, taps, cin_total, off,
                                                        cs, nch, reinterpret_cast<__half *>(out), n);
    ++g_launches;
    return check_launch("pack_weights");
}

}  // namespace dvc
