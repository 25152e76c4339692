// dvc_unshuffle.cu -- a1, PixelUnshuffle ("PixelUnshuffle operation for
// space-to-depth"; torch channel order, R12):
//   latent[t][y][x][c*s*s + i*s + j] = frames[t][c][s*y + i][s*x + j]
// A pure permutation (bit-exact).  HBM-bound: one read + one write.
//
// Fast path (16-bit, s = 8): the 8 pixels j = 0..7 of one input row segment are
// 16 contiguous bytes and land as 16 contiguous bytes of the output channel
// vector, so every 128-bit load maps to one 128-bit store.  A block stages
// 24 rows x 16 output pixels (3 colours x 8 rows, 256 B each) in shared
// memory so both the loads (256 B runs per input row) and the stores (16
// pixels x 384 B contiguous) are coalesced.
#include "dvc_norm.cuh"

namespace dvc {

constexpr int kUxb = 16;   // output pixels per block pass (fast path)
constexpr int kUpass = 4;  // passes per block: 4 independent 16-byte loads in flight per thread

__global__ void __launch_bounds__(384) unshuffle8_16bit_kernel(const uint4 *__restrict__ F, uint4 *__restrict__ L,
                                                               int T, int H, int W) {
    __shared__ uint4 tile[kUpass][24][kUxb];
    const int h = H / 8, w = W / 8;
    const int xb = blockIdx.x, y = blockIdx.y, t = blockIdx.z;
    const int k = threadIdx.x;
    {   // read: k -> (gi = c*8 + i, px): consecutive threads walk along one input row; all passes'
        // loads are issued before any is consumed (memory-level parallelism for the HBM stream)
        const int gi = k / kUxb, px = k % kUxb;
        const int c = gi >> 3, i = gi & 7;
        const uint4 *row = F + ((((size_t)t * 3 + c) * H + 8 * y + i) * W) / 8;
#pragma unroll
        for (int q = 0; q < kUpass; ++q) {
            const int x = (xb * kUpass + q) * kUxb + px;
            if (x < w) tile[q][gi][px] = __ldg(row + x);
        }
    }
    __syncthreads();
    {   // write: k -> (px, gi): consecutive threads fill consecutive 16-byte granules of the output
        const int px = k / 24, gi = k % 24;
#pragma unroll
        for (int q = 0; q < kUpass; ++q) {
            const int x = (xb * kUpass + q) * kUxb + px;
            if (x < w) L[(((size_t)t * h + y) * w + x) * 24 + gi] = tile[q][gi][px];
        }
    }
}

// Generic path (any s, any dtype): one element per thread.
template <typename T>
__global__ void unshuffle_generic_kernel(const T *__restrict__ F, T *__restrict__ L, int T_, int H, int W, int s,
                                         long n) {
    const int h = H / s, w = W / s, CL = 3 * s * s;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int k = (int)(e % CL);
        const long pix = e / CL;
        const int x = (int)(pix % w), y = (int)((pix / w) % h);
        const int t = (int)(pix / ((long)w * h));
        const int c = k / (s * s), i = (k / s) % s, j = k % s;
        L[e] = F[(((long)t * 3 + c) * H + s * y + i) * W + s * x + j];
    }
}

dvc_status unshuffle_run(const void *frames, dvc_dtype dt, int T, int H, int W, int s, void *latent,
                         cudaStream_t stream) {
    if (s == 8 && dt != DVC_F32 && ((uintptr_t)frames & 15) == 0 && ((uintptr_t)latent & 15) == 0) {
        dim3 grid(ceil_div(W / 8, kUxb * kUpass), H / 8, T);
        unshuffle8_16bit_kernel<<<grid, 384, 0, stream>>>(reinterpret_cast<const uint4 *>(frames),
                                                          reinterpret_cast<uint4 *>(latent), T, H, W);
        ++g_launches;
        return check_launch("unshuffle8");
    }
    const long n = (long)T * 3 * H * W;
    const int grid = (int)((n + 255) / 256 < 148L * 32 ? (n + 255) / 256 : 148L * 32);
    if (dt == DVC_F32)
        unshuffle_generic_kernel<float><<<grid, 256, 0, stream>>>(reinterpret_cast<const float *>(frames),
                                                                  reinterpret_cast<float *>(latent), T, H, W, s, n);
    else
        unshuffle_generic_kernel<uint16_t><<<grid, 256, 0, stream>>>(
            reinterpret_cast<const uint16_t *>(frames), reinterpret_cast<uint16_t *>(latent), T, H, W, s, n);
    ++g_launches;
    return check_launch("unshuffle_generic");
}

// ----------------------------------------------------------------- 8-bit HWC frames (R14)
// frames [T][H][W][3] bytes, value u / 255 rounded once to the latent type: fp32 = u / 255 correctly
// rounded (__fdiv_rn); 16-bit = the fp32 product u * fl(1/255) rounded to 16 bits, which equals the
// exactly rounded RNE16(u / 255) for every u in 0..255 (fp16 and bf16; exhaustive test G2).
template <typename O> __device__ __forceinline__ O u8_to(uint32_t u);
template <> __device__ __forceinline__ float u8_to<float>(uint32_t u) { return __fdiv_rn((float)u, 255.0f); }
template <> __device__ __forceinline__ __nv_bfloat16 u8_to<__nv_bfloat16>(uint32_t u) {
    return __float2bfloat16_rn((float)u * (1.0f / 255.0f));
}
template <> __device__ __forceinline__ __half u8_to<__half>(uint32_t u) { return __float2half_rn((float)u * (1.0f / 255.0f)); }

// s = 8: thread (pixel, i) reads the 24 bytes of 8 pixels x 3 colours of frame row 8y + i and writes
// channels c*64 + i*8 + [0, 8) for c = 0..2 (8 consecutive threads = one pixel's 3 x 128 contiguous
// bytes in 16-bit)
template <typename O>
__global__ void __launch_bounds__(256) unshuffle8_u8_kernel(const uint8_t *__restrict__ F, O *__restrict__ L, int T,
                                                            int H, int W) {
    const int h = H / 8, w = W / 8;
    const long n = (long)T * h * w * 8;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e & 7);
        const long pix = e >> 3;
        const int x = (int)(pix % w), y = (int)((pix / w) % h), t = (int)(pix / ((long)w * h));
        // 24 bytes = three 8-byte words (8-byte aligned: W % 8 == 0)
        const uint2 *src = reinterpret_cast<const uint2 *>(F + (((long)t * H + 8 * y + i) * W + 8 * x) * 3);
        const uint2 q0 = __ldg(src), q1 = __ldg(src + 1), q2 = __ldg(src + 2);
        const uint32_t wv[6] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y};
        uint32_t b[24];
#pragma unroll
        for (int q = 0; q < 24; ++q) b[q] = (wv[q >> 2] >> (8 * (q & 3))) & 0xFFu;
        O *dst = L + pix * 192 + i * 8;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            O v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = u8_to<O>(b[3 * j + c]);
            if constexpr (sizeof(O) == 2) {
                *reinterpret_cast<uint4 *>(dst + c * 64) = *reinterpret_cast<const uint4 *>(v);
            } else {
                *reinterpret_cast<uint4 *>(dst + c * 64) = *reinterpret_cast<const uint4 *>(v);
                *reinterpret_cast<uint4 *>(dst + c * 64 + 4) = *reinterpret_cast<const uint4 *>(v + 4);
            }
        }
    }
}

template <typename O>
__global__ void unshuffle_u8_generic_kernel(const uint8_t *__restrict__ F, O *__restrict__ L, int T_, int H, int W,
                                            int s, long n) {
    const int h = H / s, w = W / s, CL = 3 * s * s;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int k = (int)(e % CL);
        const long pix = e / CL;
        const int x = (int)(pix % w), y = (int)((pix / w) % h);
        const int t = (int)(pix / ((long)w * h));
        const int c = k / (s * s), i = (k / s) % s, j = k % s;
        L[e] = u8_to<O>(F[(((long)t * H + s * y + i) * W + s * x + j) * 3 + c]);
    }
}

template <typename O>
static void unshuffle_u8_launch(const uint8_t *F, void *L, int T, int H, int W, int s, cudaStream_t stream) {
    if (s == 8 && ((uintptr_t)L & 15) == 0 && ((uintptr_t)F & 7) == 0) {
        const long n = (long)T * (H / 8) * (W / 8) * 8;
        const int grid = (int)((n + 255) / 256 < 148L * 16 ? (n + 255) / 256 : 148L * 16);
        unshuffle8_u8_kernel<O><<<grid, 256, 0, stream>>>(F, reinterpret_cast<O *>(L), T, H, W);
    } else {
        const long n = (long)T * 3 * H * W;
        const int grid = (int)((n + 255) / 256 < 148L * 32 ? (n + 255) / 256 : 148L * 32);
        unshuffle_u8_generic_kernel<O><<<grid, 256, 0, stream>>>(F, reinterpret_cast<O *>(L), T, H, W, s, n);
    }
}

dvc_status unshuffle_u8_run(const void *frames, int T, int H, int W, int s, void *latent, dvc_dtype dt,
                            cudaStream_t stream) {
    const uint8_t *F = reinterpret_cast<const uint8_t *>(frames);
    if (dt == DVC_F32) unshuffle_u8_launch<float>(F, latent, T, H, W, s, stream);
    else if (dt == DVC_BF16) unshuffle_u8_launch<__nv_bfloat16>(F, latent, T, H, W, s, stream);
    else unshuffle_u8_launch<__half>(F, latent, T, H, W, s, stream);
    ++g_launches;
    return check_launch("unshuffle_u8");
}

}  // namespace dvc
