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

}  // namespace dvc
