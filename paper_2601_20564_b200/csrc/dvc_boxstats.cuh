// dvc_boxstats.cuh -- the canonical per-channel GroupNorm partial statistics
// ("box statistics") shared by the TMA conv engine's epilogue and the
// standalone box-stats kernel, so both produce bit-identical partials (H4:
// results independent of batching, chunking and of which kernel produced a
// tensor).
//
// For a [T][H][W][C] tensor, frame t is tiled into the spatial boxes of
// choose_box(H, W) (BY x BX <= 128 pixels, row-major box order).  For box b
// and channel c:
//   part[(t * nbox + b) * C + c] = (sum v, sum v*v) over the box's pixels,
// where v is the stored (rounded) value.  Rows r = 0..127 of a box are pixels
// (r / BX, r % BX) (0 outside the box / frame); warp w holds rows 32w..32w+31;
// each warp reduces its 32 rows with the xor butterfly 16, 8, 4, 2, 1
// (reduce-scatter; lane l ends with value index l: l < 16 -> sum of column l,
// l >= 16 -> sum of squares of column l - 16); the 4 warps are combined as
// ((w0 + w1) + w2) + w3.  All in fp32 with explicit _rn operations (no FMA
// contraction), so every producer computes the same bits.
#pragma once
#include "dvc_common.cuh"

namespace dvc {

// x[0..15] = values of 16 columns, x[16..31] = their squares; returns this lane's reduced value
__device__ __forceinline__ float box_reduce_scatter32(float (&x)[32], int lane) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const bool hi = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            const float lo_v = x[i], hi_v = x[i + m];
            const float send = hi ? lo_v : hi_v;
            const float keep = hi ? hi_v : lo_v;
            x[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, m));
        }
    }
    return x[0];
}

// per-row contribution for 16 columns: v (0 for invalid rows) and v*v
__device__ __forceinline__ void box_row_values(const float (&v)[16], bool valid, float (&x)[32]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const float a = valid ? v[i] : 0.f;
        x[i] = a;
        x[16 + i] = __fmul_rn(a, a);
    }
}

__device__ __forceinline__ float box_combine4(const float *red /*[4][32]*/, int lane) {
    return __fadd_rn(__fadd_rn(__fadd_rn(red[lane], red[32 + lane]), red[64 + lane]), red[96 + lane]);
}

}  // namespace dvc
