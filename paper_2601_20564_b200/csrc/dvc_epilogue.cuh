// dvc_epilogue.cuh -- the staged convolution epilogue shared by the fused (dvc_conv_fz.cu) and TMA
// (dvc_conv_ws.cu) engines: one 32- (or 16-) column chunk of a 128-row accumulator tile.
//
//   registers (thread = box row r, final fp32 values) -> 16-bit rounding -> a swizzled [128][32]
//   tile in shared memory (zeros for rows outside the frame) -> ONE TMA store of the output box
//   {32, BX, BY, 1} (the hardware clips rows outside the tensor) -> the box statistics of the next
//   GroupNorm read back column-wise (a lane pair per two columns, warp q4 = rows 32 q4 .. 32 q4 + 31,
//   packed fp32 pairs) and reduced with the canonical tree of dvc_boxstats.cuh: rows paired by bit 4,
//   then 3, 2, 1, 0 (the xor butterfly's tree, with commutative fp32 adds), warps combined
//   ((w0 + w1) + w2) + w3 -- bit for bit the partials every other producer writes (H4), without 62
//   shuffles per 16 columns and without 32 uncoalesced 16-byte stores per warp instruction.
// Staging layouts match the TMA swizzle of the output maps: 64-byte rows with SWIZZLE_64B (16-byte
// unit j of row r at j ^ ((r >> 1) & 3)), 32-byte rows with SWIZZLE_32B (j ^ ((r >> 2) & 1)).
// All 128 epilogue threads (named barrier 1) call it for every chunk in the same order; two staging
// buffers alternate (the issuing thread waits for the store of chunk i-1 to have read its buffer
// before anybody writes chunk i+1 into it).
#pragma once
#include "dvc_common.cuh"
#include "dvc_ptx.cuh"

namespace dvc {

constexpr int kEpiStage = 128 * 64;   // one staging buffer: 128 rows x 32 columns x 16 bit

template <typename T> struct EpiPk;
template <> struct EpiPk<__nv_bfloat16> {
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    static __device__ __forceinline__ float unpack16(uint16_t u) { return __uint_as_float((uint32_t)u << 16); }
    static __device__ __forceinline__ float2 unpack2(uint32_t u) {
        return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
    }
};
template <> struct EpiPk<__half> {
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    static __device__ __forceinline__ float unpack16(uint16_t u) { return __half2float(__ushort_as_half(u)); }
    static __device__ __forceinline__ float2 unpack2(uint32_t u) {
        return __half22float2(*reinterpret_cast<const __half2 *>(&u));
    }
};

// f[0 .. ncol) += b[0 .. ncol) (ncol = two ? 32 : 16), packed fp32 pairs (FADD2; per-element IEEE rn)
__device__ __forceinline__ void epi_add_bias(float (&f)[32], const float *b, bool two) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        if (i >= 16 && !two) break;
        const float4 e = *reinterpret_cast<const float4 *>(b + i);
        const float2 lo = __fadd2_rn(make_float2(f[i], f[i + 1]), make_float2(e.x, e.y));
        const float2 hi = __fadd2_rn(make_float2(f[i + 2], f[i + 3]), make_float2(e.z, e.w));
        f[i] = lo.x, f[i + 1] = lo.y, f[i + 2] = hi.x, f[i + 3] = hi.y;
    }
}

__device__ __forceinline__ int epi_off(bool two, int r, int j) {
    return two ? r * 64 + ((j ^ ((r >> 1) & 3)) << 4) : r * 32 + ((j ^ ((r >> 2) & 1)) << 4);
}

// f: this row's ncol (= two ? 32 : 16) final values; live: the row is a pixel of the tensor.
// store: issue the TMA store (the box is valid); (c0, x0, y0, t): the box's output coordinates.
// up2: the output maps describe the 2x upsampled tensor with element stride 2 in x and y; the box
// is stored at the four phases (2 x0 + ox, 2 y0 + oy), i.e. exact nearest 2x upsampling.
// stats_col: &stats_box[c0 * 2] (per column: sum, sum of squares) or null; red: 256 floats.
template <typename T>
__device__ __forceinline__ void epi_stage_chunk(const float (&f)[32], bool live, bool two, int r, int q4, int lane,
                                                uint8_t *st, const CUtensorMap *omap32, const CUtensorMap *omap16,
                                                bool issuer, bool store, int c0, int x0, int y0, int t,
                                                float *stats_col, float *red, bool up2 = false, uint32_t bar = 1) {
    const int ncol = two ? 32 : 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (j >= 2 && !two) break;
        uint4 u;
        u.x = live ? EpiPk<T>::pack(f[8 * j + 0], f[8 * j + 1]) : 0u;
        u.y = live ? EpiPk<T>::pack(f[8 * j + 2], f[8 * j + 3]) : 0u;
        u.z = live ? EpiPk<T>::pack(f[8 * j + 4], f[8 * j + 5]) : 0u;
        u.w = live ? EpiPk<T>::pack(f[8 * j + 6], f[8 * j + 7]) : 0u;
        *reinterpret_cast<uint4 *>(st + epi_off(two, r, j)) = u;
    }
    fence_proxy_async_smem();
    asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");   // this epilogue warpgroup's named barrier
    if (issuer) {
        if (store) {
            if (up2) {   // exact 2x nearest upsampling: maps with element stride 2 in x and y, four phases
#pragma unroll
                for (int ph = 0; ph < 4; ++ph)
                    tma_store_4d(two ? omap32 : omap16, smem_u32(st), c0, 2 * x0 + (ph & 1), 2 * y0 + (ph >> 1), t);
            } else {
                tma_store_4d(two ? omap32 : omap16, smem_u32(st), c0, x0, y0, t);
            }
            bulk_commit_group();
        }
        bulk_wait_group_read<1>();   // the other staging buffer has been read: reusable for chunk i+1
    }
    if (stats_col) {
        // lane = (column pair cp = lane / 2, row parity b0 = lane % 2): the 16 rows 32 q4 + 2i + b0 of
        // columns 2cp, 2cp + 1 in packed fp32 pairs (FMUL2 / FADD2, IEEE round-to-nearest per element).
        // The tree over i (i, i + 8), (i, i + 4), (i, i + 2), (i, i + 1) is the canonical one's levels
        // over rows differing in bit 4, 3, 2, 1; its last level (bit 0) is the lane pair (shuffle).
        const int cp = lane >> 1, b0 = lane & 1, c = 2 * cp;
        const bool lv = c < ncol;
        float2 v[16], q[16];
        if (lv) {
            const int j = c >> 3, e = (c & 7) * 2;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int rr = q4 * 32 + 2 * i + b0;
                v[i] = EpiPk<T>::unpack2(*reinterpret_cast<const uint32_t *>(st + epi_off(two, rr, j) + e));
                q[i] = __fmul2_rn(v[i], v[i]);
            }
#pragma unroll
            for (int mm = 8; mm >= 1; mm >>= 1)
#pragma unroll
                for (int k = 0; k < mm; ++k) {
                    v[k] = __fadd2_rn(v[k], v[k + mm]);
                    q[k] = __fadd2_rn(q[k], q[k + mm]);
                }
        } else {
            v[0] = q[0] = make_float2(0.f, 0.f);
        }
        float2 ov, oq;
        ov.x = __shfl_xor_sync(0xffffffffu, v[0].x, 1);
        ov.y = __shfl_xor_sync(0xffffffffu, v[0].y, 1);
        oq.x = __shfl_xor_sync(0xffffffffu, q[0].x, 1);
        oq.y = __shfl_xor_sync(0xffffffffu, q[0].y, 1);
        if (lv && b0 == 0) {   // (row 2i) + (row 2i + 1); fp32 addition is commutative
            const float2 sv = __fadd2_rn(v[0], ov), sq = __fadd2_rn(q[0], oq);
            red[q4 * 32 + c] = sv.x;
            red[q4 * 32 + c + 1] = sv.y;
            red[128 + q4 * 32 + c] = sq.x;
            red[128 + q4 * 32 + c + 1] = sq.y;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
        if (q4 < 2 && lane < ncol) {   // warp 0: sums, warp 1: sums of squares
            const float *src = red + q4 * 128;
            stats_col[lane * 2 + q4] =
                __fadd_rn(__fadd_rn(__fadd_rn(src[lane], src[32 + lane]), src[64 + lane]), src[96 + lane]);
        }
    } else {
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
    }
}

}  // namespace dvc
