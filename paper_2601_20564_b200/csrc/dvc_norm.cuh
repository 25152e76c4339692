#pragma once
#include "dvc_common.cuh"

namespace dvc {

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// One GroupNorm(+SiLU) application over the (optionally shifted) operand
// X = concat(xa[ca], xb[cb]) of T frames x HW pixels.
struct NormArgs {
    const void *xa, *xb, *carry;
    int ca, cb, cs;          // cs = shifted slice width (0 = no shift)
    int T, HW, G;
    float eps;
    const void *gamma, *beta;
    void *out;               // [T][HW][ca+cb]
    void *ws;                // gn_workspace_bytes(T, HW, G)
};

size_t gn_workspace_bytes(int T, int HW, int G, int C);

// Box statistics (dvc_boxstats.cuh) of the sources of a GN operand.
struct BoxStatsIn {
    const void *a, *b;   // [T][nbox][C_a] / [T][nbox][C_b] float2 (b may be null when C_b == 0)
    const void *carry;   // [nbox][cs] float2 of the carry slice, or null (zeros)
};
size_t box_stats_bytes(int T, int H, int W, int C);
// GN coefficients only: a.out <- float2 [T][C] (scale, beta - mean*scale) for the fused conv
dvc_status gn_coef_box_run(const NormArgs &a, const BoxStatsIn &bs, int H, int W, dvc_dtype dt, cudaStream_t stream);
// GN1/GN2 + SiLU from box statistics (no statistics pass over the operand); ws >= T*C*8 bytes
dvc_status gn_silu_box_run(const NormArgs &a, const BoxStatsIn &bs, int H, int W, dvc_dtype dt, cudaStream_t stream);
dvc_status nearest_run(const void *src, void *dst, int T, int hi, int wi, int ho, int wo, int C, dvc_dtype dt,
                       cudaStream_t stream);
dvc_status gn_silu_run(const NormArgs &a, dvc_dtype dt, cudaStream_t stream);
dvc_status shift_gather_run(const NormArgs &a, dvc_dtype dt, cudaStream_t stream);

dvc_status unshuffle_run(const void *frames, dvc_dtype dt, int T, int H, int W, int s, void *latent,
                         cudaStream_t stream);
dvc_status unshuffle_u8_run(const void *frames, int T, int H, int W, int s, void *latent, dvc_dtype dt,
                            cudaStream_t stream);   // 8-bit HWC frames (R14)

}  // namespace dvc
