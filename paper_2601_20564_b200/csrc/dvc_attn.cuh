// dvc_attn.cuh -- f1 Transformer2D block (dvc_attn.cu), internal interface.
#pragma once
#include "dvc_common.cuh"

namespace dvc {

// One Transformer2D block (device pointers, dt elements; shapes in include/dvc.h dvc_transformer).
struct TF {
    int c, groups, head_dim;
    float eps_gn, eps_ln;
    dvc_dtype dt;
    const void *gn_w, *gn_b, *proj_in_w, *proj_in_b, *ln1_w, *ln1_b, *qkv_w, *out_w, *out_b, *ln2_w, *ln2_b, *ff1_w,
        *ff1_b, *ff2_w, *ff2_b, *proj_out_w, *proj_out_b;
    // FF1 rows pre-interleaved for the GEGLU epilogue (16 value + 16 gate rows per block), or null
    // (then interleaved into the workspace on every call)
    const void *ff1_wi = nullptr, *ff1_bi = nullptr;
};
// interleave b.ff1_w / b.ff1_b into wi [8C][C] / bi [8C] (the GEGLU epilogue's row order)
dvc_status interleave_ff1(const TF &b, void *wi, void *bi, cudaStream_t s);

size_t transformer_ws_bytes(int C, int T, int H, int W, dvc_dtype dt);
dvc_status transformer_validate(const TF &b, int T, int H, int W);
// y may alias x.  stats_x: box statistics of x (null = computed here); stats_y: box statistics of y or null.
dvc_status transformer_launch(const TF &b, const void *x, int T, int H, int W, void *y, void *ws, cudaStream_t s,
                              const void *stats_x = nullptr, void *stats_y = nullptr);
// multi-head self-attention over a packed qkv [T][N][3C] -> out [T][N][C]; ws: attn_ws_bytes scratch (packed operand tiles)
size_t attn_ws_bytes(int T, int N, int C, dvc_dtype dt);
dvc_status attention_run(const void *qkv, int T, int N, int C, int D, dvc_dtype dt, void *vt, void *out,
                         cudaStream_t s);

// y = x * coef.x + coef.y per (frame, channel) (GroupNorm apply without SiLU)
dvc_status gn_affine_run(const void *x, const void *coef, int T, int HW, int C, dvc_dtype dt, void *y,
                         cudaStream_t s);

}  // namespace dvc
