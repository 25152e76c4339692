#pragma once
#include "dvc_common.cuh"

namespace dvc {

// Internal ResBlock description (device pointers, dt elements).
struct RB {
    int ca, cb, cout, G, P;
    float eps;
    dvc_dtype dt;
    const void *gn1_w, *gn1_b, *conv1_w, *conv1_b, *gn2_w, *gn2_b, *conv2_w, *conv2_b, *sc_w, *sc_b;
    // optional packed weight images (dvc_pack.cu) for the TMA engines; null = use the OHWI weights
    const void *conv1_pk = nullptr, *conv2_pk = nullptr, *sc_pk = nullptr;
};

size_t resblock_ws_bytes(int ca, int cb, int cout, int G, int T, int H, int W, dvc_dtype dt);
dvc_status resblock_validate(const RB &b, int T, int H, int W);
// up2 != 0: y receives nearest_to(block output, up_ho, up_wo) [T][up_ho][up_wo][C_out] with up_ho in
// {2H - 1, 2H}, up_wo in {2W - 1, 2W} (0: 2H / 2W) -- the 2x phase replication clipped at the far edge
// (the 16-bit engines' staged epilogues store it directly; the fp32 path upsamples a workspace copy) --
// and no statistics of y are produced (stats_y must be null).
dvc_status resblock_launch(const RB &b, const void *xa, const void *xb, int T, int H, int W, const void *carry_in,
                           void *carry_out, void *y, void *ws, cudaStream_t stream, const void *stats_a = nullptr,
                           const void *stats_b = nullptr, void *stats_y = nullptr, int up2 = 0, int up_ho = 0,
                           int up_wo = 0);

}  // namespace dvc
