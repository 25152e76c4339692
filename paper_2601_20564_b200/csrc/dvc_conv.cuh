// dvc_conv.cuh -- one description of "a convolution of the hot path", executed
// either by the tcgen05 implicit-GEMM engine (16-bit) or the fp32 SIMT engine
// (DVC_F32 validation mode).
//
// A convolution is a sum of K segments.  Segment s contributes
//   sum_{tap} sum_{c < c_src} W_s[n][col0 + tap*tapstride + c] * A_s(m, tap, c)
// where A_s is an activation gathered from `src` by an addressing mode:
//   SEG_SAME      3x3 pad 1 (taps=9) or 1x1 (taps=1) at the output resolution
//   SEG_STRIDE2   3x3 stride 2 pad 1 (down-sampler glue, R11)
//   SEG_UPNEAREST 3x3 pad 1 over nearest_to(src, ho, wo) (up-sampler glue, R11)
//   SEG_UNSHUFFLE8 1x1 over PixelUnshuffle(frames, 8) (a1 fused into a2, R12)
// Output row m = (t*ho + y)*wo + x; out[m][n] = bias0[n] (+bias1[n]) + sum + residual[m][n].
#pragma once
#include "dvc_common.cuh"

namespace dvc {

enum SegMode { SEG_SAME = 0, SEG_STRIDE2 = 1, SEG_UPNEAREST = 2, SEG_UNSHUFFLE8 = 3 };

struct ConvSeg {
    const void *src;   // activations [T][hi][wi][c_src] (or frames [T][3][8ho][8wo])
    int c_src;         // channels per src pixel (row stride in elements)
    int mode;          // SegMode
    int hi, wi;        // src spatial dims
    int taps;          // 9 or 1
    const void *w;     // weights as a 2D [cout][w_ld] matrix
    int w_ld;          // row length of w (elements)
    int w_col0;        // first column of this segment
    int w_tapstride;   // columns between taps
    int packed;        // 1: w is a packed K-chunk-major image (pack_weights_run): B tile (tap, chunk) =
                       //    rows [w_col0 + (tap*nchunks + chunk)*cout + n0, +BN) of a [rows][64] matrix,
                       //    one contiguous block; w_col0 = this segment's row base, w_ld = 64
};

// Pack a conv weight matrix W [cout][taps][cin_total] (OHWI) segment [off, off+cs) into the
// K-chunk-major image [taps][ceil(cs/64)][cout][64] (zero-padded channels).  Returns elements written.
size_t packed_elems(int cout, int taps, int cs);
dvc_status pack_weights_run(const void *W, dvc_dtype dt, int cout, int taps, int cin_total, int off, int cs, void *out,
                            cudaStream_t stream);

struct ConvDesc {
    ConvSeg seg[4];
    int nseg;
    int T, ho, wo, cout;
    const void *bias0, *bias1;   // [cout] or null
    const void *residual;        // [M][cout] or null
    void *out;                   // [M][cout]
    void *stats_out;             // per-channel box statistics of out (dvc_boxstats.cuh) or null
    dvc_dtype dt;
    // GEGLU epilogue (f1 feed-forward, TMA engine only): the weight rows come in blocks of 32 =
    // 16 "value" rows then the matching 16 "gate" rows; out is [M][cout/2] with
    // out = value * gelu(gate) (exact erf GELU); no residual, no statistics
    int geglu = 0;
    // fp8 operands (f4, TMA engine only): every segment's source and weights are E4M3 bytes; the
    // fp32 accumulator is multiplied by out_scale (the product of the two dequantisation scales)
    // before bias and the 16-bit (dt) store
    int fp8 = 0;
    float out_scale = 1.f;
    // up2 (TMA engine, staged epilogue): out is nearest_to(conv output, up_ho, up_wo) with up_ho in
    // {2 ho - 1, 2 ho} and up_wo in {2 wo - 1, 2 wo} -- exactly the 2x phase replication clipped at
    // the far edge (R11: floor(Y * ho / up_ho) = floor(Y / 2) for those sizes); no statistics
    int up2 = 0, up_ho = 0, up_wo = 0;
    long M() const { return (long)T * ho * wo; }
};

// Convolution with the GN-apply + SiLU (+ temporal shift) operand producer fused in
// (dvc_conv_fz.cu).  Segments read raw NHWC tensors through 10x18 halo boxes.
struct FzDesc {
    struct Seg {
        const void *src;   // raw operand tensor [T][H][W][c]
        int c, cglob0, taps, transform, shift;
        const void *w;
        int w_ld, col0, tapstride;
        int packed;   // as ConvSeg::packed
    };
    Seg seg[4];
    int nseg;
    int T, H, W, cout;
    int cs, cs_pad;              // shifted slice width; padded carry row length (multiple of 8)
    const void *carry_pad;       // [H][W][cs_pad] carry slice (16-byte rows) or null = zeros
    const void *coef;            // float2 [T][cop]: (scale, shift) of GN-apply (beta, mean folded)
    int cop;
    const void *bias0, *bias1, *residual;
    void *out, *stats_out;
    dvc_dtype dt;
    // up2: out is the nearest upsampling [T][up_ho][up_wo][cout] of the conv's output, up_ho in
    // {2H - 1, 2H}, up_wo in {2W - 1, 2W} (0: 2H / 2W) -- the epilogue's TMA store writes every staged
    // box four times with element stride 2, the far edge clipped by the tensor bounds; the low-res
    // output is never written; no statistics
    int up2 = 0, up_ho = 0, up_wo = 0;
};
dvc_status conv_fz_run(const FzDesc &d, cudaStream_t stream);
bool conv_fz_applicable(int H, int W, dvc_dtype dt);
// the VAE output head (dvc_conv_out.cu): out[T][H][W][oc] = conv3x3(SiLU(x * scale + shift)) + b over a
// 16-bit x [T][H][W][C] with coef float2 [T][C]; 16-bit, C in {16, 32, 48, 64}, oc <= 3
bool conv_out_applicable(int C, int oc, dvc_dtype dt);
dvc_status conv_out_run(const void *x, const void *coef, int T, int H, int W, int C, const void *w, const void *b,
                        int oc, void *out, dvc_dtype dt, cudaStream_t stream);

// spatial box of the TMA engine / box statistics for an H x W frame
void choose_box(int H, int W, int *BX, int *BY);
inline int boxes_per_frame(int H, int W) {
    int bx = 1, by = 1;
    choose_box(H, W, &bx, &by);
    return ((H + by - 1) / by) * ((W + bx - 1) / bx);
}
// standalone box statistics of a [T][H][W][C] tensor (same bits as the conv epilogue)
dvc_status box_stats_run(const void *x, int T, int H, int W, int C, dvc_dtype dt, float *stats, cudaStream_t stream);

// live per-launch event timing (dvc_profile_begin/end)
struct ProfSlot {
    int idx;   // -1 = not profiling
};
ProfSlot prof_begin(cudaStream_t stream);
struct ConvDesc;
void prof_end(ProfSlot s, cudaStream_t stream, double flops, const char *engine, const ConvDesc &d);
// non-conv kernel (not summed into the conv totals); flops: its algorithmic FLOPs, if any (attention)
void prof_end_aux(ProfSlot s, cudaStream_t stream, const char *label, double flops = 0.0);
double conv_flops(const ConvDesc &d);

// Validates the descriptor for the given engine; returns DVC_OK or an error.
dvc_status conv_check(const ConvDesc &d, bool tensor_core);
// Launches (no host sync).  16-bit: tcgen05 engine; F32: SIMT engine.
dvc_status conv_run(const ConvDesc &d, cudaStream_t stream);
// a1 + a2 fused (dvc_encode.cu): 5D-TMA unshuffle straight into the UMMA A layout + 1x1 expansion
bool encode_tma_applicable(dvc_dtype dt, int H, int W, int s, int c_lat);
dvc_status encode_tma_run(const void *frames, dvc_dtype frame_dt, int T, int H, int W, const void *w_exp,
                          const void *b_exp, int c_lat, void *latent, dvc_dtype dt, cudaStream_t stream);
dvc_status conv_tc_run(const ConvDesc &d, cudaStream_t stream);
dvc_status conv_simt_run(const ConvDesc &d, cudaStream_t stream);
dvc_status conv_ws_run(const ConvDesc &d, cudaStream_t stream);   // TMA + CTA-pair persistent engine
bool conv_ws_applicable(const ConvDesc &d);
inline bool conv_ws_applicable_dims(dvc_dtype dt) { extern int g_ws_cg; return g_ws_cg != 0 && dt != DVC_F32; }
extern int g_ws_cg;   // 2 (default): CTA pairs; 1: single CTA; 0: gather engine only

// Row-address helper shared by both engines: source pixel index of output
// pixel (t, y, x) for tap (dy, dx), or -1 when the tap falls in the zero padding.
__device__ __forceinline__ long seg_src_pixel(const ConvSeg &s, int ho, int wo, int t, int y, int x,
                                              int dy, int dx) {
    int iy, ix;
    if (s.mode == SEG_STRIDE2) {
        iy = 2 * y + dy;
        ix = 2 * x + dx;
    } else if (s.mode == SEG_UPNEAREST) {
        int uy = y + dy, ux = x + dx;
        if (uy < 0 || uy >= ho || ux < 0 || ux >= wo) return -1;
        iy = (int)(((long)uy * s.hi) / ho);
        ix = (int)(((long)ux * s.wi) / wo);
    } else {
        iy = y + dy;
        ix = x + dx;
    }
    if (iy < 0 || iy >= s.hi || ix < 0 || ix >= s.wi) return -1;
    return ((long)t * s.hi + iy) * s.wi + ix;
}


// N tile of a conv engine: the whole C_out if it fits one MMA (<= 256), else the largest divisor
// (multiple of `quantum`, half-tile a multiple of 8 rows for CTA pairs).  The TMA engine narrows it
// further only while a call fills less than half a wave (conv_ws_run): each narrower tile re-streams
// the whole A operand, which a blanket rule paid for (C5 at T = 4: 1032 -> 906 frames/s), but calls
// with a few dozen work items gain (T = 1 / 2 / 4: 375 -> 449 / 671 -> 767 / 1030 -> 1102 frames/s).
inline int choose_bn(int cout, int cg, int quantum) {
    for (int c = cout < 256 ? cout : 256; c >= 16; c -= 16)
        if (cout % c == 0 && c % quantum == 0 && (c / cg) % 8 == 0) return c;
    return 0;
}
}  // namespace dvc
