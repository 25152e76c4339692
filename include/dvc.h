/*
 * dvc.h -- C-ABI of libdvc.so, the B200-native (sm_100a) decode hot path of
 * DiffVC-RT (arXiv 2601.20564).
 *
 * Citations: P:<line> = the paper's text (/root/reference/PAPER.md at build
 * time), S:<line> = its CPU-program specification, R<n> = the
 * readings listed in DESIGN.md section 3 (the paper is silent there).
 *
 * Conventions (all entry points):
 *   - Every tensor pointer is a DEVICE pointer unless stated; the caller owns
 *     every buffer.  The library owns only the opaque handles it creates.
 *   - Activations are NHWC ("[T,h,w,C]", frames of one chain packed on the
 *     batch dimension), contiguous, 16-byte aligned.  Frames are NCHW.
 *     Conv weights are OHWI [C_out][k][k][C_in]; 1x1 weights [C_out][C_in].
 *   - dtype: DVC_BF16 (the paper's U-Net precision), DVC_F16, or DVC_F32
 *     (validation mode: fp32 storage, fp32 SIMT arithmetic, no tensor cores).
 *     In 16-bit modes all weights, biases and GN affine parameters are in the
 *     same 16-bit dtype; the tensor-core convolutions accumulate in fp32 (TMEM).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).  No
 *     entry point synchronises the host or allocates device memory on the
 *     forward path; calls are stream-ordered and asynchronous.
 *   - Argument, shape, divisibility and architecture errors are detected and
 *     returned BEFORE any launch: no partial writes.  Asynchronous CUDA faults
 *     surface as DVC_ERR_CUDA from a later call.  There is no CPU fallback:
 *     a device that is not sm_100 returns DVC_ERR_UNSUPPORTED.
 *   - dvc_last_error() returns a thread-local human-readable detail string.
 */
#ifndef DVC_H_
#define DVC_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DVC_API __attribute__((visibility("default")))
#else
#define DVC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DVC_ABI_VERSION 3

typedef enum {
    DVC_OK = 0,
    DVC_ERR_ARG = 1,          /* null pointer / bad enum / negative size            */
    DVC_ERR_DIVISIBILITY = 2, /* H%s, W%s, C%P, C%G                   */
    DVC_ERR_SHAPE = 3,        /* shape mismatch between arguments           */
    DVC_ERR_UNSUPPORTED = 4,  /* not sm_100, or a shape the kernels do not cover    */
    DVC_ERR_WORKSPACE = 5,    /* workspace too small                                */
    DVC_ERR_CUDA = 6,         /* a CUDA runtime error (including earlier async ones) */
    DVC_ERR_NCCL = 7          /* an NCCL error (multi-GPU halo)                     */
} dvc_status;

/* DVC_U8: 8-bit frames only (dvc_encode_pixelunshuffle's frame_dt), HWC layout, value u / 255 (R14) */
typedef enum { DVC_BF16 = 0, DVC_F16 = 1, DVC_F32 = 2, DVC_U8 = 3 } dvc_dtype;

DVC_API const char *dvc_status_string(dvc_status s);
DVC_API const char *dvc_last_error(void);
DVC_API int dvc_abi_version(void);

/* ------------------------------------------------------------------------
 * a1 + a2.  Encoder front end: PixelUnshuffle ("PixelUnshuffle
 * operation for space-to-depth") fused with the Latent Channel Expansion
 * ("expanding the latent dimension ... to 256"; 1x1 conv + bias, R13).
 *
 *   frames    frame_dt = DVC_BF16 / DVC_F16 / DVC_F32: [T,3,H,W] NCHW, values in [0,1];
 *             frame_dt = DVC_U8: [T,H,W,3] HWC bytes u, value RNE_{latent_dt}(u / 255) exactly rounded
 *             (reading R14; S:366 `to_latent` on decoded 8-bit frames)
 *   w_exp     [c_lat][3*s*s], b_exp [c_lat]  (latent_dt), or both NULL
 *   latent    [T,H/s,W/s,c_lat] NHWC in latent_dt (== frame_dt unless frame_dt is DVC_U8)
 *
 * w_exp == NULL: unshuffle only, c_lat must be 3*s*s; the result is a pure
 * permutation (of the converted bytes for DVC_U8), bit-exact:
 *   latent[t,y,x,c*s*s+i*s+j] = frames[t,c,s*y+i,s*x+j]   (torch channel order, R12).
 * Otherwise E = b + W.L with fp32 accumulation, computed on tcgen05 tensor cores (16-bit
 * latent_dt, s == 8; DVC_U8 frames also need W % 16 == 0) with the 3*s*s-channel latent never
 * written to memory; the fp32 validation mode runs the SIMT engine.
 * Errors: DIVISIBILITY if H%s or W%s; ARG on nulls / T<1 / bad dtypes; UNSUPPORTED for a
 * frame_dt != latent_dt pair other than DVC_U8 frames, or DVC_U8 latents.
 * ------------------------------------------------------------------------ */
DVC_API dvc_status dvc_encode_pixelunshuffle(const void *frames, dvc_dtype frame_dt, int T, int H, int W, int s,
                                     const void *w_exp, const void *b_exp, int c_lat,
                                     void *latent, dvc_dtype latent_dt, void *stream);

/* ------------------------------------------------------------------------
 * a3-a8.  One OTSM ResBlock over T consecutive frames of one chain (P:320,
 * App. A; P:151 Batch-dimension OTSM).  Input X = concat(x_a[c_a], x_b[c_b])
 * along channels (c_b = 0 except on the U-Net's up path).  Reading R2/R5:
 *
 *   Xs   = shift(X, carry_in)        frame t gets frame t-1's channels [0,C_in/P)
 *                                     (intra-batch); frame 0 gets carry_in
 *                                     (inter-batch)
 *   H1   = SiLU(GN1(Xs))             GN per (frame, group), biased var, eps (R3, R4)
 *   Y1   = conv3x3(H1) + b1          tensor cores (16-bit) / SIMT (F32)
 *   H2   = SiLU(GN2(Y1))
 *   Out  = S(X) + conv3x3(H2) + b2   S = identity if C_in == C_out, else a 1x1
 *                                     conv + bias on the UNSHIFTED X
 *   carry_out = X[T-1][..., 0:C_in/P]  (raw block input, for the next batch)
 *
 * Requirements: C_in = c_a + c_b; C_in % P == 0; C_in/P <= c_a; G | C_in and
 * G | C_out; c_a, c_b, C_out multiples of 16 on the tensor-core path (16-bit)
 * and of 8 in F32; T >= 1.
 * carry_in: [H,W,C_in/P] or NULL (= zeros: chain start, R8).
 * carry_out: [H,W,C_in/P] or NULL; may equal carry_in (in-place carry update: it is
 *            written after every read of carry_in), must not overlap it otherwise.
 * y: [T,H,W,C_out]; must not alias inputs.
 * workspace: device scratch of at least dvc_resblock_workspace_size() bytes,
 * 256-byte aligned.
 * ------------------------------------------------------------------------ */
typedef struct {
    int c_a, c_b, c_out, groups, shift_p;
    float eps;
    dvc_dtype dt;
    const void *gn1_w, *gn1_b, *conv1_w, *conv1_b; /* conv1_w [c_out][3][3][c_in] */
    const void *gn2_w, *gn2_b, *conv2_w, *conv2_b; /* conv2_w [c_out][3][3][c_out] */
    const void *sc_w, *sc_b;                       /* [c_out][c_in]; NULL iff c_in == c_out */
} dvc_resblock;

DVC_API dvc_status dvc_resblock_workspace_size(const dvc_resblock *b, int T, int H, int W, size_t *bytes);
DVC_API dvc_status dvc_resblock_tsm_forward(const dvc_resblock *b, const void *x_a, const void *x_b,
                                    int T, int H, int W, const void *carry_in, void *carry_out,
                                    void *y, void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Test-only: materialise Xs = shift(X, carry) (a3) with the same addressing
 * function the GN/SiLU operand producer uses.  xs [T,H,W,C_in] in dt.
 * ------------------------------------------------------------------------ */
DVC_API dvc_status dvc_debug_shift_gather(const void *x_a, const void *x_b, int c_a, int c_b, int shift_p,
                                  dvc_dtype dt, int T, int H, int W, const void *carry_in,
                                  void *xs, void *stream);

/* ------------------------------------------------------------------------
 * f1.  One self-attention Transformer2D block of the full U-Net (the
 * U-Net of SD-2.1 via AdcSR; 444.78 M parameters with these blocks;
 * readings R24-R27 in DESIGN.md): SD-2.1's Transformer2DModel with the text
 * cross-attention removed, frames independent (no temporal shift):
 *   a  = GN(x)             groups, eps_gn (1e-6), per frame, no SiLU
 *   h0 = a proj_in_w^T + proj_in_b                  ([C][C])
 *   q|k|v = LN1(h0) qkv_w^T                         ([3C][C], no bias)
 *   o  = per head j (channels [j*d,(j+1)*d)): softmax(q_j k_j^T / sqrt d) v_j
 *        over the H*W tokens of the frame (row-major y, x)
 *   h1 = o out_w^T + out_b + h0                     ([C][C])
 *   f  = LN2(h1) ff1_w^T + ff1_b                    ([8C][C]); g = f[:4C] * gelu(f[4C:])
 *   h2 = g ff2_w^T + ff2_b + h1                     ([C][4C])
 *   y  = h2 proj_out_w^T + proj_out_b + x           ([C][C])
 * LayerNorms: eps_ln (1e-5), per-channel affine.  gelu is the exact erf form.
 * x, y [T,H,W,C] NHWC device pointers in dt; y MAY alias x (in place).
 * Requirements: C % 16 == 0, C <= 1024, C % groups == 0, head_dim in
 * {16, 32, 48, 64} dividing C, 1 <= T < 256.  16-bit dt: tensor cores
 * (tcgen05) for the linear layers and the attention; DVC_F32: SIMT validation
 * path.  Errors return before any launch.
 * ------------------------------------------------------------------------ */
typedef struct {
    int c, groups, head_dim;
    float eps_gn, eps_ln;
    dvc_dtype dt;
    const void *gn_w, *gn_b, *proj_in_w, *proj_in_b, *ln1_w, *ln1_b, *qkv_w, *out_w, *out_b;
    const void *ln2_w, *ln2_b, *ff1_w, *ff1_b, *ff2_w, *ff2_b, *proj_out_w, *proj_out_b;
} dvc_transformer;

DVC_API dvc_status dvc_transformer_workspace_size(const dvc_transformer *b, int T, int H, int W, size_t *bytes);
DVC_API dvc_status dvc_transformer_forward(const dvc_transformer *b, const void *x, int T, int H, int W, void *y,
                                           void *workspace, size_t ws_bytes, void *stream);

/* The attention step alone: qkv [T,N,3C] (q | k | v channel blocks, head j at
 * channels [j*d,(j+1)*d) of each) -> out [T,N,C], softmax(q k^T / sqrt d) v per
 * frame and head.  workspace >= dvc_attention_workspace_size (the transposed V). */
DVC_API dvc_status dvc_attention_workspace_size(int T, int N, int C, dvc_dtype dt, size_t *bytes);
/* head_dim in {16, 32, 48, 64, 256} (256: the VAE decoder's single-head attention). */
DVC_API dvc_status dvc_attention_forward(const void *qkv, int T, int N, int C, int head_dim, dvc_dtype dt, void *out,
                                         void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * a9 + a10 + e.  The pruned U-Net's ResBlock skeleton over a group of frames
 * (reading R1):
 *   x0 = conv_in(concat(Lbar_t, Cm_t))                 (P:110, 512 -> width[0])
 *   levels 0..3: 2 OTSM ResBlocks each, a stride-2 3x3 conv after levels 0..2
 *   mid: 2 OTSM ResBlocks
 *   up levels 3..0: 3 OTSM ResBlocks on concat(h, skip) each, nearest resize to
 *   the next skip's size + 3x3 conv after the first three (R11)
 *   out = conv_out(SiLU(GN_out(h)))                    (width[0] -> c_lat)
 * head_dim == 0: the 16 self-attention Transformer2D blocks are elided
 * (identity; the ResBlock skeleton of SURVEY 8a).  head_dim > 0 (f1, the full
 * U-Net): a Transformer2D block (dvc_transformer, groups/eps_gn 1e-6/eps_ln
 * 1e-5) follows every ResBlock of down levels 0-2, mid.r0 and every ResBlock
 * of up levels 2-0 (R26); its 17 tensors (gn_w, gn_b, proj_in_w, proj_in_b,
 * ln1_w, ln1_b, qkv_w, out_w, out_b, ln2_w, ln2_b, ff1_w, ff1_b, ff2_w, ff2_b,
 * proj_out_w, proj_out_b) follow that ResBlock's in the blob.
 *
 * Weight blob (host memory, dt elements, concatenated in this order):
 *   conv_in{w [W0][3][3][c_lat+c_ctx], b}
 *   the 22 ResBlocks in U-Net order (down0.r0, down0.r1, ..., mid.r1, up0.r0 .. up3.r2),
 *     each {gn1_w, gn1_b, conv1_w, conv1_b, gn2_w, gn2_b, conv2_w, conv2_b[, sc_w, sc_b]},
 *     with the stride-2 conv {w, b} after down_l.r1 (l = 0..2) and the
 *     post-resize conv {w, b} after up_u.r2 (u = 0..2)
 *   gn_out{w, b}; conv_out{w [c_lat][3][3][W0], b}
 * Packed carries: the 22 slices [h_l][w_l][C_in_k/P] of block k's input,
 * concatenated in block order (dvc_unet_carry_size gives the element count).
 * ------------------------------------------------------------------------ */
typedef struct {
    int width[4];      /* 240, 480, 960, 960 (SD-2.1 widths x 0.75, R1) */
    int c_lat, c_ctx;  /* 256, 256 -> conv_in input 512 */
    int groups, shift_p;
    float eps;
    dvc_dtype dt;
    int h, w;          /* latent size, e.g. 90x160 (720p), 135x240 (1080p) */
    int max_T;         /* largest T_local per call; sizes the workspace */
    int head_dim;      /* 0 = skeleton (attention elided); 16/32/48/64 = full U-Net (48: R25) */
} dvc_unet_config;

typedef struct dvc_unet dvc_unet;
typedef struct dvc_comm dvc_comm;

DVC_API dvc_status dvc_unet_create(const dvc_unet_config *cfg, const void *host_weights, size_t bytes,
                           dvc_unet **out);
DVC_API dvc_status dvc_unet_destroy(dvc_unet *n);
/* Number of blob elements the config expects. */
DVC_API dvc_status dvc_unet_weight_count(const dvc_unet_config *cfg, size_t *elems);
/* Element count of the packed 22-slice carry. */
DVC_API dvc_status dvc_unet_carry_size(const dvc_unet *n, size_t *elems);
DVC_API dvc_status dvc_unet_workspace_size(const dvc_unet *n, int T_local, size_t *bytes);

/* One call decodes T_local consecutive frames [t0, t0+T_local) of one chain.
 *   lat, ctx  [T_local,h,w,c_lat] / [T_local,h,w,c_ctx]: Lbar_t and C^m_t
 *   out       [T_local,h,w,c_lat]: Lhat_t
 *   carry_in  packed carry of frame t0-1, or NULL = chain start (zeros, R8).
 *             With comm and rank > 0 the carry comes from rank-1 instead.
 *   carry_out packed carry of the last frame, or NULL.  With comm, only the
 *             last rank writes it.
 *   comm      NULL = single GPU; else the halo of every ResBlock moves from
 *             rank r to rank r+1 (contiguous frame chunks) over the
 *             communicator's transport (P2P peer copies or NCCL, see below). */
DVC_API dvc_status dvc_unet_decode_gop(dvc_unet *n, dvc_comm *comm, const void *lat, const void *ctx,
                               int T_local, const void *carry_in, void *carry_out, void *out,
                               void *workspace, size_t ws_bytes, void *stream);

/* The configuration a handle was created with (NULL for a NULL handle). */
DVC_API const dvc_unet_config *dvc_unet_get_config(const dvc_unet *n);

/* ------------------------------------------------------------------------
 * f3.  Asynchronous and Parallel Decoding Pipeline (Fig. APDP).
 * The in-loop Latent Compressor produces (Lbar_t, C^m_t) frame by frame on
 * the caller's stream; the out-of-loop Frame Reconstructor (the U-Net) runs
 * on the pipeline's own stream over batches of N frames taken from a FIFO of
 * `fifo_batches` slots, with the Batch-dimension OTSM carry passed from batch
 * to batch (Inter-batch Shift).  Latency is N-1 frames.
 *   push(lat_t, ctx_t): device pointers [h,w,c_lat] / [h,w,c_ctx] in the
 *     net's dtype, valid on `stream`; copied into the FIFO (stream-ordered,
 *     no host sync).  When N frames are buffered their decode is enqueued on
 *     the pipeline stream (after an event on `stream`).  DVC_ERR_ARG if all
 *     slots hold decoded batches nobody popped (pop first).
 *   pop(out, stream, &frames, &first): if the oldest batch is complete on the
 *     host's bookkeeping, enqueue (on `stream`, after the decode's event) the
 *     copy of its `frames` reconstructed latents into out [frames,h,w,c_lat]
 *     (or, with a VAE, the decoded frames [frames,8h,8w,out_ch])
 *     and return the index of its first frame; frames = 0 if none is ready.
 *   flush(): enqueue the decode of a partial last batch (T < N, R18).
 *   reset(): the next push starts a new chain (zero carry, R8/R9); flushes
 *     a partial batch first.
 * Frames t of one chain come out bit-identical to one dvc_unet_decode_gop
 * call over the whole chain (batch == online, P9).
 * ------------------------------------------------------------------------ */
typedef struct dvc_pipeline dvc_pipeline;
typedef struct dvc_vae dvc_vae;   /* f2, below */
/* vae: NULL = the pipeline outputs Lhat; else the VAE decoder (same h, w, c_lat, dt; max_T >= N)
 * runs after the U-Net on the pipeline stream and pop() returns frames [n, 8h, 8w, out_ch]. */
DVC_API dvc_status dvc_pipeline_create(dvc_unet *net, dvc_vae *vae, int batch_n, int fifo_batches,
                                       dvc_pipeline **out);
DVC_API dvc_status dvc_pipeline_destroy(dvc_pipeline *p);
DVC_API dvc_status dvc_pipeline_push(dvc_pipeline *p, const void *lat, const void *ctx, void *stream);
DVC_API dvc_status dvc_pipeline_pop(dvc_pipeline *p, void *out, void *stream, int *frames, long long *first_frame);
DVC_API dvc_status dvc_pipeline_flush(dvc_pipeline *p);
DVC_API dvc_status dvc_pipeline_reset(dvc_pipeline *p);

/* ------------------------------------------------------------------------
 * f2.  Pruned VAE Decoder ("Pruned VAE Decoder reduces intermediate
 * channels by 50%"; P:108 256-channel latent interface; Table 8 P:525;
 * readings R29-R31): SD-2.1's AutoencoderKL decoder with block widths x0.5.
 *   x = conv_in(Lhat)                  3x3, c_lat -> width[3], latent resolution
 *   mid: ResBlock, [single-head self-attention: x += out(softmax(q k^T/sqrt C) v),
 *        q|k|v|out linear + bias on GN(x)], ResBlock
 *   up level i = 0..3 (widths width[3], width[2], width[1], width[0]):
 *        3 ResBlocks (first maps the incoming width); i < 3: nearest 2x, 3x3 conv
 *   frames = conv_out(SiLU(GN_out(x)))  3x3, width[0] -> out_ch, 8x resolution
 * ResBlocks as dvc_resblock without the temporal shift; GroupNorm `groups`, `eps`
 * (SD: 32, 1e-6).  Frames independent.  Output NHWC [T, 8h, 8w, out_ch].
 * Weight blob (dt elements, in this order): conv_in{w [W3][3][3][c_lat], b};
 * mid.r0; [mid attention {gn_w, gn_b, q_w [W3][W3], q_b, k_w, k_b, v_w, v_b,
 * out_w, out_b}]; mid.r1; per up level 3 ResBlocks then (i < 3) the
 * post-upsample conv{w, b}; gn_out{w, b}; conv_out{w [out_ch][3][3][W0], b}.
 * Requirements: widths multiples of 16, groups dividing them, out_ch <= 16,
 * mid attention needs width[3] in {16,32,48,64,256}.
 * ------------------------------------------------------------------------ */
typedef struct {
    int width[4];      /* 64, 128, 256, 256 (SD-2.1 decoder x 0.5) */
    int c_lat;         /* 256 */
    int out_ch;        /* 3 */
    int groups;        /* 32 */
    float eps;         /* 1e-6 */
    int mid_attn;      /* 1: the mid-block self-attention; 0: elided */
    dvc_dtype dt;
    int h, w;          /* latent size; frames are 8h x 8w */
    int max_T;
} dvc_vae_config;
DVC_API dvc_status dvc_vae_weight_count(const dvc_vae_config *cfg, size_t *elems);
DVC_API dvc_status dvc_vae_create(const dvc_vae_config *cfg, const void *host_weights, size_t bytes, dvc_vae **out);
DVC_API dvc_status dvc_vae_destroy(dvc_vae *v);
DVC_API const dvc_vae_config *dvc_vae_get_config(const dvc_vae *v);
DVC_API dvc_status dvc_vae_workspace_size(const dvc_vae *v, int T, size_t *bytes);
DVC_API dvc_status dvc_vae_decode(dvc_vae *v, const void *lat, int T, void *frames, void *workspace, size_t ws_bytes,
                                  void *stream);

/* ------------------------------------------------------------------------
 * f4 variant: fp8 (E4M3) convolutions on the tensor cores (kind::f8f6f4).
 *   dvc_quantize_e4m3: q[i] = E4M3(RNE(x[i] / scale)), saturating to +-448 (fp32
 *     quotient); x in dt (n % 8 == 0, 16-byte aligned), q bytes.
 *   dvc_conv_fp8: y = (sx * sw) * conv(x8, w8) + bias with fp32 accumulation;
 *     x8 [T,H,W,cin] E4M3 NHWC, w8 [cout][taps][cin] E4M3 (OHWI, taps 9 = 3x3 pad 1,
 *     1 = 1x1), bias [cout] in out_dt or NULL, y [T,H,W,cout] in out_dt (bf16/fp16).
 *     cin % 32 == 0, cout % 16 == 0.  A variant of the decode's convolutions
 *     (SURVEY 8f rank 4), not used by dvc_unet_decode_gop.
 * ------------------------------------------------------------------------ */
/* One plain convolution y = conv(x, w) + bias in dt (the engines the decode uses; a building
 * block and the 16-bit reference point of dvc_conv_fp8): same layouts, dt in {bf16, fp16, f32}. */
DVC_API dvc_status dvc_conv(const void *x, const void *w, const void *bias, int T, int H, int W, int cin, int cout,
                            int taps, dvc_dtype dt, void *y, void *stream);
DVC_API dvc_status dvc_quantize_e4m3(const void *x, dvc_dtype dt, size_t n, float scale, void *q, void *stream);
DVC_API dvc_status dvc_conv_fp8(const void *x8, float sx, const void *w8, float sw, const void *bias, int T, int H,
                                int W, int cin, int cout, int taps, dvc_dtype out_dt, void *y, void *stream);

/* Multi-GPU halo communicators (row e: SURVEY 8e; "passes the partial channels of the last
 * sample ... to the subsequent batch").  Rank r of `world` decodes frames [t0_r, t0_r + T_local) of one
 * chain (contiguous chunks); before ResBlock k it sends the C_in/P-channel slice of its last frame's
 * block input to rank r+1 and receives rank r-1's slice as the carry of its first frame.  The send runs
 * on the communicator's own (high-priority) stream and overlaps block k; only the receive is on the
 * compute stream's critical path.  A communicator is bound to the device current at creation, is
 * single-owner, and every rank must make the same sequence of dvc_unet_decode_gop calls.
 *
 * P2P transport (the default of the Python binding): each rank owns a receive region (two epoch slots
 * of carry_bytes, arrival flags, acknowledgement words) allocated here.  The sender writes its slice
 * directly into the successor's slot with a copy-engine peer copy (NVLink; no SM, no staging) and
 * raises the successor's flag with a stream memory write; the receiver's stream waits on the flag
 * (cuStreamWaitValue32: the stream front end blocks, no kernel spins).  carry_bytes = carry elements
 * (dvc_unet_carry_size) x element size.  Connect every rank before its first decode:
 *   - ranks in different processes: exchange the 64-byte dvc_comm_ipc_handle of every rank (e.g.
 *     torch.distributed.all_gather_object) and call dvc_comm_connect_ipc(c, handle of rank+1 or NULL
 *     on the last rank, handle of rank-1 or NULL on rank 0);
 *   - ranks of one process (one GPU, the tests' loopback): dvc_comm_connect_local(c, next, prev).
 * Errors: DVC_ERR_ARG (wrong neighbours, already connected), DVC_ERR_CUDA (IPC / allocation),
 * DVC_ERR_UNSUPPORTED (no stream memory operations). */
DVC_API dvc_status dvc_comm_create_p2p(int rank, int world, size_t carry_bytes, dvc_comm **out);
DVC_API dvc_status dvc_comm_ipc_handle(const dvc_comm *c, void *handle64);
DVC_API dvc_status dvc_comm_connect_ipc(dvc_comm *c, const void *next_handle64, const void *prev_handle64);
DVC_API dvc_status dvc_comm_connect_local(dvc_comm *c, const dvc_comm *next, const dvc_comm *prev);
/* NCCL transport (loaded at run time from the process's libnccl.so.2): the slice is staged in the
 * decode workspace and moved by ncclSend/ncclRecv in one group on the comm stream.  id128: 128-byte
 * ncclUniqueId, created on rank 0 and broadcast by the caller (e.g. torch.distributed). */
DVC_API dvc_status dvc_comm_unique_id(void *id128);
DVC_API dvc_status dvc_comm_create(int rank, int world, const void *id128, dvc_comm **out);
DVC_API dvc_status dvc_comm_destroy(dvc_comm *c);

/* Live measurement of the dominant kernel (bench.py, roofline): between
 * dvc_profile_begin and dvc_profile_end every convolution launch (tcgen05 or
 * SIMT engine) is bracketed by CUDA events recorded on its launch stream.
 * dvc_profile_end waits for the last event and returns the summed kernel time
 * (ms), the summed algorithmic FLOPs (2*M*N*K over the real, unpadded K) and
 * the number of launches.  max_launches bounds the event pool. */
DVC_API dvc_status dvc_profile_begin(int max_launches);
DVC_API dvc_status dvc_profile_end(double *conv_ms, double *conv_flops, int *conv_launches);
/* Record i (0 <= i < dvc_profile_record_count()) of the last dvc_profile_end window: the
 * launch's event time (ms), its algorithmic FLOPs and a label "<engine> T=.. HxW K=.. N=.."
 * (engine: fz1/fz2 fused GN/SiLU/shift convs, ws persistent TMA conv, tc gather conv,
 * simt fp32).  Any output pointer may be null; label is truncated to label_cap bytes.
 * DVC_ERR_ARG if i is out of range. */
DVC_API dvc_status dvc_profile_record(int i, double *ms, double *flops, char *label, int label_cap);
/* Records kept by the last dvc_profile_end: the convolution launches plus the other
 * instrumented kernels of the path (GroupNorm coefficients / apply, box statistics, nearest,
 * encoder; label "<kernel> ...", flops 0).  dvc_profile_end's sums cover convolutions only. */
DVC_API int dvc_profile_record_count(void);

/* Convolution engine selection (tuning / A-B testing; default 2; experiment builds also read
 * DVC_CONV_ENGINE at load):
 *   2 = TMA-fed persistent tcgen05 engines with CTA pairs (cta_group::2, M=256): the fused
 *       GN/SiLU/shift engine for frames with H >= 32, the TMA engine otherwise and for raw
 *       operands -- including the stride-2 down-samplers (TMA boxes with element stride 2)
 *   1 = the TMA engine with single-CTA MMAs (M=128), no fused engine
 *   0 = gather-fed tcgen05 engine only (cp.async producer warps)
 * The gather engine also serves shapes the TMA engines do not take (the nearest-resize operand
 * of engine 0, the 16-bit expansion when the fused encoder does not apply). */
DVC_API dvc_status dvc_set_conv_engine(int engine);

/* Device / build introspection (no compute). */
DVC_API dvc_status dvc_device_check(int device);   /* DVC_OK iff the device is sm_100 */
DVC_API int dvc_kernel_launch_count(void);         /* kernels launched by this process so far */

#ifdef __cplusplus
}
#endif
#endif /* DVC_H_ */
