/*
 * dvc_oracle.c -- fp64 CPU oracle for the DiffVC-RT decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2601_20564_b200/csrc); neither side includes or links the other.
 *
 * Every routine is the plain textbook definition, written as direct loops in
 * fp64, in the order the definition states; nothing is blocked, fused or
 * reordered.  Citations: P:<line> = /root/reference/PAPER.md, S:<line> =
 * /root/reference/SPEC.md, R<n> = the readings listed in DESIGN.md §3.
 *
 * Layouts: frames NCHW [T][C][H][W]; activations NHWC [T][H][W][C];
 * conv weights OHWI [Cout][k][k][Cin].
 *
 * Pins (see tests/test_oracle_pins.py): unshuffle shape / s=1 / round trip /
 * torch.pixel_unshuffle; conv identity / all-ones 9-6-4 / brute
 * force / F.conv2d; group-norm constant group -> beta, two-value
 * closed form, F.group_norm; silu(0)=0; rounding 65520 -> inf (fp16),
 * pi -> 3.140625 (bf16) and exhaustive agreement with numpy's
 * correctly rounded binary16 conversion.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define IDX4(a, b, c, d, B, C, D) ((((size_t)(a) * (B) + (b)) * (C) + (c)) * (D) + (d))

/* ---------------------------------------------------------------------------
 * PixelUnshuffle ("PixelUnshuffle operation for space-to-depth";
 * S:53-61).  Channel order follows torch.nn.PixelUnshuffle (reading R12):
 *   L[t, y, x, c*s*s + i*s + j] = F[t, c, s*y + i, s*x + j].
 * Returns 0 on success, 2 on a divisibility error.
 * ------------------------------------------------------------------------- */
int orc_unshuffle(const double *F, int T, int C, int H, int W, int s, double *L)
{
    if (s < 1 || H % s || W % s) return 2;
    int h = H / s, w = W / s, CL = C * s * s;
    for (int t = 0; t < T; ++t)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                for (int c = 0; c < C; ++c)
                    for (int i = 0; i < s; ++i)
                        for (int j = 0; j < s; ++j)
                            L[IDX4(t, y, x, c * s * s + i * s + j, h, w, CL)] =
                                F[IDX4(t, c, s * y + i, s * x + j, C, H, W)];
    return 0;
}

/* PixelShuffle, the exact inverse: F[t,c,s*y+i,s*x+j] = L[t,y,x,c*s*s+i*s+j].
 * C = number of frame channels; L has C*s*s channels. */
int orc_shuffle(const double *L, int T, int C, int h, int w, int s, double *F)
{
    if (s < 1) return 2;
    int H = h * s, W = w * s, CL = C * s * s;
    for (int t = 0; t < T; ++t)
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < s; ++i)
                for (int j = 0; j < s; ++j)
                    for (int y = 0; y < h; ++y)
                        for (int x = 0; x < w; ++x)
                            F[IDX4(t, c, s * y + i, s * x + j, C, H, W)] =
                                L[IDX4(t, y, x, c * s * s + i * s + j, h, w, CL)];
    return 0;
}

/* ---------------------------------------------------------------------------
 * conv2d: direct cross-correlation with zero padding.
 *   Y[t,oy,ox,o] = b[o] + sum_{ky,kx} sum_c W[o,ky,kx,c] * X[t, oy*st-pad+ky, ox*st-pad+kx, c]
 * with X = 0 outside the frame.  Ho = (H + 2 pad - k)/st + 1.  The sum runs
 * over taps (ky, kx) in order, then channels c in order.  b may be NULL.
 * Parallel over output pixels only (each output's sum order is fixed).
 * ------------------------------------------------------------------------- */
void orc_conv2d(const double *X, int T, int H, int W, int Cin,
                const double *Wt, const double *b, int Cout,
                int k, int st, int pad, double *Y)
{
    int Ho = (H + 2 * pad - k) / st + 1, Wo = (W + 2 * pad - k) / st + 1;
    long npix = (long)T * Ho * Wo;
#pragma omp parallel for schedule(dynamic, 4)
    for (long p = 0; p < npix; ++p) {
        int t = (int)(p / ((long)Ho * Wo));
        int oy = (int)((p / Wo) % Ho);
        int ox = (int)(p % Wo);
        double *out = Y + (size_t)p * Cout;
        for (int o = 0; o < Cout; ++o) {
            double acc = b ? b[o] : 0.0;
            for (int ky = 0; ky < k; ++ky) {
                int iy = oy * st - pad + ky;
                if (iy < 0 || iy >= H) continue;
                for (int kx = 0; kx < k; ++kx) {
                    int ix = ox * st - pad + kx;
                    if (ix < 0 || ix >= W) continue;
                    const double *xp = X + IDX4(t, iy, ix, 0, H, W, Cin);
                    const double *wp = Wt + IDX4(o, ky, kx, 0, k, k, Cin);
                    for (int c = 0; c < Cin; ++c) acc += wp[c] * xp[c];
                }
            }
            out[o] = acc;
        }
    }
}

/* ---------------------------------------------------------------------------
 * GroupNorm per (frame, group) (SD ResBlock; readings R3, R4):
 *   mu = (1/n) sum x,   var = (1/n) sum (x - mu)^2   (biased, two-pass),
 *   Y = (x - mu) / sqrt(var + eps) * gamma[c] + beta[c],
 * n = (C/G) * HW, groups are contiguous channel ranges [g*C/G, (g+1)*C/G).
 * Returns 2 if G does not divide C.
 * ------------------------------------------------------------------------- */
int orc_groupnorm(const double *X, int T, int HW, int C, int G,
                  const double *gamma, const double *beta, double eps, double *Y)
{
    if (G < 1 || C % G) return 2;
    int cg = C / G;
    double n = (double)cg * HW;
#pragma omp parallel for collapse(2)
    for (int t = 0; t < T; ++t)
        for (int g = 0; g < G; ++g) {
            const double *xt = X + (size_t)t * HW * C;
            double *yt = Y + (size_t)t * HW * C;
            double s = 0.0;
            for (int p = 0; p < HW; ++p)
                for (int c = g * cg; c < (g + 1) * cg; ++c) s += xt[(size_t)p * C + c];
            double mu = s / n;
            double v = 0.0;
            for (int p = 0; p < HW; ++p)
                for (int c = g * cg; c < (g + 1) * cg; ++c) {
                    double d = xt[(size_t)p * C + c] - mu;
                    v += d * d;
                }
            double var = v / n;
            double inv = 1.0 / sqrt(var + eps);
            for (int p = 0; p < HW; ++p)
                for (int c = g * cg; c < (g + 1) * cg; ++c)
                    yt[(size_t)p * C + c] = (xt[(size_t)p * C + c] - mu) * inv * gamma[c] + beta[c];
        }
    return 0;
}

/* SiLU(z) = z / (1 + exp(-z))  (SD activation). */
void orc_silu(const double *X, size_t n, double *Y)
{
    for (size_t i = 0; i < n; ++i) Y[i] = X[i] / (1.0 + exp(-X[i]));
}

/* ---------------------------------------------------------------------------
 * Nearest resize to an explicit size (reading R11):
 *   U[t,y,x,c] = V[t, floor(y*H/Ho), floor(x*W/Wo), c]   in exact integer arithmetic.
 * ------------------------------------------------------------------------- */
void orc_nearest_to(const double *V, int T, int H, int W, int C, int Ho, int Wo, double *U)
{
    for (int t = 0; t < T; ++t)
        for (int y = 0; y < Ho; ++y)
            for (int x = 0; x < Wo; ++x) {
                int sy = (int)(((long)y * H) / Ho), sx = (int)(((long)x * W) / Wo);
                for (int c = 0; c < C; ++c)
                    U[IDX4(t, y, x, c, Ho, Wo, C)] = V[IDX4(t, sy, sx, c, H, W, C)];
            }
}

/* ---------------------------------------------------------------------------
 * Round-to-nearest-even from fp64 directly to a 16-bit format (reading R15;
 * S:36-43 round_to_precision).  mode 0: identity, 1: IEEE binary16,
 * 2: bfloat16.  Direct from the exact double, never through fp32.
 *   binary16: 11-bit significand, emin = -14, max finite 65504.
 *   bfloat16: 8-bit significand,  emin = -126, max finite (2 - 2^-7) 2^127.
 * Overflow: |x| at or above (max + half ulp) rounds to +-inf (ties-to-even
 * goes to the odd->even neighbour, which is the overflow value).
 * ------------------------------------------------------------------------- */
double orc_round1(double x, int mode)
{
    if (mode == 0 || isnan(x) || isinf(x) || x == 0.0) return x;
    int p, emin;
    double ovf;
    if (mode == 1) { p = 11; emin = -14; ovf = 65520.0; }
    else { p = 8; emin = -126; ovf = ldexp(2.0 - ldexp(1.0, -8), 127); }
    double a = fabs(x);
    if (a >= ovf) return copysign(INFINITY, x);
    int e2;
    frexp(a, &e2);            /* a = m 2^e2, m in [0.5, 1)  =>  floor(log2 a) = e2 - 1 */
    int e = e2 - 1;
    if (e < emin) e = emin;   /* subnormal range keeps the emin quantum */
    double q = ldexp(a, -(e - (p - 1)));  /* exact: a / ulp */
    double r = nearbyint(q);              /* default rounding mode: ties to even */
    return copysign(ldexp(r, e - (p - 1)), x);
}

void orc_round(double *x, size_t n, int mode)
{
    if (mode == 0) return;
    for (size_t i = 0; i < n; ++i) x[i] = orc_round1(x[i], mode);
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
