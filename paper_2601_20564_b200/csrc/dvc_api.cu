// dvc_api.cu -- C-ABI entry points (include/dvc.h): argument validation,
// workspace carving and launch order.  No host sync and no allocation on the
// forward path; every check happens before the first launch.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>
#include <string>
#include <mutex>
#include <map>
#include <tuple>
#include <nvtx3/nvToolsExt.h>
#include "dvc_conv.cuh"
#include "dvc_norm.cuh"
#include "dvc_resblock.cuh"

namespace dvc {

int g_launches = 0;
static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Raise a kernel's dynamic shared memory limit once per (kernel, device, size): the cache records a
// size only after cudaFuncSetAttribute succeeded, so a failed call is retried (and reported) next time.
NvtxRange::NvtxRange(const char *fmt, ...) {
    char name[96];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(name, sizeof(name), fmt, ap);
    va_end(ap);
    nvtxRangePushA(name);
}
NvtxRange::~NvtxRange() { nvtxRangePop(); }

dvc_status ensure_smem(const void *kern, int smem) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static const void *keys[64];
    static int vals[64];
    static int n = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const void *key = reinterpret_cast<const char *>(kern) + dev;   // per device
    int i = 0;
    while (i < n && keys[i] != key) ++i;
    if (i < n && vals[i] >= smem) return DVC_OK;
    DVC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (i < n) vals[i] = smem;
    else if (n < 64) keys[n] = key, vals[n++] = smem;
    return DVC_OK;
}

bool pdl_enabled() {
    static const bool on = !(dvc_knob("DVC_PDL") && atoi(dvc_knob("DVC_PDL")) == 0);
    return on;
}

dvc_status check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return DVC_ERR_CUDA;
    }
    return DVC_OK;
}

dvc_status check_device() {
    int dev = 0;
    DVC_CUDA(cudaGetDevice(&dev));
    static int cached[64];   // 0 unknown, 1 ok, 2 bad
    if (dev >= 0 && dev < 64 && cached[dev] == 1) return DVC_OK;
    cudaDeviceProp prop;
    DVC_CUDA(cudaGetDeviceProperties(&prop, dev));
    bool ok = prop.major == 10 && prop.minor == 0;
    if (dev >= 0 && dev < 64) cached[dev] = ok ? 1 : 2;
    DVC_CHECK_ARG(ok, DVC_ERR_UNSUPPORTED, "device %d is sm_%d%d; libdvc is built for sm_100a only (no fallback)",
                  dev, prop.major, prop.minor);
    // surface earlier asynchronous faults
    cudaError_t e = cudaPeekAtLastError();
    DVC_CHECK_ARG(e == cudaSuccess, DVC_ERR_CUDA, "pending CUDA error: %s", cudaGetErrorString(e));
    return DVC_OK;
}

// ----------------------------------------------------------------- live profiling
namespace {
struct Prof {
    bool on = false;
    int cap = 0, used = 0;
    std::vector<cudaEvent_t> ev;   // 2 per launch
    std::vector<double> flops, ms;
    std::vector<char> conv;   // 1: convolution launch (summed by dvc_profile_end); 0: other kernel
    std::vector<std::string> label;
    int done = 0;   // records kept by dvc_profile_end for dvc_profile_record
} g_prof;
}  // namespace

ProfSlot prof_begin(cudaStream_t stream) {
    if (!g_prof.on || g_prof.used >= g_prof.cap) return ProfSlot{-1};
    int i = g_prof.used++;
    cudaEventRecord(g_prof.ev[2 * i], stream);
    return ProfSlot{i};
}

void prof_end(ProfSlot s, cudaStream_t stream, double flops, const char *engine, const ConvDesc &d) {
    if (s.idx < 0) return;
    cudaEventRecord(g_prof.ev[2 * s.idx + 1], stream);
    g_prof.flops[s.idx] = flops;
    g_prof.conv[s.idx] = 1;
    char buf[128];
    int k = 0;
    for (int i = 0; i < d.nseg; ++i) k += d.seg[i].taps * d.seg[i].c_src;
    snprintf(buf, sizeof(buf), "%s T=%d %dx%d K=%d N=%d segs=%d", engine, d.T, d.ho, d.wo, k, d.cout, d.nseg);
    g_prof.label[s.idx] = buf;
}

void prof_end_aux(ProfSlot s, cudaStream_t stream, const char *label, double flops) {
    if (s.idx < 0) return;
    cudaEventRecord(g_prof.ev[2 * s.idx + 1], stream);
    g_prof.flops[s.idx] = flops;
    g_prof.conv[s.idx] = 0;
    g_prof.label[s.idx] = label;
}

// ----------------------------------------------------------------- identity weights
// [c][c] identity in dt, one per (device, c, dt), allocated on first use and kept for the
// process lifetime (the fused conv's identity-skip segment).  First use synchronises
// (cudaMalloc / cudaMemcpy): not inside stream capture.
static const void *identity_weights(int c, dvc_dtype dt) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, void *> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, c, (int)dt);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<uint16_t> h((size_t)c * c, 0);
    const uint16_t one = dt == DVC_BF16 ? 0x3F80 : 0x3C00;
    for (int i = 0; i < c; ++i) h[(size_t)i * c + i] = one;
    void *d = nullptr;
    if (cudaMalloc(&d, h.size() * 2) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    cache[key] = d;
    return d;
}

// ----------------------------------------------------------------- ResBlock (a3-a8)
static bool box_mode(const RB &b) {
    const int cin = b.ca + b.cb, cs = b.P > 0 ? cin / b.P : 0, cg = cin / b.G;
    return cs % cg == 0;   // the shifted slice is whole GN groups: statistics from box partials
}

size_t resblock_ws_bytes(int ca, int cb, int cout, int G, int T, int H, int W, dvc_dtype dt) {
    const size_t es = dt_size(dt);
    const int cin = ca + cb, HW = H * W;
    return align256(gn_workspace_bytes(T, HW, G, cin > cout ? cin : cout)) + align256((size_t)T * HW * cin * es) +
           2 * align256((size_t)T * HW * cout * es) + box_stats_bytes(T, H, W, ca) + box_stats_bytes(T, H, W, cb) +
           box_stats_bytes(1, H, W, cin) + box_stats_bytes(T, H, W, cout) + 4 * 256;
}

dvc_status resblock_validate(const RB &b, int T, int H, int W) {
    const int cin = b.ca + b.cb;
    DVC_CHECK_ARG(dt_valid(b.dt), DVC_ERR_ARG, "bad dtype");
    DVC_CHECK_ARG(T >= 1 && H >= 1 && W >= 1, DVC_ERR_ARG, "T, H, W must be >= 1");
    DVC_CHECK_ARG(b.ca > 0 && b.cb >= 0 && b.cout > 0, DVC_ERR_ARG, "bad channel counts");
    // P = 0: no temporal shift (the VAE decoder's ResBlocks, f2)
    DVC_CHECK_ARG(b.P == 0 || (b.P >= 1 && cin % b.P == 0), DVC_ERR_DIVISIBILITY, "shift_p=%d must divide C_in=%d", b.P,
                  cin);
    DVC_CHECK_ARG(b.G >= 1 && cin % b.G == 0 && b.cout % b.G == 0, DVC_ERR_DIVISIBILITY,
                  "groups=%d must divide C_in=%d and C_out=%d", b.G, cin, b.cout);
    DVC_CHECK_ARG(b.P == 0 || cin / b.P <= b.ca, DVC_ERR_UNSUPPORTED, "shift slice C_in/P must lie in x_a");
    DVC_CHECK_ARG(b.gn1_w && b.gn1_b && b.conv1_w && b.conv1_b && b.gn2_w && b.gn2_b && b.conv2_w && b.conv2_b,
                  DVC_ERR_ARG, "null ResBlock parameter");
    DVC_CHECK_ARG((b.sc_w == nullptr) == (cin == b.cout), DVC_ERR_SHAPE,
                  "sc_w must be given iff C_in != C_out (C_in=%d, C_out=%d)", cin, b.cout);
    DVC_CHECK_ARG(b.sc_w == nullptr || b.sc_b != nullptr, DVC_ERR_ARG, "sc_b missing");
    DVC_CHECK_ARG(b.sc_w != nullptr || b.cb == 0, DVC_ERR_UNSUPPORTED, "identity shortcut needs one source");
    const int q = b.dt == DVC_F32 ? 8 : 16;
    DVC_CHECK_ARG(b.ca % q == 0 && b.cb % q == 0 && b.cout % q == 0, DVC_ERR_UNSUPPORTED,
                  "channel counts must be multiples of %d", q);
    DVC_CHECK_ARG(cin <= 2048 && b.cout <= 2048, DVC_ERR_UNSUPPORTED, "at most 2048 channels");
    DVC_CHECK_ARG(T < 256 && H < 4096 && W < 4096, DVC_ERR_UNSUPPORTED, "T < 256, H, W < 4096");
    return DVC_OK;
}

// The block as a launch sequence.  ws holds GN scratch, H1 [T][HW][C_in], Y1 and H2
// [T][HW][C_out] and the box statistics.  stats_a / stats_b: box statistics of x_a /
// x_b if the caller has them (produced by the previous conv's epilogue), else they
// are computed here; stats_y: where to put the box statistics of y (or null).
static dvc_status resblock_body(const RB &b, const void *xa, const void *xb, int T, int H, int W,
                                const void *carry_in, void *y, void *ws, cudaStream_t stream, const void *stats_a,
                                const void *stats_b, void *stats_y, int up2, int up_ho, int up_wo) {
    const int HW = H * W, cin = b.ca + b.cb, cs = b.P > 0 ? cin / b.P : 0;
    if (up2) {
        up_ho = up_ho ? up_ho : 2 * H;
        up_wo = up_wo ? up_wo : 2 * W;
        DVC_CHECK_ARG((up_ho == 2 * H || up_ho == 2 * H - 1) && (up_wo == 2 * W || up_wo == 2 * W - 1), DVC_ERR_UNSUPPORTED,
                      "resblock: upsampled output must be 2H (- 1) x 2W (- 1)");
    }
    if (cs == 0) carry_in = nullptr;   // no shift: no carry
    const size_t es = dt_size(b.dt);
    uint8_t *p = reinterpret_cast<uint8_t *>(ws);
    void *gnws = p;
    p += align256(gn_workspace_bytes(T, HW, b.G, cin > b.cout ? cin : b.cout));
    void *h1 = p;
    p += align256((size_t)T * HW * cin * es);
    void *y1 = p;
    p += align256((size_t)T * HW * b.cout * es);
    void *h2 = p;
    p += align256((size_t)T * HW * b.cout * es);
    void *st_a = p;
    p += box_stats_bytes(T, H, W, b.ca);
    void *st_b = p;
    p += box_stats_bytes(T, H, W, b.cb);
    void *st_k = p;
    p += box_stats_bytes(1, H, W, cin);
    void *st_y1 = p;
    dvc_status st;
    const bool boxed = box_mode(b);
    if (boxed && conv_fz_applicable(H, W, b.dt)) {
        // ---- fused path: GN statistics from box partials, GN-apply + SiLU + shift inside the convs
        if (!stats_a) {
            if ((st = box_stats_run(xa, T, H, W, b.ca, b.dt, reinterpret_cast<float *>(st_a), stream)) != DVC_OK)
                return st;
            stats_a = st_a;
        }
        if (b.cb > 0 && !stats_b) {
            if ((st = box_stats_run(xb, T, H, W, b.cb, b.dt, reinterpret_cast<float *>(st_b), stream)) != DVC_OK)
                return st;
            stats_b = st_b;
        }
        const void *stats_k = nullptr;
        void *carry_pad = nullptr;
        const int cs_pad = (cs + 7) & ~7;
        if (carry_in) {
            if ((st = box_stats_run(carry_in, 1, H, W, cs, b.dt, reinterpret_cast<float *>(st_k), stream)) != DVC_OK)
                return st;
            stats_k = st_k;
            carry_pad = h1;   // [HW][cs_pad]: 16-byte rows for the TMA halo map (h1 is not used on this path)
            if (cs_pad != cs) DVC_CUDA(cudaMemsetAsync(carry_pad, 0, (size_t)HW * cs_pad * es, stream));
            DVC_CUDA(cudaMemcpy2DAsync(carry_pad, cs_pad * es, carry_in, cs * es, cs * es, HW,
                                       cudaMemcpyDeviceToDevice, stream));
        }
        void *coef = gnws;
        NormArgs n1{xa, xb, carry_in, b.ca, b.cb, cs, T, HW, b.G, b.eps, b.gn1_w, b.gn1_b, coef, nullptr};
        if ((st = gn_coef_box_run(n1, BoxStatsIn{stats_a, b.cb > 0 ? stats_b : nullptr, stats_k}, H, W, b.dt,
                                  stream)) != DVC_OK)
            return st;
        FzDesc f1{};
        if (b.conv1_pk) {
            const int rows_a = 9 * ((b.ca + 63) / 64) * b.cout;
            f1.seg[0] = FzDesc::Seg{xa, b.ca, 0, 9, 1, cs > 0 ? 1 : 0, b.conv1_pk, 64, 0, 0, 1};
            f1.nseg = 1;
            if (b.cb > 0) f1.seg[f1.nseg++] = FzDesc::Seg{xb, b.cb, b.ca, 9, 1, 0, b.conv1_pk, 64, rows_a, 0, 1};
        } else {
            f1.seg[0] = FzDesc::Seg{xa, b.ca, 0, 9, 1, cs > 0 ? 1 : 0, b.conv1_w, 9 * cin, 0, cin, 0};
            f1.nseg = 1;
            if (b.cb > 0) f1.seg[f1.nseg++] = FzDesc::Seg{xb, b.cb, b.ca, 9, 1, 0, b.conv1_w, 9 * cin, b.ca, cin, 0};
        }
        f1.T = T;
        f1.H = H;
        f1.W = W;
        f1.cout = b.cout;
        f1.cs = cs;
        f1.cs_pad = cs_pad;
        f1.carry_pad = carry_pad;
        f1.coef = coef;
        f1.cop = cin;
        f1.bias0 = b.conv1_b;
        f1.out = y1;
        f1.stats_out = st_y1;
        f1.dt = b.dt;
        {
            ConvDesc prof{};
            prof.seg[0] = ConvSeg{xa, cin, SEG_SAME, H, W, 9, b.conv1_w, 9 * cin, 0, cin};
            prof.nseg = 1, prof.T = T, prof.ho = H, prof.wo = W, prof.cout = b.cout;
            ProfSlot slot = prof_begin(stream);
            st = conv_fz_run(f1, stream);
            prof_end(slot, stream, conv_flops(prof), "fz1", prof);
            if (st != DVC_OK) return st;
        }
        NormArgs n2{y1, nullptr, nullptr, b.cout, 0, 0, T, HW, b.G, b.eps, b.gn2_w, b.gn2_b, coef, nullptr};
        if ((st = gn_coef_box_run(n2, BoxStatsIn{st_y1, nullptr, nullptr}, H, W, b.dt, stream)) != DVC_OK) return st;
        FzDesc f2{};
        if (b.conv2_pk) f2.seg[0] = FzDesc::Seg{y1, b.cout, 0, 9, 1, 0, b.conv2_pk, 64, 0, 0, 1};
        else f2.seg[0] = FzDesc::Seg{y1, b.cout, 0, 9, 1, 0, b.conv2_w, 9 * b.cout, 0, b.cout, 0};
        f2.nseg = 1;
        if (b.sc_w) {
            if (b.sc_pk) {
                const int rows_a = ((b.ca + 63) / 64) * b.cout;
                f2.seg[f2.nseg++] = FzDesc::Seg{xa, b.ca, 0, 1, 0, 0, b.sc_pk, 64, 0, 0, 1};
                if (b.cb > 0) f2.seg[f2.nseg++] = FzDesc::Seg{xb, b.cb, 0, 1, 0, 0, b.sc_pk, 64, rows_a, 0, 1};
            } else {
                f2.seg[f2.nseg++] = FzDesc::Seg{xa, b.ca, 0, 1, 0, 0, b.sc_w, cin, 0, 0, 0};
                if (b.cb > 0) f2.seg[f2.nseg++] = FzDesc::Seg{xb, b.cb, 0, 1, 0, 0, b.sc_w, cin, b.ca, 0, 0};
            }
            f2.bias1 = b.sc_b;
        } else {
            // identity skip (C_in == C_out): X . I as a 1x1 raw segment -- the tensor core adds the
            // residual into the fp32 accumulator (exact products), no residual tile in the epilogue
            DVC_CHECK_ARG(b.cb == 0 && b.ca == b.cout, DVC_ERR_UNSUPPORTED, "identity skip needs C_in == C_out");
            const void *eye = identity_weights(b.cout, b.dt);
            DVC_CHECK_ARG(eye != nullptr, DVC_ERR_CUDA, "identity weights: %s", "allocation failed");
            f2.seg[f2.nseg++] = FzDesc::Seg{xa, b.ca, 0, 1, 0, 0, eye, b.cout, 0, 0, 0};
        }
        f2.T = T;
        f2.H = H;
        f2.W = W;
        f2.cout = b.cout;
        f2.coef = coef;
        f2.cop = b.cout;
        f2.bias0 = b.conv2_b;
        f2.out = y;
        f2.stats_out = up2 ? nullptr : stats_y;
        f2.up2 = up2;
        f2.up_ho = up_ho;
        f2.up_wo = up_wo;
        f2.dt = b.dt;
        ConvDesc prof{};
        prof.seg[0] = ConvSeg{y1, b.cout, SEG_SAME, H, W, 9, b.conv2_w, 9 * b.cout, 0, b.cout};
        prof.nseg = 1, prof.T = T, prof.ho = H, prof.wo = W, prof.cout = b.cout;
        if (b.sc_w) prof.seg[prof.nseg++] = ConvSeg{xa, cin, SEG_SAME, H, W, 1, b.sc_w, cin, 0, 0};
        ProfSlot slot = prof_begin(stream);
        st = conv_fz_run(f2, stream);
        prof_end(slot, stream, conv_flops(prof), "fz2", prof);
        return st;
    }
    // a3 + a4: H1 = SiLU(GN1(shift(X, carry)))
    NormArgs n1{xa, xb, carry_in, b.ca, b.cb, cs, T, HW, b.G, b.eps, b.gn1_w, b.gn1_b, h1, gnws};
    if (boxed) {
        if (!stats_a) {
            if ((st = box_stats_run(xa, T, H, W, b.ca, b.dt, reinterpret_cast<float *>(st_a), stream)) != DVC_OK)
                return st;
            stats_a = st_a;
        }
        if (b.cb > 0 && !stats_b) {
            if ((st = box_stats_run(xb, T, H, W, b.cb, b.dt, reinterpret_cast<float *>(st_b), stream)) != DVC_OK)
                return st;
            stats_b = st_b;
        }
        const void *stats_k = nullptr;
        if (carry_in) {
            if ((st = box_stats_run(carry_in, 1, H, W, cs, b.dt, reinterpret_cast<float *>(st_k), stream)) != DVC_OK)
                return st;
            stats_k = st_k;
        }
        st = gn_silu_box_run(n1, BoxStatsIn{stats_a, b.cb > 0 ? stats_b : nullptr, stats_k}, H, W, b.dt, stream);
    } else {
        st = gn_silu_run(n1, b.dt, stream);
    }
    if (st != DVC_OK) return st;
    // a5: Y1 = conv3x3(H1) + b1   (+ box statistics of Y1 from the epilogue)
    ConvDesc c1{};
    const bool pk = b.dt != DVC_F32 && conv_ws_applicable_dims(b.dt);
    if (pk && b.conv1_pk && b.cb == 0) c1.seg[0] = ConvSeg{h1, cin, SEG_SAME, H, W, 9, b.conv1_pk, 64, 0, 0, 1};
    else c1.seg[0] = ConvSeg{h1, cin, SEG_SAME, H, W, 9, b.conv1_w, 9 * cin, 0, cin};
    c1.nseg = 1;
    c1.T = T;
    c1.ho = H;
    c1.wo = W;
    c1.cout = b.cout;
    c1.bias0 = b.conv1_b;
    c1.out = y1;
    c1.stats_out = boxed ? st_y1 : nullptr;
    c1.dt = b.dt;
    if ((st = conv_run(c1, stream)) != DVC_OK) return st;
    // a6: H2 = SiLU(GN2(Y1))
    NormArgs n2{y1, nullptr, nullptr, b.cout, 0, 0, T, HW, b.G, b.eps, b.gn2_w, b.gn2_b, h2, gnws};
    st = boxed ? gn_silu_box_run(n2, BoxStatsIn{st_y1, nullptr, nullptr}, H, W, b.dt, stream)
               : gn_silu_run(n2, b.dt, stream);
    if (st != DVC_OK) return st;
    // a7 + a8: Out = S(X) + conv3x3(H2) + b2; the 1x1 shortcut on the UNSHIFTED X is
    // extra K segments of the same GEMM (same fp32 accumulator), identity = epilogue add.
    ConvDesc c2{};
    if (pk && b.conv2_pk) c2.seg[0] = ConvSeg{h2, b.cout, SEG_SAME, H, W, 9, b.conv2_pk, 64, 0, 0, 1};
    else c2.seg[0] = ConvSeg{h2, b.cout, SEG_SAME, H, W, 9, b.conv2_w, 9 * b.cout, 0, b.cout};
    c2.nseg = 1;
    if (b.sc_w) {
        if (pk && b.sc_pk) {
            const int rows_a = ((b.ca + 63) / 64) * b.cout;
            c2.seg[c2.nseg++] = ConvSeg{xa, b.ca, SEG_SAME, H, W, 1, b.sc_pk, 64, 0, 0, 1};
            if (b.cb > 0) c2.seg[c2.nseg++] = ConvSeg{xb, b.cb, SEG_SAME, H, W, 1, b.sc_pk, 64, rows_a, 0, 1};
        } else {
            c2.seg[c2.nseg++] = ConvSeg{xa, b.ca, SEG_SAME, H, W, 1, b.sc_w, cin, 0, 0};
            if (b.cb > 0) c2.seg[c2.nseg++] = ConvSeg{xb, b.cb, SEG_SAME, H, W, 1, b.sc_w, cin, b.ca, 0};
        }
        c2.bias1 = b.sc_b;
    } else {
        c2.residual = xa;
    }
    c2.T = T;
    c2.ho = H;
    c2.wo = W;
    c2.cout = b.cout;
    c2.bias0 = b.conv2_b;
    c2.stats_out = up2 ? nullptr : stats_y;
    c2.dt = b.dt;
    if (up2 && conv_ws_applicable(c2)) {   // the TMA engine's staged epilogue stores the upsampled tensor
        c2.up2 = 1, c2.up_ho = up_ho, c2.up_wo = up_wo;
        c2.out = y;
        return conv_run(c2, stream);
    }
    c2.out = up2 ? y1 : y;   // up2 (fp32 / gather engine): the low-res output in Y1's (consumed) region, then upsampled
    if ((st = conv_run(c2, stream)) != DVC_OK || !up2) return st;
    return nearest_run(y1, y, T, H, W, up_ho, up_wo, b.cout, b.dt, stream);
}

dvc_status resblock_launch(const RB &b, const void *xa, const void *xb, int T, int H, int W, const void *carry_in,
                           void *carry_out, void *y, void *ws, cudaStream_t stream, const void *stats_a,
                           const void *stats_b, void *stats_y, int up2, int up_ho, int up_wo) {
    const int cs = b.P > 0 ? (b.ca + b.cb) / b.P : 0;
    DVC_CHECK_ARG(!up2 || stats_y == nullptr, DVC_ERR_ARG, "an upsampled block output has no statistics");
    dvc_status st = resblock_body(b, xa, xb, T, H, W, carry_in, y, ws, stream, stats_a, stats_b, stats_y, up2, up_ho,
                                  up_wo);
    if (st != DVC_OK || !carry_out || cs == 0) return st;
    // carry_out = X[T-1][..., 0:C_in/P] (the raw block input; y never aliases x), enqueued after every
    // reader of carry_in, so an in-place carry update (carry_out == carry_in) is well defined
    const size_t es = dt_size(b.dt);
    DVC_CUDA(cudaMemcpy2DAsync(carry_out, cs * es,
                               reinterpret_cast<const uint8_t *>(xa) + (size_t)(T - 1) * H * W * b.ca * es,
                               b.ca * es, cs * es, (size_t)H * W, cudaMemcpyDeviceToDevice, stream));
    return DVC_OK;
}

static RB rb_from_abi(const dvc_resblock *b) {
    RB r;
    r.ca = b->c_a;
    r.cb = b->c_b;
    r.cout = b->c_out;
    r.G = b->groups;
    r.P = b->shift_p;
    r.eps = b->eps;
    r.dt = b->dt;
    r.gn1_w = b->gn1_w;
    r.gn1_b = b->gn1_b;
    r.conv1_w = b->conv1_w;
    r.conv1_b = b->conv1_b;
    r.gn2_w = b->gn2_w;
    r.gn2_b = b->gn2_b;
    r.conv2_w = b->conv2_w;
    r.conv2_b = b->conv2_b;
    r.sc_w = b->sc_w;
    r.sc_b = b->sc_b;
    return r;
}

}  // namespace dvc

using namespace dvc;

extern "C" {

const char *dvc_status_string(dvc_status s) {
    switch (s) {
        case DVC_OK: return "DVC_OK";
        case DVC_ERR_ARG: return "DVC_ERR_ARG";
        case DVC_ERR_DIVISIBILITY: return "DVC_ERR_DIVISIBILITY";
        case DVC_ERR_SHAPE: return "DVC_ERR_SHAPE";
        case DVC_ERR_UNSUPPORTED: return "DVC_ERR_UNSUPPORTED";
        case DVC_ERR_WORKSPACE: return "DVC_ERR_WORKSPACE";
        case DVC_ERR_CUDA: return "DVC_ERR_CUDA";
        case DVC_ERR_NCCL: return "DVC_ERR_NCCL";
    }
    return "DVC_ERR_UNKNOWN";
}

const char *dvc_last_error(void) { return g_err; }

dvc_status dvc_set_conv_engine(int engine) {
    DVC_CHECK_ARG(engine >= 0 && engine <= 2, DVC_ERR_ARG, "engine must be 0, 1 or 2");
    g_ws_cg = engine;
    return DVC_OK;
}

dvc_status dvc_profile_begin(int max_launches) {
    DVC_CHECK_ARG(max_launches >= 1 && max_launches <= (1 << 20), DVC_ERR_ARG, "bad max_launches");
    if ((int)g_prof.ev.size() < 2 * max_launches) {
        size_t old = g_prof.ev.size();
        g_prof.ev.resize(2 * (size_t)max_launches);
        for (size_t i = old; i < g_prof.ev.size(); ++i) DVC_CUDA(cudaEventCreate(&g_prof.ev[i]));
    }
    g_prof.flops.assign(max_launches, 0.0);
    g_prof.ms.assign(max_launches, 0.0);
    g_prof.conv.assign(max_launches, 0);
    g_prof.label.assign(max_launches, std::string());
    g_prof.done = 0;
    g_prof.cap = max_launches;
    g_prof.used = 0;
    g_prof.on = true;
    return DVC_OK;
}

dvc_status dvc_profile_end(double *conv_ms, double *conv_flops, int *conv_launches) {
    DVC_CHECK_ARG(conv_ms && conv_flops && conv_launches, DVC_ERR_ARG, "null output");
    g_prof.on = false;
    double ms = 0, fl = 0;
    int nconv = 0;
    for (int i = 0; i < g_prof.used; ++i) {
        DVC_CUDA(cudaEventSynchronize(g_prof.ev[2 * i + 1]));
        float t = 0.f;
        DVC_CUDA(cudaEventElapsedTime(&t, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]));
        if (g_prof.conv[i]) {
            ms += t;
            fl += g_prof.flops[i];
            ++nconv;
        }
        g_prof.ms[i] = t;
    }
    g_prof.done = g_prof.used;
    *conv_ms = ms;
    *conv_flops = fl;
    *conv_launches = nconv;
    g_prof.used = 0;
    return DVC_OK;
}
int dvc_profile_record_count(void) { return g_prof.done; }
dvc_status dvc_profile_record(int i, double *ms, double *flops, char *label, int label_cap) {
    DVC_CHECK_ARG(i >= 0 && i < g_prof.done, DVC_ERR_ARG, "record %d not available (%d kept)", i, g_prof.done);
    if (ms) *ms = g_prof.ms[i];
    if (flops) *flops = g_prof.flops[i];
    if (label && label_cap > 0) snprintf(label, (size_t)label_cap, "%s", g_prof.label[i].c_str());
    return DVC_OK;
}
int dvc_abi_version(void) { return DVC_ABI_VERSION; }
int dvc_kernel_launch_count(void) { return g_launches; }

dvc_status dvc_device_check(int device) {
    int cur = 0;
    DVC_CUDA(cudaGetDevice(&cur));
    if (device != cur) DVC_CUDA(cudaSetDevice(device));
    dvc_status st = check_device();
    if (device != cur) cudaSetDevice(cur);
    return st;
}

dvc_status dvc_encode_pixelunshuffle(const void *frames, dvc_dtype frame_dt, int T, int H, int W, int s,
                                     const void *w_exp, const void *b_exp, int c_lat, void *latent, dvc_dtype dt,
                                     void *stream) {
    NvtxRange nv("dvc_encode_pixelunshuffle T=%d %dx%d", T, H, W);
    DVC_CHECK_ARG(frames && latent, DVC_ERR_ARG, "null frames/latent");
    DVC_CHECK_ARG(dt_valid(dt) && (dt_valid(frame_dt) || frame_dt == DVC_U8), DVC_ERR_ARG, "bad dtype");
    DVC_CHECK_ARG(frame_dt == dt || frame_dt == DVC_U8, DVC_ERR_UNSUPPORTED,
                  "frame_dt must equal latent_dt (or be DVC_U8)");
    DVC_CHECK_ARG(T >= 1 && H >= 1 && W >= 1 && s >= 1, DVC_ERR_ARG, "T, H, W, s must be >= 1");
    DVC_CHECK_ARG(H % s == 0 && W % s == 0, DVC_ERR_DIVISIBILITY, "H=%d and W=%d must be multiples of s=%d", H, W,
                  s);
    DVC_CHECK_ARG((w_exp == nullptr) == (b_exp == nullptr), DVC_ERR_ARG, "w_exp and b_exp go together");
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    cudaStream_t strm = reinterpret_cast<cudaStream_t>(stream);
    if (w_exp == nullptr) {
        DVC_CHECK_ARG(c_lat == 3 * s * s, DVC_ERR_SHAPE, "unshuffle only: c_lat must be 3*s*s=%d", 3 * s * s);
        if (frame_dt == DVC_U8) return unshuffle_u8_run(frames, T, H, W, s, latent, dt, strm);
        return unshuffle_run(frames, dt, T, H, W, s, latent, strm);
    }
    DVC_CHECK_ARG(s == 8, DVC_ERR_UNSUPPORTED, "fused expansion needs s == 8");
    DVC_CHECK_ARG(c_lat >= 16 && c_lat % 16 == 0, DVC_ERR_UNSUPPORTED, "c_lat must be a multiple of 16");
    if (frame_dt == DVC_U8) {
        DVC_CHECK_ARG(encode_tma_applicable(dt, H, W, s, c_lat) && W % 16 == 0, DVC_ERR_UNSUPPORTED,
                      "8-bit frames with expansion: 16-bit latent, c_lat <= 256, W %% 16 == 0");
        return encode_tma_run(frames, DVC_U8, T, H, W, w_exp, b_exp, c_lat, latent, dt, strm);
    }
    if (encode_tma_applicable(dt, H, W, s, c_lat) && !dvc_knob("DVC_ENCODE_GATHER"))
        return encode_tma_run(frames, dt, T, H, W, w_exp, b_exp, c_lat, latent, dt, strm);
    ConvDesc d{};
    d.seg[0] = ConvSeg{frames, 192, SEG_UNSHUFFLE8, H, W, 1, w_exp, 192, 0, 0};
    d.nseg = 1;
    d.T = T;
    d.ho = H / 8;
    d.wo = W / 8;
    d.cout = c_lat;
    d.bias0 = b_exp;
    d.out = latent;
    d.dt = dt;
    return conv_run(d, strm);
}

dvc_status dvc_resblock_workspace_size(const dvc_resblock *b, int T, int H, int W, size_t *bytes) {
    DVC_CHECK_ARG(b && bytes, DVC_ERR_ARG, "null argument");
    RB r = rb_from_abi(b);
    DVC_CHECK_ARG(r.G >= 1 && r.ca >= 0 && r.cb >= 0 && r.cout >= 0 && T >= 1 && H >= 1 && W >= 1, DVC_ERR_ARG,
                  "bad sizes");
    *bytes = resblock_ws_bytes(r.ca, r.cb, r.cout, r.G, T, H, W, r.dt);
    return DVC_OK;
}

dvc_status dvc_resblock_tsm_forward(const dvc_resblock *b, const void *x_a, const void *x_b, int T, int H, int W,
                                    const void *carry_in, void *carry_out, void *y, void *workspace,
                                    size_t ws_bytes, void *stream) {
    NvtxRange nv("dvc_resblock_tsm_forward T=%d %dx%d", T, H, W);
    DVC_CHECK_ARG(b && x_a && y && workspace, DVC_ERR_ARG, "null argument");
    RB r = rb_from_abi(b);
    dvc_status st = resblock_validate(r, T, H, W);
    if (st != DVC_OK) return st;
    DVC_CHECK_ARG(r.cb == 0 || x_b != nullptr, DVC_ERR_ARG, "x_b is null but c_b > 0");
    DVC_CHECK_ARG(ws_bytes >= resblock_ws_bytes(r.ca, r.cb, r.cout, r.G, T, H, W, r.dt), DVC_ERR_WORKSPACE,
                  "workspace too small");
    DVC_CHECK_ARG(((uintptr_t)workspace & 255) == 0, DVC_ERR_ARG, "workspace must be 256-byte aligned");
    if (carry_in && carry_out && r.P > 0) {
        const size_t cb = (size_t)H * W * ((r.ca + r.cb) / r.P) * dt_size(r.dt);
        const uintptr_t a = (uintptr_t)carry_in, o = (uintptr_t)carry_out;
        DVC_CHECK_ARG(a == o || a + cb <= o || o + cb <= a, DVC_ERR_ARG,
                      "carry_out must equal carry_in or not overlap it");
    }
    if ((st = check_device()) != DVC_OK) return st;
    return resblock_launch(r, x_a, r.cb ? x_b : nullptr, T, H, W, carry_in, carry_out, y, workspace,
                           reinterpret_cast<cudaStream_t>(stream));
}

dvc_status dvc_debug_shift_gather(const void *x_a, const void *x_b, int c_a, int c_b, int shift_p, dvc_dtype dt,
                                  int T, int H, int W, const void *carry_in, void *xs, void *stream) {
    DVC_CHECK_ARG(x_a && xs && (c_b == 0 || x_b), DVC_ERR_ARG, "null argument");
    DVC_CHECK_ARG(dt_valid(dt) && T >= 1 && H >= 1 && W >= 1 && c_a > 0 && c_b >= 0, DVC_ERR_ARG, "bad sizes");
    DVC_CHECK_ARG(shift_p >= 1 && (c_a + c_b) % shift_p == 0, DVC_ERR_DIVISIBILITY, "P must divide C");
    dvc_status st = check_device();
    if (st != DVC_OK) return st;
    NormArgs a{x_a, c_b ? x_b : nullptr, carry_in, c_a, c_b, (c_a + c_b) / shift_p, T, H * W, 1, 0.f,
               nullptr, nullptr, xs, nullptr};
    return shift_gather_run(a, dt, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
