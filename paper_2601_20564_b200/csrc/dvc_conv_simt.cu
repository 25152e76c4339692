// dvc_conv_simt.cu -- fp32 SIMT convolution engine for the DVC_F32 validation
// mode.  tf32 tensor cores are too inexact for the 1e-5 gate, so
// this is plain fp32 FMA.  To keep rounding error well under 1e-5 at
// K = 17 280 it accumulates each (segment, tap, 64-channel chunk) into a
// partial sum and adds the partials into the output accumulator.
// Tile: 64 output pixels x 64 output channels per 256-thread block, 4x4 per thread.
#include "dvc_conv.cuh"

namespace dvc {

struct SimtParams {
    ConvSeg seg[4];
    int nseg, T, ho, wo, cout;
    long M;
    const float *bias0, *bias1, *residual;
    float *out;
};

constexpr int SBM = 64, SBN = 64, SBK = 16;

__global__ void __launch_bounds__(256) conv_simt_kernel(const SimtParams p) {
    __shared__ float As[SBK][SBM + 4];
    __shared__ float Bs[SBK][SBN + 4];
    __shared__ int rowinfo[SBM];
    const int tid = threadIdx.x;
    const long m0 = (long)blockIdx.x * SBM;
    const int n0 = blockIdx.y * SBN;
    const int tm = (tid & 15) * 4, tn = (tid >> 4) * 4;
    if (tid < SBM) {
        long m = m0 + tid;
        if (m < p.M) {
            int hw = p.ho * p.wo;
            int t = (int)(m / hw), rem = (int)(m % hw);
            rowinfo[tid] = (t << 24) | ((rem / p.wo) << 12) | (rem % p.wo);
        } else {
            rowinfo[tid] = -1;
        }
    }
    __syncthreads();
    float acc[4][4] = {};
    float part[4][4] = {};
    for (int s = 0; s < p.nseg; ++s) {
        const ConvSeg &sg = p.seg[s];
        const float *src = reinterpret_cast<const float *>(sg.src);
        const float *w = reinterpret_cast<const float *>(sg.w);
        for (int tap = 0; tap < sg.taps; ++tap) {
            const int dy = sg.taps == 9 ? tap / 3 - 1 : 0, dx = sg.taps == 9 ? tap % 3 - 1 : 0;
            for (int c0 = 0; c0 < sg.c_src; c0 += SBK) {
                // A tile: SBK channels x SBM pixels
                for (int e = tid; e < SBK * SBM; e += 256) {
                    int r = e % SBM, k = e / SBM;
                    int info = rowinfo[r];
                    float v = 0.f;
                    int c = c0 + k;
                    if (info >= 0 && c < sg.c_src) {
                        int t = info >> 24, y = (info >> 12) & 0xFFF, x = info & 0xFFF;
                        if (sg.mode == SEG_UNSHUFFLE8) {
                            int col = c / 64, i = (c / 8) % 8, jj = c % 8;
                            v = src[(((long)t * 3 + col) * sg.hi + 8 * y + i) * sg.wi + 8 * x + jj];
                        } else {
                            long pix = seg_src_pixel(sg, p.ho, p.wo, t, y, x, dy, dx);
                            if (pix >= 0) v = src[pix * sg.c_src + c];
                        }
                    }
                    As[k][r] = v;
                }
                for (int e = tid; e < SBK * SBN; e += 256) {
                    int nn = e % SBN, k = e / SBN;
                    int n = n0 + nn, c = c0 + k;
                    Bs[k][nn] = (n < p.cout && c < sg.c_src)
                                    ? w[(long)n * sg.w_ld + sg.w_col0 + tap * sg.w_tapstride + c]
                                    : 0.f;
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < SBK; ++k) {
                    float a[4], b[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i] = As[k][tm + i];
#pragma unroll
                    for (int i = 0; i < 4; ++i) b[i] = Bs[k][tn + i];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int jn = 0; jn < 4; ++jn) part[i][jn] = fmaf(a[i], b[jn], part[i][jn]);
                }
                __syncthreads();
                if (((c0 + SBK) % 64) == 0 || c0 + SBK >= sg.c_src) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int jn = 0; jn < 4; ++jn) {
                            acc[i][jn] += part[i][jn];
                            part[i][jn] = 0.f;
                        }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        long m = m0 + tm + i;
        if (m >= p.M) continue;
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) {
            int n = n0 + tn + jn;
            if (n >= p.cout) continue;
            float v = acc[i][jn];
            if (p.bias0) v += p.bias0[n];
            if (p.bias1) v += p.bias1[n];
            if (p.residual) v += p.residual[m * p.cout + n];
            p.out[m * p.cout + n] = v;
        }
    }
}

dvc_status conv_simt_run(const ConvDesc &d, cudaStream_t stream) {
    dvc_status st = conv_check(d, false);
    if (st != DVC_OK) return st;
    SimtParams p;
    for (int s = 0; s < d.nseg; ++s) p.seg[s] = d.seg[s];
    p.nseg = d.nseg;
    p.T = d.T;
    p.ho = d.ho;
    p.wo = d.wo;
    p.cout = d.cout;
    p.M = d.M();
    p.bias0 = reinterpret_cast<const float *>(d.bias0);
    p.bias1 = reinterpret_cast<const float *>(d.bias1);
    p.residual = reinterpret_cast<const float *>(d.residual);
    p.out = reinterpret_cast<float *>(d.out);
    dim3 grid(ceil_div(p.M, SBM), ceil_div(d.cout, SBN));
    conv_simt_kernel<<<grid, 256, 0, stream>>>(p);
    ++g_launches;
    return check_launch("conv_simt_kernel");
}

dvc_status conv_check(const ConvDesc &d, bool tc) {
    DVC_CHECK_ARG(d.nseg >= 1 && d.nseg <= 4, DVC_ERR_ARG, "conv: 1..4 segments");
    DVC_CHECK_ARG(d.T >= 1 && d.ho >= 1 && d.wo >= 1 && d.cout >= 1, DVC_ERR_ARG, "conv: empty shape");
    DVC_CHECK_ARG(d.T < 256 && d.ho < 4096 && d.wo < 4096, DVC_ERR_UNSUPPORTED,
                  "conv: T < 256 and spatial dims < 4096 required");
    DVC_CHECK_ARG(d.out != nullptr, DVC_ERR_ARG, "conv: null output");
    for (int s = 0; s < d.nseg; ++s) {
        const ConvSeg &g = d.seg[s];
        DVC_CHECK_ARG(g.src && g.w && g.c_src > 0 && (g.taps == 1 || g.taps == 9), DVC_ERR_ARG,
                      "conv: bad segment %d", s);
        DVC_CHECK_ARG(g.c_src % 8 == 0, DVC_ERR_UNSUPPORTED, "conv: channels must be a multiple of 8");
        if (tc) {
            DVC_CHECK_ARG(g.c_src % 16 == 0, DVC_ERR_UNSUPPORTED,
                          "tensor-core conv: channels must be a multiple of 16 (got %d)", g.c_src);
            DVC_CHECK_ARG(g.w_ld % 8 == 0, DVC_ERR_UNSUPPORTED, "tensor-core conv: weight rows 16-byte aligned");
        }
        if (g.mode == SEG_UNSHUFFLE8)
            DVC_CHECK_ARG(g.c_src == 192 && g.taps == 1 && g.hi == 8 * d.ho && g.wi == 8 * d.wo, DVC_ERR_SHAPE,
                          "conv: unshuffle segment shape");
    }
    if (tc) DVC_CHECK_ARG(d.cout % 16 == 0, DVC_ERR_UNSUPPORTED, "tensor-core conv: cout must be a multiple of 16");
    return DVC_OK;
}

double conv_flops(const ConvDesc &d) {
    double k = 0;
    for (int s = 0; s < d.nseg; ++s) k += (double)d.seg[s].taps * d.seg[s].c_src;
    return 2.0 * (double)d.M() * d.cout * k;
}

dvc_status conv_run(const ConvDesc &d, cudaStream_t stream) {
    ProfSlot slot = prof_begin(stream);
    const bool ws = d.dt != DVC_F32 && conv_ws_applicable(d);
    DVC_CHECK_ARG(!d.geglu || ws, DVC_ERR_UNSUPPORTED, "GEGLU epilogue needs the TMA conv engine");
    dvc_status st = d.dt == DVC_F32 ? conv_simt_run(d, stream) : ws ? conv_ws_run(d, stream) : conv_tc_run(d, stream);
    prof_end(slot, stream, conv_flops(d), d.dt == DVC_F32 ? "simt" : ws ? "ws" : "tc", d);
    if (st == DVC_OK && d.stats_out != nullptr && !ws)   // engines without the fused epilogue statistics
        st = box_stats_run(d.out, d.T, d.ho, d.wo, d.cout, d.dt, reinterpret_cast<float *>(d.stats_out), stream);
    return st;
}

}  // namespace dvc
