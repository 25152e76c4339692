// dvc_conv_tc.cu -- tcgen05 / TMEM implicit-GEMM convolution engine (sm_100a).
//
// GEMM view of one convolution:
//   M = T*ho*wo output pixels (frames packed on the batch dim)
//   N = C_out (tiled by BN <= 256, a multiple of 16)
//   K = sum over segments of taps * C_src (consumed in 64-channel stages)
// Per CTA: NACC accumulators of 128 rows x BN fp32 columns in TMEM; every stage
// stages an A tile (NACC*128 gathered pixel rows x 64 channels) and a B tile
// (BN weight rows x 64 channels) in shared memory in the UMMA K-major
// SWIZZLE_128B canonical layout and issues NACC * (valid channels / 16)
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) from one thread.
//
// Warp roles (192 threads):
//   warps 0-3  A producer: per-row gather addressing (3x3 taps, zero padding,
//              stride-2, nearest-up, unshuffle) with 16-byte cp.async
//              (zero-fill for padding), manual 128B swizzle; then the epilogue
//              (TMEM -> registers -> bias / residual -> 16-bit global stores).
//   warp 4     B producer: TMA 2D tile loads of the weight matrix (SW128).
//   warp 5     TMEM allocator + MMA issuer (one elected lane).
// Pipeline: STAGES-deep ring of {A,B} tiles with full/empty mbarriers; the
// MMA commits (tcgen05.commit) free a stage; a final commit signals the epilogue.
#include <cuda.h>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include "dvc_conv.cuh"
#include "dvc_ptx.cuh"

namespace dvc {

// ----------------------------------------------------------------- kernel params
struct TcParams {
    CUtensorMap bmap[2];   // weight matrices (segment's b index)
    ConvSeg seg[4];
    int bidx[4];           // tensor map per segment
    int nseg;
    int T, ho, wo, cout, bn;
    long M;
    const void *bias0, *bias1, *residual;
    void *out;
    uint32_t idesc;
};

constexpr int kThreads = 192;

__device__ __forceinline__ int pack_row(long m, int ho, int wo) {
    int hw = ho * wo;
    int t = (int)(m / hw);
    int rem = (int)(m - (long)t * hw);
    int y = rem / wo, x = rem - y * wo;
    return (t << 24) | (y << 12) | x;
}

template <typename T, int NACC, int STAGES>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ TcParams p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so the compiler keeps the
    // shared address space (an integer round trip would turn every access generic)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int BN = p.bn;
    constexpr int A_TILE = 128 * 128;          // bytes per 128-row x 64-ch tile
    constexpr int A_STAGE = NACC * A_TILE;
    const int B_STAGE = BN * 128;
    uint8_t *sA = smem;
    uint8_t *sB = sA + STAGES * A_STAGE;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * B_STAGE);
    uint64_t *empty = full + STAGES;
    uint64_t *accf = empty + STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);
    int *rowinfo = reinterpret_cast<int *>(tmem_slot + 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long m0 = (long)blockIdx.x * (NACC * 128);
    const int n0 = blockIdx.y * BN;
    const uint32_t ncols = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128
                         : (NACC * BN <= 256) ? 256 : 512;

    if (warp == 4 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 128 + 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
        tma_prefetch(&p.bmap[0]);
        if (p.nseg > 1) tma_prefetch(&p.bmap[1]);
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int r = tid; r < NACC * 128; r += kThreads) {
        long m = m0 + r;
        rowinfo[r] = m < p.M ? pack_row(m, p.ho, p.wo) : -1;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();     // predecessor grid complete: activations may be read / written
    griddep_launch();   // the successor may be scheduled on SMs that free up

    if (warp < 4) {
        // ===================== A producer (gather + cp.async) =====================
        const int j = tid & 7;          // 16-byte granule within the 128-byte row
        const int rb = tid >> 3;        // rows rb, rb+16, ...
        constexpr int NR = NACC * 8;    // rows per thread
        int ry[NR], rx[NR], rt[NR];     // output pixel of each row (t < 0: row beyond M)
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const int info = rowinfo[rb + 16 * i];
            rt[i] = info >> 24;          // -1 when invalid (sign extends)
            ry[i] = (info >> 12) & 0xFFF;
            rx[i] = info & 0xFFF;
        }
        int stage = 0;
        uint32_t phase = 0;
        for (int s = 0; s < p.nseg; ++s) {
            const ConvSeg &sg = p.seg[s];
            const int nch = (sg.c_src + 63) >> 6;
            const T *src = reinterpret_cast<const T *>(sg.src);
            const int mode = sg.mode, hi = sg.hi, wi = sg.wi, csrc = sg.c_src;
            for (int tap = 0; tap < sg.taps; ++tap) {
                const int dy = sg.taps == 9 ? tap / 3 - 1 : 0;
                const int dx = sg.taps == 9 ? tap % 3 - 1 : 0;
                // per-row source pixel for this tap (channel-independent), -1 = zero padding
                long pix[NR];
#pragma unroll
                for (int i = 0; i < NR; ++i) {
                    if (rt[i] < 0) {
                        pix[i] = -1;
                    } else if (mode == SEG_SAME) {
                        const int iy = ry[i] + dy, ix = rx[i] + dx;
                        pix[i] = ((unsigned)iy < (unsigned)hi && (unsigned)ix < (unsigned)wi)
                                     ? ((long)rt[i] * hi + iy) * wi + ix : -1;
                    } else if (mode == SEG_UNSHUFFLE8) {
                        pix[i] = 0;
                    } else {
                        pix[i] = seg_src_pixel(sg, p.ho, p.wo, rt[i], ry[i], rx[i], dy, dx);
                    }
                }
                for (int ch = 0; ch < nch; ++ch) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t base = smem_u32(sA + stage * A_STAGE);
                    const int c = ch * 64 + j * 8;
                    const bool cvalid = c < csrc;
#pragma unroll
                    for (int i = 0; i < NR; ++i) {
                        const int r = rb + 16 * i;
                        const T *g = src;
                        uint32_t nbytes = 0;
                        if (pix[i] >= 0 && cvalid) {
                            if (mode == SEG_UNSHUFFLE8) {
                                // a1: latent channel ch*64 + j*8 + (0..7) = frame (colour ch, row 8y+j, cols 8x..8x+7)
                                g = src + (((long)rt[i] * 3 + ch) * hi + 8 * ry[i] + j) * (long)wi + 8 * rx[i];
                            } else {
                                g = src + pix[i] * csrc + c;
                            }
                            nbytes = 16;
                        }
                        const uint32_t dst = base + (uint32_t)(r >> 7) * A_TILE + (uint32_t)(r & 127) * 128 +
                                             (uint32_t)((j ^ (r & 7)) << 4);
                        cp_async_16(dst, g, nbytes);
                    }
                    cp_async_arrive_noinc(&full[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        // ===================== epilogue =====================
        mbar_wait(accf, 0);
        tc_fence_after();
        const T *b0 = reinterpret_cast<const T *>(p.bias0);
        const T *b1 = reinterpret_cast<const T *>(p.bias1);
        const T *res = reinterpret_cast<const T *>(p.residual);
        T *out = reinterpret_cast<T *>(p.out);
#pragma unroll 1
        for (int a = 0; a < NACC; ++a) {
            const int r = a * 128 + warp * 32 + lane;
            const long m = m0 + r;
            const bool rvalid = m < p.M;
#pragma unroll 1
            for (int cc = 0; cc < BN; cc += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a * BN + cc), v);
                const int n = n0 + cc;
                if (rvalid && n < p.cout) {
                    float f[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
                    if (b0) {
                        float bb[8];
                        load8(b0 + n, bb);
#pragma unroll
                        for (int i = 0; i < 8; ++i) f[i] += bb[i];
                        load8(b0 + n + 8, bb);
#pragma unroll
                        for (int i = 0; i < 8; ++i) f[8 + i] += bb[i];
                    }
                    if (b1) {
                        float bb[8];
                        load8(b1 + n, bb);
#pragma unroll
                        for (int i = 0; i < 8; ++i) f[i] += bb[i];
                        load8(b1 + n + 8, bb);
#pragma unroll
                        for (int i = 0; i < 8; ++i) f[8 + i] += bb[i];
                    }
                    if (res) {
                        float rr[8];
                        load8(res + m * p.cout + n, rr);
#pragma unroll
                        for (int i = 0; i < 8; ++i) f[i] += rr[i];
                        load8(res + m * p.cout + n + 8, rr);
#pragma unroll
                        for (int i = 0; i < 8; ++i) f[8 + i] += rr[i];
                    }
                    float lo[8], hi[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        lo[i] = f[i];
                        hi[i] = f[8 + i];
                    }
                    store8(out + m * p.cout + n, lo);
                    store8(out + m * p.cout + n + 8, hi);
                }
            }
        }
    } else if (warp == 4) {
        // ===================== B producer (TMA) =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int s = 0; s < p.nseg; ++s) {
                const ConvSeg &sg = p.seg[s];
                const int nch = (sg.c_src + 63) >> 6;
                const CUtensorMap *map = &p.bmap[p.bidx[s]];
                for (int tap = 0; tap < sg.taps; ++tap) {
                    for (int ch = 0; ch < nch; ++ch) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_arrive_expect_tx(&full[stage], (uint32_t)B_STAGE);
                        tma_load_2d(sB + stage * B_STAGE, map, &full[stage],
                                    sg.w_col0 + tap * sg.w_tapstride + ch * 64, n0);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            bool first = true;
            for (int s = 0; s < p.nseg; ++s) {
                const ConvSeg &sg = p.seg[s];
                const int nch = (sg.c_src + 63) >> 6;
                for (int tap = 0; tap < sg.taps; ++tap) {
                    for (int ch = 0; ch < nch; ++ch) {
                        mbar_wait(&full[stage], phase);
                        fence_proxy_async();
                        tc_fence_after();
                        const int valid = min(64, sg.c_src - ch * 64);
                        const int ksteps = valid >> 4;
                        const uint32_t a0 = smem_u32(sA + stage * A_STAGE);
                        const uint32_t b0 = smem_u32(sB + stage * B_STAGE);
                        for (int k = 0; k < ksteps; ++k) {
                            const uint64_t bd = sdesc_sw128(b0 + k * 32);
#pragma unroll
                            for (int a = 0; a < NACC; ++a) {
                                const uint64_t ad = sdesc_sw128(a0 + a * A_TILE + k * 32);
                                tc_mma(tmem + (uint32_t)(a * BN), ad, bd, p.idesc, first ? 0u : 1u);
                            }
                            first = false;
                        }
                        tc_commit(&empty[stage]);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
            tc_commit(accf);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
    }
}

// ----------------------------------------------------------------- host side
// cuTensorMapEncodeTiled behind a small cache: a decode step encodes ~400 tensor maps (every conv
// launch describes its activations, weights and output), almost always with the same arguments as the
// previous step, so the host cost of a repeated call drops to a hash lookup (the key is every argument
// of the encode; the cache is cleared when it grows past 8192 entries).
static PFN_encodeTiled_t g_encode_raw = nullptr;
namespace {
struct MapKey {
    uint64_t w[26];
    bool operator==(const MapKey &o) const { return memcmp(w, o.w, sizeof(w)) == 0; }
};
struct MapKeyHash {
    size_t operator()(const MapKey &k) const {
        uint64_t h = 1469598103934665603ull;
        for (uint64_t v : k.w) h = (h ^ v) * 1099511628211ull;
        return (size_t)h;
    }
};
}  // namespace
static CUresult encode_cached(CUtensorMap *map, CUtensorMapDataType dt, cuuint32_t rank, void *addr,
                              const cuuint64_t *gdim, const cuuint64_t *gstride, const cuuint32_t *box,
                              const cuuint32_t *estr, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                              CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
    if (rank < 1 || rank > 5) return g_encode_raw(map, dt, rank, addr, gdim, gstride, box, estr, il, sw, l2, oob);
    MapKey k;
    memset(&k, 0, sizeof(k));
    k.w[0] = (uint64_t)dt | ((uint64_t)rank << 8) | ((uint64_t)il << 16) | ((uint64_t)sw << 24) |
             ((uint64_t)l2 << 32) | ((uint64_t)oob << 40);
    k.w[1] = (uint64_t)(uintptr_t)addr;
    for (cuuint32_t i = 0; i < rank; ++i) {
        k.w[2 + i] = gdim[i];
        k.w[7 + i] = i + 1 < rank ? gstride[i] : 0;
        k.w[12 + i] = box[i];
        k.w[17 + i] = estr[i];
    }
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(k);
        if (it != cache.end()) {
            *map = it->second;
            return CUDA_SUCCESS;
        }
    }
    const CUresult r = g_encode_raw(map, dt, rank, addr, gdim, gstride, box, estr, il, sw, l2, oob);
    if (r == CUDA_SUCCESS) {
        std::lock_guard<std::mutex> lock(mu);
        if (cache.size() > 8192) cache.clear();
        cache.emplace(k, *map);
    }
    return r;
}

PFN_encodeTiled_t get_encode_fn() {
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode_raw = reinterpret_cast<PFN_encodeTiled_t>(ptr);
    });
    return g_encode_raw ? encode_cached : nullptr;
}

// 2D [rows][cols] 16-bit matrix, box {64 cols, box_rows}, SWIZZLE_128B, OOB zero fill.
dvc_status make_bmap_rows(CUtensorMap *map, const void *ptr, dvc_dtype dt, long rows, long cols, int box_rows) {
    PFN_encodeTiled_t enc = get_encode_fn();
    DVC_CHECK_ARG(enc != nullptr, DVC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DVC_CHECK_ARG(((uintptr_t)ptr & 15) == 0 && (cols * 2) % 16 == 0, DVC_ERR_ARG,
                  "weight matrix must be 16-byte aligned with 16-byte rows");
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)(cols * 2)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, dt == DVC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                     const_cast<void *>(ptr), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DVC_CHECK_ARG(r == CUDA_SUCCESS, DVC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return DVC_OK;
}

template <typename T, int NACC, int STAGES>
static dvc_status launch_tc(const TcParams &p, int grid_m, int grid_n, cudaStream_t stream) {
    size_t smem = 1024 + (size_t)STAGES * (NACC * 16384 + p.bn * 128) + 8 * (2 * STAGES + 1) + 16 + NACC * 128 * 4;
    auto kern = conv_tc_kernel<T, NACC, STAGES>;
    {   // host cost: the attribute is set once per kernel / size
        dvc_status ss_ = ensure_smem((const void *)kern, (int)smem);
        if (ss_ != DVC_OK) return ss_;
    }
    DVC_CUDA(launch_pdl(kern, dim3(grid_m, grid_n), dim3(kThreads), smem, stream, 1, p));
    ++g_launches;
    return check_launch("conv_tc_kernel");
}

dvc_status conv_tc_run(const ConvDesc &d, cudaStream_t stream) {
    dvc_status st = conv_check(d, true);
    if (st != DVC_OK) return st;
    TcParams p;
    memset(&p, 0, sizeof(p));
    p.nseg = d.nseg;
    p.T = d.T;
    p.ho = d.ho;
    p.wo = d.wo;
    p.cout = d.cout;
    p.M = d.M();
    p.bias0 = d.bias0;
    p.bias1 = d.bias1;
    p.residual = d.residual;
    p.out = d.out;
    // N tile: the whole of cout if <= 256, else the largest multiple of 16 <= 256 dividing cout
    int bn = d.cout;
    if (bn > 256) {
        bn = 0;
        for (int c = 256; c >= 16; c -= 16)
            if (d.cout % c == 0) {
                bn = c;
                break;
            }
    }
    DVC_CHECK_ARG(bn >= 16, DVC_ERR_UNSUPPORTED, "no N tile for cout=%d", d.cout);
    p.bn = bn;
    int nb = 0;
    const void *bw[2] = {nullptr, nullptr};
    for (int s = 0; s < d.nseg; ++s) {
        p.seg[s] = d.seg[s];
        int idx = -1;
        for (int k = 0; k < nb; ++k)
            if (bw[k] == d.seg[s].w) idx = k;
        if (idx < 0) {
            DVC_CHECK_ARG(nb < 2, DVC_ERR_UNSUPPORTED, "at most two weight matrices per conv");
            idx = nb++;
            bw[idx] = d.seg[s].w;
            st = make_bmap_rows(&p.bmap[idx], d.seg[s].w, d.dt, d.cout, d.seg[s].w_ld, bn);
            if (st != DVC_OK) return st;
        }
        p.bidx[s] = idx;
    }
    const int bf = d.dt == DVC_BF16;
    p.idesc = make_idesc(bf, 128, bn);
    const int grid_n = d.cout / bn;
    const long M = d.M();
    // two accumulators (M = 256 rows per CTA, weights reused twice) when that
    // still gives >= 2 waves on 148 SMs; else one (more CTAs for small levels)
    const bool two = ((M + 255) / 256) * grid_n >= 2 * 148 && 2 * bn <= 512;
    if (two) {
        if (bf) return launch_tc<__nv_bfloat16, 2, 3>(p, ceil_div(M, 256), grid_n, stream);
        return launch_tc<__half, 2, 3>(p, ceil_div(M, 256), grid_n, stream);
    }
    if (bf) return launch_tc<__nv_bfloat16, 1, 4>(p, ceil_div(M, 128), grid_n, stream);
    return launch_tc<__half, 1, 4>(p, ceil_div(M, 128), grid_n, stream);
}

}  // namespace dvc
