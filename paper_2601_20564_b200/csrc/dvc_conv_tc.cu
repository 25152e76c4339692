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
#include "dvc_conv.cuh"

namespace dvc {

// ----------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t a = smem_u32(b);
    while (!mbar_try_wait(a, parity)) {
    }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: rows of 128 B, 8-row
// swizzle atoms 1024 B apart (SBO), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;               // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;     // SBO
    d |= (uint64_t)1 << 46;               // version
    d |= (uint64_t)2 << 61;               // SWIZZLE_128B
    return d;
}
// Instruction descriptor kind::f16: D fp32, A/B fp16 (0) or bf16 (1), both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int ab_bf16, int M, int N) {
    return (1u << 4) | ((uint32_t)ab_bf16 << 7) | ((uint32_t)ab_bf16 << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

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
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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

    if (warp < 4) {
        // ===================== A producer (gather + cp.async) =====================
        const int j = tid & 7;          // 16-byte granule within the 128-byte row
        const int rb = tid >> 3;        // rows rb, rb+16, ...
        int stage = 0;
        uint32_t phase = 0;
        for (int s = 0; s < p.nseg; ++s) {
            const ConvSeg &sg = p.seg[s];
            const int nch = (sg.c_src + 63) >> 6;
            const T *src = reinterpret_cast<const T *>(sg.src);
            for (int tap = 0; tap < sg.taps; ++tap) {
                const int dy = sg.taps == 9 ? tap / 3 - 1 : 0;
                const int dx = sg.taps == 9 ? tap % 3 - 1 : 0;
                for (int ch = 0; ch < nch; ++ch) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t base = smem_u32(sA + stage * A_STAGE);
                    const int c = ch * 64 + j * 8;
                    const bool cvalid = c < sg.c_src;
#pragma unroll 4
                    for (int i = 0; i < NACC * 8; ++i) {
                        const int r = rb + 16 * i;
                        const int info = rowinfo[r];
                        const T *g = src;
                        uint32_t nbytes = 0;
                        if (info >= 0 && cvalid) {
                            const int t = info >> 24, y = (info >> 12) & 0xFFF, x = info & 0xFFF;
                            if (sg.mode == SEG_UNSHUFFLE8) {
                                // a1: latent channel ch*64 + j*8 + (0..7) = frame (color ch, row 8y+j, cols 8x..8x+7)
                                const long H = sg.hi, W = sg.wi;
                                g = src + (((long)t * 3 + ch) * H + 8 * y + j) * W + 8 * x;
                                nbytes = 16;
                            } else {
                                long pix = seg_src_pixel(sg, p.ho, p.wo, t, y, x, dy, dx);
                                if (pix >= 0) {
                                    g = src + pix * sg.c_src + c;
                                    nbytes = 16;
                                }
                            }
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
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                     const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                     CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                     CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    });
    return fn;
}

// 2D [rows][cols] 16-bit matrix, box {64 cols, box_rows}, SWIZZLE_128B, OOB zero fill.
static dvc_status make_bmap(CUtensorMap *map, const void *ptr, dvc_dtype dt, long rows, long cols, int box_rows) {
    PFN_encodeTiled enc = get_encode();
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
    DVC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<dim3(grid_m, grid_n), kThreads, smem, stream>>>(p);
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
            st = make_bmap(&p.bmap[idx], d.seg[s].w, d.dt, d.cout, d.seg[s].w_ld, bn);
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
