// Microbenchmark: cycles per tcgen05.mma (kind::f16, SS operands from shared memory, cta_group::1,
// M = 128, K = 16) issued back to back by one thread, for N in {16, 32, 64, 128, 256}, with one
// accumulator (dependent chain) or two (alternating), and with the issuing code either precomputed
// descriptors (lean) or per-MMA elect + predicate (as mma_stage).  Operand contents are irrelevant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2601_20564_b200/csrc umma_rate.cu
#include <cstdio>
#include <cstdint>
#include "dvc_ptx.cuh"
using namespace dvc;

__device__ __forceinline__ uint32_t make_idesc_bf16(int M, int N) {
    // kind::f16: D fp32 (bits 4-5 = 1), A/B bf16 (bits 7-9 = 1, 10-12 = 1), K-major, N >> 3 at 17, M >> 4 at 24
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int NACC, int MODE>   // MODE 0: lean loop; 1: mma_stage (4 MMAs + commit per stage) + a passed-barrier wait
__global__ void __launch_bounds__(128, 1) umma_rate(int N, int nmma, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) tmem_alloc<1>(smem_u32(&tslot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t idesc = make_idesc_bf16(128, N);
        const uint32_t a_lo = desc_lo(smem_u32(smem), 16), b_lo = desc_lo(smem_u32(smem + 65536), 16);
        long long t0 = 0, t1 = 0;
        if constexpr (MODE == 1) {   // converged warp, as the fused engine's MMA issuer
            __shared__ uint64_t sb[2];
            if (threadIdx.x == 0) { mbar_init(&sb[0], 1); mbar_init(&sb[1], 1); }
            __syncwarp();
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sb[1])) : "memory");
            __syncwarp();
            t0 = clock64();
            uint32_t acc = 0;
            for (int i = 0; i < nmma / 4; ++i) {
                mbar_wait_spin_addr(smem_u32(&sb[1]), 0);   // completed phase 0: returns at once
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)((i % NACC) * 256);
                mma_stage<1>(d, a_lo, kDescHiSw128, 2u, b_lo, kDescHiSw128, idesc, 4u, acc, smem_u32(&sb[0]));
                acc = 1;
            }
            commit_elected<1>(smem_u32(&bar));
            t1 = clock64();
        } else if (elect_one()) {
            t0 = clock64();
            for (int i = 0; i < nmma; ++i) {
                const uint64_t ad = ((uint64_t)kDescHiSw128 << 32) | (a_lo + 2u * (i & 3));
                const uint64_t bd = ((uint64_t)kDescHiSw128 << 32) | (b_lo + 2u * (i & 3));
                const uint32_t d = tmem + (uint32_t)((i % NACC) * 256);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                             ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(i >= NACC ? 1 : 0) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(smem_u32(&bar)) : "memory");
            t1 = clock64();
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        const long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tmem, 512); }
}

int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    const int smem = 160 * 1024;
    cudaFuncSetAttribute(umma_rate<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(umma_rate<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(umma_rate<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nmma = 4096;
    for (int N : {16, 32, 64, 128, 256})
        for (int nacc : {1, 2, 3}) {   // 3: one accumulator, mma_stage issue path
            for (int rep = 0; rep < 2; ++rep) {
                if (nacc == 1) umma_rate<1, 0><<<1, 128, smem>>>(N, nmma, d);
                else if (nacc == 2) umma_rate<2, 0><<<1, 128, smem>>>(N, nmma, d);
                else umma_rate<1, 1><<<1, 128, smem>>>(N, nmma, d);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            }
            const cudaError_t e = cudaGetLastError();
            printf("N=%3d acc=%d  issue %.1f cyc/mma  complete %.1f cyc/mma  (math floor %.1f)  %s\n", N, nacc,
                   (double)h[0] / nmma, (double)h[1] / nmma, 128.0 * N * 16 / 4096.0, cudaGetErrorString(e));
        }
    return 0;
}
