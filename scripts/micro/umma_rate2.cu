// Microbenchmark (diagnostic, not product): tcgen05.mma throughput with the issue loop the
// product kernels use -- descriptors in uniform registers, 8 MMAs (one K=128 chunk) unrolled
// per loop trip -- for cta_group::1 (M=128) and cta_group::2 (M=256 over a CTA pair).
// umma_rate.cu (round 1) issued from a thread-0 branch, which compiles to a per-MMA
// R2UR.BROADCAST waterfall loop; this version checks whether its ~80-cycle floor was issue cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate2 umma_rate2.cu && ./umma_rate2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

template <int CG, int N, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) k(int trips, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    for (int i = threadIdx.x; i < 131072 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (CG == 2) cluster_sync();
    if (threadIdx.x < 32) {
        if (CG == 1) {
            tmem_alloc<512>(slot);
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x < 32 && rank == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
        constexpr uint32_t id = idesc_bf16(128 * CG, N, 0, 0);
        if (elect_one()) {
            unsigned long long t0 = clock64();
            for (int t = 0; t < trips; ++t) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    if (CG == 1) {
                        if (A_TMEM) umma_ts(tmem, tmem + 256 + kk * 8, sdesc_sw128(b + off, 16, 1024), id, 1);
                        else umma_ss(tmem, sdesc_sw128(a + off, 16, 1024), sdesc_sw128(b + off, 16, 1024), id, 1);
                    } else {
                        if (A_TMEM) mma2_ts(tmem, tmem + 256 + kk * 8, sdesc_sw128(b + off, 16, 1024), id, 1);
                        else mma2_ss(tmem, sdesc_sw128(a + off, 16, 1024), sdesc_sw128(b + off, 16, 1024), id, 1);
                    }
                }
            }
            if (CG == 1) {
                umma_commit(bar);
            } else {
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                             ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
            }
            mbar_wait(bar, 0);
            cyc[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    } else if (CG == 2 && threadIdx.x == 0) {
        mbar_wait(bar, 0);  // the leader's commit arrives here too
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    if (threadIdx.x < 32) {
        tc_fence_after();
        if (CG == 1) tmem_dealloc<512>(tmem);
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

template <int CG, int N, bool A_TMEM>
void run() {
    const int trips = 2048;
    const int sms = 148;
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    cudaMemset(d, 0, sizeof(unsigned long long) * sms);
    auto kern = k<CG, N, A_TMEM>;
    const int smem = 131072 + 64 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, kern, 16, d);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, kern, trips, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double mmas = 8.0 * trips;
    // work per SM per instruction: 128 x N x 16 (cta_group::2: each SM of the pair does 128 rows)
    const double flops = 2.0 * 128 * N * 16 * mmas * sms;
    printf("cta_group::%d M=%d N=%3d A=%s : %.1f cycles/instr (issuer clock), %.0f TFLOP/s chip  [%s]\n", CG, 128 * CG, N,
           A_TMEM ? "tmem" : "smem", (double)h[0] / mmas, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<1, 64, false>(); run<1, 128, false>(); run<1, 256, false>();
    run<1, 64, true>(); run<1, 128, true>(); run<1, 256, true>();
    run<2, 64, false>(); run<2, 128, false>(); run<2, 256, false>();
    run<2, 128, true>(); run<2, 256, true>();
    return 0;
}
