// Microbenchmark (diagnostic, not product): tcgen05.mma issue rate for the tile shapes the
// attention kernels use.  One CTA per SM (or two), one thread issues `iters` MMAs of shape
// M=128 x N x K=16 (bf16, f32 accumulate) back to back, A from SMEM or TMEM, B from SMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu && ./umma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

template <int N, bool A_TMEM, int NCTA_COLS, int NACC>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    // zero operands (values irrelevant)
    for (int i = threadIdx.x; i < (65536 + 32768) / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<NCTA_COLS>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        constexpr uint32_t id = idesc_bf16(128, N, 0, 0);
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t kk = i & 7;
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            const uint32_t d = tmem + (NACC > 1 ? (i % NACC) * N : 0);
            if (A_TMEM) umma_ts(d, tmem + 256 + kk * 8, sdesc_sw128(b + off, 16, 1024), id, 1);
            else umma_ss(d, sdesc_sw128(a + off, 16, 1024), sdesc_sw128(b + off, 16, 1024), id, 1);
        }
        umma_commit(bar);
        mbar_wait(bar, 0);
        unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<NCTA_COLS>(tmem); }
}

template <int N, bool A_TMEM, int NACC = 1>
void run(int ctas_per_sm) {
    const int iters = 8192;
    int sms = 148;
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms * 2);
    auto kern = k<N, A_TMEM, 512, NACC>;
    int smem = 65536 + 32768 + 64 + 1024;
    if (ctas_per_sm == 2) { smem = 100 * 1024; }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<sms, 128, smem>>>(64, d);
    cudaEventRecord(e0);
    kern<<<sms, 128, smem>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double flops = 2.0 * 128 * N * 16 * (double)iters * sms;
    printf("M=128 N=%3d K=16 nacc=%d A=%s : %.1f cycles/mma (SM clock), %.0f TFLOP/s chip, err=%s\n", N, NACC, A_TMEM ? "tmem" : "smem",
           (double)h[0] / iters, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<64, false>(1); run<128, false>(1); run<256, false>(1);
    run<64, true>(1); run<128, true>(1); run<256, true>(1);
    run<64, false, 2>(1); run<64, false, 4>(1); run<128, false, 2>(1);
    run<64, true, 4>(1); run<128, true, 2>(1);
    return 0;
}
