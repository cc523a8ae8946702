// Diagnostic: tcgen05.ld / tcgen05.st throughput (32x32b.x32) per SM with 4 or 8 warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

template <int WARPS, bool STORE>
__global__ void __launch_bounds__(WARPS * 32, 1) k(int iters, float* out) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int warp = threadIdx.x / 32;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col = (warp / 4) * 128;
    uint32_t r[32];
    for (int x = 0; x < 32; ++x) r[x] = x;
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        const uint32_t c = col + (i & 3) * 32;
        if (STORE) {
            VMB_TMEM_ST32(tmem + lane_base + c, r);
            tmem_st_wait();
        } else {
            VMB_TMEM_LD32(tmem + lane_base + c, r);
            tmem_ld_wait();
            acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int WARPS, bool STORE>
void run() {
    float* d; cudaMalloc(&d, 148 * 1024 * 4);
    const int iters = 20000;
    k<WARPS, STORE><<<148, WARPS * 32>>>(100, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<WARPS, STORE><<<148, WARPS * 32>>>(iters, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)WARPS * 32 * 32 * 4 * iters;  // per SM
    printf("%s warps=%d: %.1f B/clk/SM @1.9GHz (%.1f GB/s per SM) err=%s\n", STORE ? "STTM.x32" : "LDTM.x32", WARPS,
           bytes / (ms * 1e-3) / 1.9e9, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}
int main() { run<4, false>(); run<8, false>(); run<16, false>(); run<4, true>(); run<8, true>(); return 0; }
