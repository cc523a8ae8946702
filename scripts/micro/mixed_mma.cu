// Diagnostic: does tcgen05.mma kind::f16 accept A = f16 (TMEM) with B = bf16 (SMEM)?
// And the issue rate of ex2.approx.f16x2 vs ex2.approx.f32.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

__host__ __device__ constexpr uint32_t idesc_mixed(uint32_t M, uint32_t N, uint32_t atype, uint32_t btype) {
    return (1u << 4) | (atype << 7) | (btype << 10) | (0u << 15) | (0u << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) k(float* out, uint32_t atype, uint32_t btype, uint16_t aval, uint16_t bval) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    uint16_t* b = reinterpret_cast<uint16_t*>(smem);
    for (int i = threadIdx.x; i < 16384; i += 128) b[i] = bval;   // B: 128 x 128, all bval
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<256>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    // A in TMEM cols [128, 192): row t = 128 elements = 64 packed columns, all aval
    uint32_t r[32];
    for (int x = 0; x < 32; ++x) r[x] = (uint32_t)aval | ((uint32_t)aval << 16);
    const uint32_t lane_base = (uint32_t)((threadIdx.x / 32) * 32) << 16;
    VMB_TMEM_ST32(tmem + lane_base + 128, r);
    VMB_TMEM_ST32(tmem + lane_base + 160, r);
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_mixed(128, 128, atype, btype);
        for (int kk = 0; kk < 8; ++kk)
            umma_ts(tmem, tmem + 128 + kk * 8, sdesc_sw128(smem_u32(smem) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), id, kk > 0);
        umma_commit(bar);
        mbar_wait(bar, 0);
    }
    __syncthreads();
    tc_fence_after();
    uint32_t o[32];
    VMB_TMEM_LD32(tmem + lane_base, o);
    tmem_ld_wait();
    out[threadIdx.x] = __uint_as_float(o[0]);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

__global__ void ex2rate(float* out, int iters, int mode) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.5f, a2 = a0 + 0.25f, a3 = a0 + 0.125f;
    uint32_t h0 = 0x3c003c00u, h1 = 0x38003800u, h2 = 0x34003400u, h3 = 0x30003000u;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
        } else if (mode == 1) {
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
        } else {
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + __uint_as_float(h0 ^ h1 ^ h2 ^ h3);
}

int main() {
    float* d; cudaMalloc(&d, 4 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    // f16 2.0 = 0x4000, bf16 3.0 = 0x4040, f16 3.0 = 0x4200, bf16 2.0 = 0x4000
    struct { uint32_t at, bt; uint16_t av, bv; const char* what; } cases[] = {
        {1, 1, 0x4000, 0x4040, "bf16 x bf16 (2*3*128 = 768 expected)"},
        {0, 0, 0x4000, 0x4200, "f16 x f16 (768 expected)"},

    };
    for (auto& c : cases) {
        k<<<1, 128, 40000>>>(d, c.at, c.bt, c.av, c.bv);
        float h[128];
        cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-48s -> %g %g (%s)\n", c.what, h[0], h[77], cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    for (int mode = 0; mode < 3; ++mode) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        ex2rate<<<148 * 8, 256>>>(d, 100, mode);
        cudaEventRecord(e0);
        const int iters = 4096;
        ex2rate<<<148 * 8, 256>>>(d, iters, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = 148.0 * 8 * 256 * iters * 4;
        printf("ex2 mode %d (%s): %.2f Gop/s per SM = %.2f ops/clk/SM @1.9GHz (instr count)\n", mode,
               mode == 0 ? "f32" : (mode == 1 ? "f16x2" : "bf16x2"), ops / (ms * 1e-3) / 148 / 1e9, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
    return 0;
}
