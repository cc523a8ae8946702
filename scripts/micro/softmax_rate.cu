// Microbenchmark (diagnostic, not product): issue/MUFU throughput of the softmax exponent pass
// of the attention kernels (per element pair: FFMA2 scale-and-shift, 2x MUFU.EX2 or the
// FMA-pipe polynomial, FADD2 row sum, F2FP bf16 pack, FMNMX3 running max), on register data,
// with W warps per SM sub-partition.  Reports cycles per 128x128 score tile per SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o softmax_rate softmax_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t x, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t x, uint64_t y) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
    return d;
}
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t ex2_emu2(uint64_t x2) {
    const uint64_t xx = pk2(fmaxf(lo2(x2), -126.f), fmaxf(hi2(x2), -126.f));
    const uint64_t t = fadd2(xx, pk2(12582912.f, 12582912.f));
    const uint64_t f = fadd2(xx, fadd2(pk2(-12582912.f, -12582912.f), t) ^ 0x8000000080000000ull);
    uint64_t p = ffma2(pk2(0.05592203512787819f, 0.05592203512787819f), f, pk2(0.24264007806777954f, 0.24264007806777954f));
    p = ffma2(p, f, pk2(0.6931210160255432f, 0.6931210160255432f));
    p = ffma2(p, f, pk2(0.9999244809150696f, 0.9999244809150696f));
    const uint32_t r0 = (uint32_t)p + ((uint32_t)t << 23);
    const uint32_t r1 = (uint32_t)(p >> 32) + ((uint32_t)(t >> 32) << 23);
    return (uint64_t)r0 | ((uint64_t)r1 << 32);
}

// ELEMS elements per thread per "tile" (128 = one row of a 128-key tile); EMU: one pair in EMU
// via the polynomial (EMU > ELEMS/2: none); MAXF: fused running max
template <int ELEMS, int EMU, bool MAXF>
__global__ void sm(int iters, float* out, unsigned long long* cyc) {
    uint32_t sr[ELEMS];
#pragma unroll
    for (int x = 0; x < ELEMS; ++x) sr[x] = __float_as_uint((float)((threadIdx.x * 7 + x * 13) % 97) * -0.01f);
    float m = -0.5f, l = 0.f, tm = -INFINITY;
    uint32_t sink = 0;
    const uint64_t sc = pk2(1.3f, 1.3f);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint64_t negm2 = pk2(-m, -m);
        const uint64_t* s2 = reinterpret_cast<const uint64_t*>(sr);
        uint64_t acc0 = 0, acc1 = 0;
        float t0m = -INFINITY, t1m = -INFINITY;
#pragma unroll
        for (int x = 0; x < ELEMS / 2; ++x) {
            const uint64_t sv = s2[x];
            if (MAXF) {
                if (x & 1) t1m = fmax3(t1m, lo2(sv), hi2(sv));
                else t0m = fmax3(t0m, lo2(sv), hi2(sv));
            }
            const uint64_t t2 = ffma2(sv, sc, negm2);
            uint64_t pp;
            if ((x % EMU) == EMU - 1) pp = ex2_emu2(t2);
            else pp = pk2(ex2(lo2(t2)), ex2(hi2(t2)));
            if (x & 1) acc1 = fadd2(acc1, pp);
            else acc0 = fadd2(acc0, pp);
            sink ^= pack_bf16(lo2(pp), hi2(pp));
        }
        const uint64_t acc = fadd2(acc0, acc1);
        l += lo2(acc) + hi2(acc);
        tm = fmaxf(tm, fmaxf(t0m, t1m));
        m += 1e-7f * l;  // loop-carried dependence: keeps the pass from being hoisted
    }
    unsigned long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = l + tm + (float)sink;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ELEMS, int EMU, bool MAXF>
void run(const char* name, int warps_per_smsp) {
    const int iters = 2000, threads = 128 * warps_per_smsp;
    float* o;
    unsigned long long* c;
    cudaMalloc(&o, 148 * threads * 4);
    cudaMalloc(&c, 148 * 8);
    sm<ELEMS, EMU, MAXF><<<148, threads>>>(10, o, c);
    sm<ELEMS, EMU, MAXF><<<148, threads>>>(iters, o, c);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    // per SMSP: warps_per_smsp warps x ELEMS elements x 32 rows each iteration; a 128x128 tile
    // is 32 rows x 128 elements per SMSP
    const double elems_per_smsp = (double)iters * warps_per_smsp * ELEMS * 32;
    printf("%-28s W=%d/SMSP: %7.1f cycles per 128x128 tile per SMSP  [%s]\n", name, warps_per_smsp,
           (double)h / (elems_per_smsp / (32.0 * 128)), cudaGetErrorString(cudaGetLastError()));
    cudaFree(o);
    cudaFree(c);
}

int main() {
    for (int w : {1, 2, 4}) {
        run<128, 1000, false>("128/thr mufu", w);
        run<128, 1000, true>("128/thr mufu+max", w);
        run<64, 1000, true>("64/thr mufu+max", w);
        run<128, 4, true>("128/thr emu 1/4 +max", w);
        run<128, 3, true>("128/thr emu 1/3 +max", w);
        run<128, 2, true>("128/thr emu 1/2 +max", w);
    }
    return 0;
}
