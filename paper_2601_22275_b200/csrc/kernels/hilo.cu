// hilo.cu — the fp32 parity mode's operand split for the tensor cores: x = hi + lo with
// hi = bf16(x) and lo = bf16(x - hi) (16 mantissa bits together), written as two contiguous
// (U, rows, d) bf16 tensors.  HBM-bound: 4 B read, 4 B written per element.
#include <cuda_bf16.h>

#include "../internal.hpp"

namespace vmb {
namespace {

// one thread per 4 consecutive head-dim elements of a row (u, t): float4 in, 2 x 8 B out
__global__ void __launch_bounds__(256) split_hilo_kernel(View v, int64_t U, int64_t rows, int64_t d,
                                                          __nv_bfloat16* hi, __nv_bfloat16* lo) {
    const int64_t q = d / 4;
    const int64_t total = U * rows * q;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = (e % q) * 4, r = e / q;
        const int64_t t = r % rows, u = r / rows;
        const float* src = static_cast<const float*>(v.base) + (u / v.H) * v.sB + (u % v.H) * v.sH + t * v.sc + x;
        const float4 f = *reinterpret_cast<const float4*>(src);
        const __nv_bfloat162 h01 = __floats2bfloat162_rn(f.x, f.y), h23 = __floats2bfloat162_rn(f.z, f.w);
        const __nv_bfloat162 l01 = __floats2bfloat162_rn(f.x - __low2float(h01), f.y - __high2float(h01));
        const __nv_bfloat162 l23 = __floats2bfloat162_rn(f.z - __low2float(h23), f.w - __high2float(h23));
        uint2 ho, lw;
        ho.x = *reinterpret_cast<const uint32_t*>(&h01);
        ho.y = *reinterpret_cast<const uint32_t*>(&h23);
        lw.x = *reinterpret_cast<const uint32_t*>(&l01);
        lw.y = *reinterpret_cast<const uint32_t*>(&l23);
        *reinterpret_cast<uint2*>(hi + r * d + x) = ho;
        *reinterpret_cast<uint2*>(lo + r * d + x) = lw;
    }
}

__global__ void __launch_bounds__(256) merge_hilo_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, float* out,
                                                          int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = __bfloat162float(hi[e]) + __bfloat162float(lo[e]);
}

}  // namespace

void merge_hilo(const void* hi, const void* lo, float* out, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    merge_hilo_kernel<<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(hi), static_cast<const __nv_bfloat16*>(lo),
                                             out, n);
    count_launch();
    check_launch("merge_hilo");
}

void split_hilo(const View& v, int64_t U, int64_t rows, int64_t d, void* hi, void* lo, cudaStream_t s) {
    const int64_t total = U * rows * (d / 4);
    if (total == 0) return;
    VMB_REQUIRE_DIM(d % 4 == 0, "hi/lo split needs d % 4 == 0");
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    ProfScope ps(kKSimt, s);  // timed with the CUDA-core kernels
    split_hilo_kernel<<<blocks, 256, 0, s>>>(v, U, rows, d, static_cast<__nv_bfloat16*>(hi),
                                             static_cast<__nv_bfloat16*>(lo));
    count_launch();
    check_launch("split_hilo");
}

}  // namespace vmb
