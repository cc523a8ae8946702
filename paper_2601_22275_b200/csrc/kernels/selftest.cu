// selftest.cu — unit test of the tcgen05 / TMA building blocks used by fa_tc.cu and
// lstep_tc.cu (descriptor encodings, swizzle, TMEM A-operand layout).  Exposed through
// vmb_selftest_umma() for tests/test_gpu_primitives.py.
//   mode 0: C = A * B^T   (A, B K-major: S = Q K^T)
//   mode 1: C = A * B     (B MN-major:    O = P V with P in smem)
//   mode 2: C = A * B     (A staged in TMEM as packed bf16, B MN-major: O += P V)
//   mode 3: C = A^T * B   (A MN-major: aR = L^T Qb)
#include <cuda_bf16.h>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;
constexpr uint32_t kPanel = 128 * 128;

struct Params {
    CUtensorMap tmA, tmB;
    const __nv_bfloat16* A;
    float* C;
    int mode;
};

__global__ void __launch_bounds__(128) selftest_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint8_t* sA = smem;
    uint8_t* sB = smem + 2 * kPanel;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * kPanel);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 4 * kPanel + 64);
    const int warp = warp_id(), t = threadIdx.x;
    if (warp == 0) {
        if (elect_one()) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<256>(slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;

    if (p.mode == 2) {
        // thread t writes row t of A (128 bf16) into TMEM columns [128, 192) as bf16 pairs
        const uint32_t* arow = reinterpret_cast<const uint32_t*>(p.A + t * 128);
        uint32_t r[32];
#pragma unroll
        for (int x = 0; x < 32; ++x) r[x] = arow[x];
        VMB_TMEM_ST32(tmem + lane_base + 128, r);
#pragma unroll
        for (int x = 0; x < 32; ++x) r[x] = arow[32 + x];
        VMB_TMEM_ST32(tmem + lane_base + 160, r);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0 && elect_one()) {
        mbar_arrive_expect_tx(bar, 4 * kPanel);
        tma_load_5d(sA, &p.tmA, bar, 0, 0, 0, 0, 0);
        tma_load_5d(sA + kPanel, &p.tmA, bar, 64, 0, 0, 0, 0);
        tma_load_5d(sB, &p.tmB, bar, 0, 0, 0, 0, 0);
        tma_load_5d(sB + kPanel, &p.tmB, bar, 64, 0, 0, 0, 0);
        mbar_wait(bar, 0);
        tc_fence_after();
        const uint32_t a = smem_u32(sA), b = smem_u32(sB);
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t koff = (kk >> 2) * kPanel + (kk & 3) * 32;
            if (p.mode == 0) {
                umma_ss(tmem, sdesc_sw128(a + koff, 16, 1024), sdesc_sw128(b + koff, 16, 1024),
                        idesc_bf16(128, 128, 0, 0), kk > 0);
            } else if (p.mode == 1) {
                umma_ss(tmem, sdesc_sw128(a + koff, 16, 1024),
                        sdesc_sw128(b + kk * 2048, kPanel, 1024), idesc_bf16(128, 128, 0, 1), kk > 0);
            } else if (p.mode == 2) {
                umma_ts(tmem, tmem + 128 + kk * 8, sdesc_sw128(b + kk * 2048, kPanel, 1024),
                        idesc_bf16(128, 128, 0, 1), kk > 0);
            } else {
                umma_ss(tmem, sdesc_sw128(a + kk * 2048, kPanel, 1024),
                        sdesc_sw128(b + kk * 2048, kPanel, 1024), idesc_bf16(128, 128, 1, 1), kk > 0);
            }
        }
        umma_commit(bar + 1);
    }
    __syncwarp();
    mbar_wait(bar + 1, 0);
    tc_fence_after();
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t r[32];
        VMB_TMEM_LD32(tmem + lane_base + cc * 32, r);
        tmem_ld_wait();
        for (int x = 0; x < 32; ++x) p.C[t * 128 + cc * 32 + x] = __uint_as_float(r[x]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

}  // namespace

void selftest_umma(int mode, const void* A, const void* B, float* C, cudaStream_t s) {
    Params p;
    const uint64_t dims[5] = {128, 128, 1, 1, 1};
    const uint64_t strides[4] = {256, 256 * 128, 256 * 128, 256 * 128};
    const uint32_t box[5] = {64, 128, 1, 1, 1};
    p.tmA = make_tmap_bf16_5d(A, dims, strides, box);
    p.tmB = make_tmap_bf16_5d(B, dims, strides, box);
    p.A = static_cast<const __nv_bfloat16*>(A);
    p.C = C;
    p.mode = mode;
    const size_t smem = 4 * kPanel + 128 + 1024;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    selftest_kernel<<<1, 128, smem, s>>>(p);
    count_launch();
    check_launch("selftest_umma");
}

}  // namespace vmb
