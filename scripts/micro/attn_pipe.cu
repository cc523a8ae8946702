// Microbenchmark (diagnostic, not product): the MMA + TMA pipeline of the attention kernels
// with no softmax, to find what bounds it.  One CTA per SM streams 128-key tiles from L2
// through a TMA ring; the MMA thread issues per tile S = Q K^T (M=128, N=128, K=d=128) and
// O += P [K|V] (P read from TMEM, as in the product kernels).  The variants differ in where
// the S MMA's A operand (Q) lives -- shared memory (SS, as in fa2/fa3/fa4) or TMEM (TS) --
// and in the value operand (V = K for the R half-step, separate V, or [K | V] N = 256).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o attn_pipe attn_pipe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

constexpr int kPanel = 128 * 128;          // 128 rows x 64 bf16
constexpr int kTile = 2 * kPanel;          // 128 x 128 bf16

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
                 : "memory");
}

// VMODE 0: V = K (R half-step), PV N = 128 over the K tile
// VMODE 1: separate V tile, PV N = 128
// VMODE 2: [K | V], PV N = 256
template <int VMODE, bool Q_TMEM, int STAGES>
__global__ void __launch_bounds__(128, 1) pipe(const __grid_constant__ CUtensorMap mk, int tiles, int rows_total,
                                               unsigned long long* cyc) {
    constexpr int NB = VMODE == 0 ? 1 : 2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sq = smem;
    uint8_t* skv = smem + kTile;
    uint64_t* full = reinterpret_cast<uint64_t*>(skv + STAGES * NB * kTile);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
    for (int i = threadIdx.x; i < kTile / 16; i += 128) reinterpret_cast<uint4*>(sq)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<512>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const int row0 = (int)((blockIdx.x * 977ull) % (unsigned)(rows_total / 128 - tiles * NB)) * 128;
    if (threadIdx.x < 32) {
        if (elect_one()) {
            for (int t = 0; t < tiles; ++t) {
                const int st = t % STAGES;
                if (t >= STAGES) mbar_wait(&empty[st], ((t / STAGES) - 1) & 1);
                mbar_arrive_expect_tx(&full[st], NB * kTile);
                uint8_t* dst = skv + st * NB * kTile;
                for (int b = 0; b < NB; ++b) {
                    tma2d(dst + b * kTile, &mk, &full[st], 0, row0 + (t * NB + b) * 128);
                    tma2d(dst + b * kTile + kPanel, &mk, &full[st], 64, row0 + (t * NB + b) * 128);
                }
            }
        }
    } else if (threadIdx.x < 64) {
        if (elect_one()) {
            constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t idPV = idesc_bf16(128, VMODE == 2 ? 256 : 128, 0, 1);
            const uint32_t qa = smem_u32(sq), kva = smem_u32(skv);
            const uint32_t tS = tmem, tQ = tmem + 128, tO = tmem + 256;
            unsigned long long t0 = clock64();
            for (int t = 0; t < tiles; ++t) {
                const int st = t % STAGES;
                mbar_wait(&full[st], (t / STAGES) & 1);
                tc_fence_after();
                const uint32_t ka = kva + st * NB * kTile;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
                    if (Q_TMEM) umma_ts(tS, tQ + kk * 8, sdesc_sw128(ka + off, 16, 1024), idS, kk > 0);
                    else umma_ss(tS, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(ka + off, 16, 1024), idS, kk > 0);
                }
                const uint32_t va = ka + (VMODE == 1 ? kTile : 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_ts(tO, tS + kk * 8, sdesc_sw128(va + kk * 2048, kPanel, 1024), idPV, 1u);
                umma_commit(&empty[st]);
            }
            umma_commit(done);
            mbar_wait(done, 0);
            cyc[blockIdx.x] = clock64() - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int VMODE, bool Q_TMEM, int STAGES>
void run(const char* name, void* buf, int rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    constexpr int NB = VMODE == 0 ? 1 : 2;
    const int smem = kTile + STAGES * NB * kTile + 1024 + 256;
    auto kern = pipe<VMODE, Q_TMEM, STAGES>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int tiles = 2048;
    kern<<<148, 128, smem>>>(m, 64, rows, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<148, 128, smem>>>(m, tiles, rows, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148;
    const double flop_tile = 2.0 * 128 * 128 * 128 + 2.0 * 128 * (VMODE == 2 ? 256 : 128) * 128;
    const double ideal = 512 + (VMODE == 2 ? 1024 : 512);
    printf("%-34s: %6.0f cycles/tile (ideal %4.0f, %.0f%%), %5.0f TFLOP/s chip, smem stages %d  [%s]\n", name,
           avg / tiles, ideal, 100.0 * ideal / (avg / tiles), flop_tile * tiles * 148 / (ms * 1e-3) / 1e12, STAGES,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    const int rows = 1 << 18;  // 64 MB of bf16 rows: L2-resident streams, as the product kernels see
    void* buf;
    cudaMalloc(&buf, (size_t)rows * 256);
    cudaMemset(buf, 0, (size_t)rows * 256);
    run<0, false, 4>("V=K     S:SS  (fa2-like)", buf, rows);
    run<0, true, 4>("V=K     S:TS  (Q in TMEM)", buf, rows);
    run<1, false, 3>("V sep   S:SS  (fa3-like, 1 Q)", buf, rows);
    run<1, true, 3>("V sep   S:TS  (Q in TMEM)", buf, rows);
    run<2, false, 3>("[K|V]   S:SS  (fa4-like, N=256)", buf, rows);
    run<2, true, 3>("[K|V]   S:TS  (Q in TMEM, N=256)", buf, rows);
    run<0, false, 6>("V=K     S:SS  6 stages", buf, rows);
    run<0, true, 6>("V=K     S:TS  6 stages", buf, rows);
    return 0;
}
