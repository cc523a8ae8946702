// Microbenchmark (diagnostic, not product): the memory pattern of the L half-step at C4 with no
// compute.  Per spatial position i of unit u: TMA-load Qb[i] (m rows of 256 B at a b*256-B
// stride) and aL[i] (m*256 B contiguous), optionally spin DELAY ns (a stand-in for the
// MMA -> softmax -> MMA -> epilogue chain), then TMA-store the Qb tile to aR[i] (strided, as
// the product kernel does).  3 * U*N*256 B move per launch.  Variants:
//   NPOS   positions per CTA (1, 2, 4), boxes position-major in smem (dims reordered so each
//          position's rows stay contiguous, as the MMA descriptors need)
//   RING   0: one tile set per CTA (non-persistent, grid = positions / NPOS)
//          S>0: persistent, 148*CPS CTAs looping over positions with an S-stage ring
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lstep_bw lstep_bw.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2601_22275_b200/csrc/kernels/sm100_ptx.cuh"
using namespace vmb::ptx;

struct Args {
    CUtensorMap tmQ, tmAL, tmOut;
    int b, U, R, npos_total;
    long long delay_ns;
};

__device__ __forceinline__ void spin(long long ns) {
    if (ns <= 0) return;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint64_t t1 = t0;
    while ((long long)(t1 - t0) < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
}

// one tile set = NPOS positions: Qb [pos][2 panels][R rows][128 B], aL the same
template <int NPOS>
__device__ __forceinline__ void issue_loads(const Args& a, uint8_t* base, uint64_t* bar, int i0, int u) {
    const uint32_t panel = (uint32_t)a.R * 128u;
    mbar_arrive_expect_tx(bar, 4u * panel * NPOS);
    // Q map dims (64-col, j, i, 1, u); box (64, R, NPOS)
    tma_load_5d(base, &a.tmQ, bar, 0, 0, i0, 0, u);
    tma_load_5d(base + NPOS * panel, &a.tmQ, bar, 64, 0, i0, 0, u);
    uint8_t* al = base + 2 * NPOS * panel;
    tma_load_5d(al, &a.tmAL, bar, 0, 0, i0, 0, u);
    tma_load_5d(al + NPOS * panel, &a.tmAL, bar, 64, 0, i0, 0, u);
}

template <int NPOS>
__device__ __forceinline__ void issue_store(const Args& a, uint8_t* base, int i0, int u) {
    const uint32_t panel = (uint32_t)a.R * 128u;
    tma_store_5d(&a.tmOut, base, 0, 0, i0, 0, u);
    tma_store_5d(&a.tmOut, base + NPOS * panel, 64, 0, i0, 0, u);
    tma_store_commit();
}

template <int NPOS>
__global__ void __launch_bounds__(128) oneshot(const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t set = 4u * a.R * 128u * NPOS;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + set);
    const int i0 = blockIdx.x * NPOS, u = blockIdx.y;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        issue_loads<NPOS>(a, smem, bar, i0, u);
        mbar_wait(bar, 0);
        spin(a.delay_ns);
        issue_store<NPOS>(a, smem, i0, u);
        tma_store_wait_read();
    }
    __syncthreads();
}

template <int NPOS, int S>
__global__ void __launch_bounds__(128) ring(const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t set = 4u * a.R * 128u * NPOS;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * set);
    const int per_u = a.b / NPOS;
    const int items = per_u * a.U;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        int it = blockIdx.x, n = 0;
        // prologue
        for (int s = 0; s < S && it + s * (int)gridDim.x < items; ++s) {
            const int x = it + s * gridDim.x;
            issue_loads<NPOS>(a, smem + s * set, &full[s], (x % per_u) * NPOS, x / per_u);
        }
        for (; it < items; it += gridDim.x, ++n) {
            const int s = n % S;
            mbar_wait(&full[s], (n / S) & 1);
            spin(a.delay_ns);
            issue_store<NPOS>(a, smem + s * set, (it % per_u) * NPOS, it / per_u);
            const int nx = it + S * gridDim.x;
            if (nx < items) {
                tma_store_wait_read();  // slot reusable once the store has read it
                issue_loads<NPOS>(a, smem + s * set, &full[s], (nx % per_u) * NPOS, nx / per_u);
            }
        }
        tma_store_wait_read();
    }
    __syncthreads();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap map5(void* base, cuuint64_t d1, cuuint64_t d2, cuuint64_t d4, cuuint64_t s1, cuuint64_t s2,
                        cuuint64_t s4, cuuint32_t b1, cuuint32_t b2) {
    CUtensorMap m;
    cuuint64_t dims[5] = {128, d1, d2, 1, d4};
    cuuint64_t strides[4] = {s1, s2, s4, s4};
    cuuint32_t box[5] = {64, b1, b2, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

int main() {
    const int U = 40, m = 81, b = 1456, R = 96;
    const long long N = (long long)m * b;
    const size_t bytes = (size_t)U * N * 256;
    void *q, *al, *out, *flush;
    cudaMalloc(&q, bytes);
    cudaMalloc(&al, bytes);
    cudaMalloc(&out, bytes);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(q, 0, bytes);
    cudaMemset(al, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double moved = 3.0 * U * N * 256;
    auto bench = [&](const char* name, auto launch) {
        float best = 1e30f, sum = 0;
        const int reps = 5;
        for (int r = 0; r < reps + 1; ++r) {
            cudaMemsetAsync(flush, r, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r) { best = ms < best ? ms : best; sum += ms; }
        }
        cudaError_t err = cudaGetLastError();
        printf("%-44s best %.3f ms  mean %.3f ms  %.0f GB/s%s\n", name, best, sum / reps, moved / best / 1e6,
               err ? cudaGetErrorString(err) : "");
    };
    for (int al_fm : {0, 1})
    for (long long delay : {0LL, 1000LL, 2000LL, 4000LL}) {
        printf("--- delay %lld ns, aL %s\n", delay, al_fm ? "frame-major (U,m,b,d)" : "position-major (U,b,m,d)");
        auto mk = [&](int npos) {
            Args a;
            // Q / out: (64-col, j: m @ b*256, i: b @ 256, u @ N*256), box (64, R, npos)
            a.tmQ = map5(q, m, b, U, (cuuint64_t)b * 256, 256, (cuuint64_t)N * 256, R, npos);
            a.tmOut = map5(out, m, b, U, (cuuint64_t)b * 256, 256, (cuuint64_t)N * 256, R, npos);
            // aL (U, b, m, d): (64-col, k: m @ 256, i: b @ m*256, u)
            a.tmAL = al_fm ? map5(al, m, b, U, (cuuint64_t)b * 256, 256, (cuuint64_t)N * 256, R, npos)
                           : map5(al, m, b, U, 256, (cuuint64_t)m * 256, (cuuint64_t)N * 256, R, npos);
            a.b = b; a.U = U; a.R = R; a.npos_total = b * U; a.delay_ns = delay;
            return a;
        };
        auto one = [&](auto kern, int npos, int ctas_per_sm, const char* nm) {
            Args a = mk(npos);
            int smem = 4 * R * 128 * npos + 1024 + 64;
            int need = 227 * 1024 / ctas_per_sm - 1024;
            if (need > smem) smem = need;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            char buf[96];
            snprintf(buf, sizeof buf, "%s cps=%d", nm, ctas_per_sm);
            bench(buf, [&] { kern<<<dim3(b / npos, U), 128, smem>>>(a); });
        };
        one(oneshot<1>, 1, 4, "oneshot npos=1");
        one(oneshot<1>, 1, 8, "oneshot npos=1");
        one(oneshot<2>, 2, 2, "oneshot npos=2");
        one(oneshot<2>, 2, 4, "oneshot npos=2");
        one(oneshot<4>, 4, 2, "oneshot npos=4");
        auto rg = [&](auto kern, int npos, int S, int cps, const char* nm) {
            Args a = mk(npos);
            int smem = S * 4 * R * 128 * npos + 1024 + 64;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            char buf[96];
            snprintf(buf, sizeof buf, "%s cps=%d", nm, cps);
            bench(buf, [&] { kern<<<148 * cps, 128, smem>>>(a); });
        };
        rg(ring<1, 2>, 1, 2, 2, "ring npos=1 S=2");
        rg(ring<1, 4>, 1, 4, 1, "ring npos=1 S=4");
        rg(ring<2, 2>, 2, 2, 1, "ring npos=2 S=2");
        rg(ring<1, 3>, 1, 3, 1, "ring npos=1 S=3");
    }
    return 0;
}
