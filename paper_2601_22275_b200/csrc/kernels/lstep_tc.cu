// lstep_tc.cu — tcgen05 L half-step and the permutation-folded Monarch apply (bf16, d = 128,
// m <= 128).
//
// One CTA per (unit u, spatial position i).  Reference semantics (monarch.hpp:105-147):
//   S[j,k]  = <Qb[i,j], aL[i,k]> * qscale - cL[i,k]        GEMM 1 (M=j, N=k, K=d)
//   L[j,:]  = softmax_k(S[j,:])                             thread j owns row j (TMEM lane j)
//   ITER : cR[k,i] = sum_j L[j,k]                           column sums from the smem copy of L
//          aR[k,i] = sum_j L[j,k] Qb[i,j]                   GEMM 2 (M=k, N=d, K=j): A = L^T
//                                                           read MN-major from the same tile
//   FINAL: O[j*b+i] = sum_k L[j,k] y[k,i]                   GEMM 2 (M=j, N=d, K=k), the
//          assembly of monarch.hpp:187-190 with the reshape-transpose permutation folded
//          into the TMA coordinates of Qb / y and the row address of O.
// Qb[i] rows are the tokens j*b+i of Q (stride b*d): a (d, i, j) box of the 5-D TMA map,
// so no permuted copy of Q ever exists (mat.hpp:99-113 / perm.hpp:19-50 are addressing only).
//
// Memory-bound stage: per i it reads Qb, aL (+ y) and writes aR (or O).
#include <cuda_bf16.h>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 128;
constexpr uint32_t kPanel = 128 * 128;     // 128 rows x 64 bf16, SW128
constexpr uint32_t kTileB = 2 * kPanel;    // 128 x 128 bf16

struct Params {
    TcLstepArgs a;
};

template <bool FINAL>
struct Smem {
    static constexpr uint32_t qb = 0;
    static constexpr uint32_t al = kTileB;                  // aL, later overwritten by L
    static constexpr uint32_t y = 2 * kTileB;               // FINAL only
    static constexpr uint32_t cl = (FINAL ? 3 : 2) * kTileB;  // 128 floats
    static constexpr uint32_t bars = cl + 512;
    static constexpr uint32_t slot = bars + 32;
    static constexpr uint32_t bytes = slot + 16;
    static constexpr uint32_t alloc = bytes + 1024;
};

template <bool FINAL>
__global__ void __launch_bounds__(kThreads) lstep_tc_kernel(const __grid_constant__ Params p) {
    using SM = Smem<FINAL>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar_load = reinterpret_cast<uint64_t*>(smem + SM::bars);
    uint64_t* bar_mma1 = bar_load + 1;
    uint64_t* bar_mma2 = bar_load + 2;
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + SM::slot);
    float* s_cl = reinterpret_cast<float*>(smem + SM::cl);

    const TcLstepArgs& a = p.a;
    const int i = blockIdx.x, u = blockIdx.y;
    const int m = a.m;
    const int warp = warp_id();
    const int t = threadIdx.x;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t n_pad = (uint32_t)((m + 15) & ~15);     // GEMM-1 N and GEMM-2 K extent

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch_desc(&a.tmQ);
            tma_prefetch_desc(&a.tmAL);
            if (FINAL) tma_prefetch_desc(&a.tmY);
            mbar_init(bar_load, 1);
            mbar_init(bar_mma1, 1);
            mbar_init(bar_mma2, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<128>(slot);
    }
    // cL[i, 0..m) -> smem (all rows of this block share it)
    const float* cl = a.cL + ((int64_t)u * a.b + i) * m;
    for (int k = t; k < 128; k += kThreads) s_cl[k] = (k < m) ? cl[k] : 0.f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;

    const uint32_t qb_addr = smem_u32(smem + SM::qb);
    const uint32_t al_addr = smem_u32(smem + SM::al);
    const uint32_t y_addr = smem_u32(smem + SM::y);
    const bool leader = (warp == 0) && elect_one();

    if (leader) {
        const int qbb = u / a.H, qh = u % a.H;
        mbar_arrive_expect_tx(bar_load, (FINAL ? 3 : 2) * kTileB);
        tma_load_5d(smem + SM::qb, &a.tmQ, bar_load, 0, i, 0, qh, qbb);
        tma_load_5d(smem + SM::qb + kPanel, &a.tmQ, bar_load, 64, i, 0, qh, qbb);
        tma_load_5d(smem + SM::al, &a.tmAL, bar_load, 0, 0, i, 0, u);
        tma_load_5d(smem + SM::al + kPanel, &a.tmAL, bar_load, 64, 0, i, 0, u);
        if (FINAL) {
            tma_load_5d(smem + SM::y, &a.tmY, bar_load, 0, i, 0, 0, u);
            tma_load_5d(smem + SM::y + kPanel, &a.tmY, bar_load, 64, i, 0, 0, u);
        }
        mbar_wait(bar_load, 0);
        tc_fence_after();
        const uint32_t id1 = idesc_bf16(128, n_pad, 0, 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
            umma_ss(tmem, sdesc_sw128(qb_addr + off, 16, 1024), sdesc_sw128(al_addr + off, 16, 1024),
                    id1, kk > 0);
        }
        umma_commit(bar_mma1);
    }
    __syncwarp();

    // ---- softmax of row j = t over k < m   (monarch.hpp:124-138)
    mbar_wait(bar_mma1, 0);
    tc_fence_after();
    uint32_t sr[128];
    VMB_TMEM_LD32(tmem + lane_base + 0, (sr + 0));
    VMB_TMEM_LD32(tmem + lane_base + 32, (sr + 32));
    VMB_TMEM_LD32(tmem + lane_base + 64, (sr + 64));
    VMB_TMEM_LD32(tmem + lane_base + 96, (sr + 96));
    tmem_ld_wait();
    float* s = reinterpret_cast<float*>(sr);
    const bool row_valid = t < m;
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < 128; ++k) {
        s[k] = (k < m) ? fmaf(s[k], a.qscale, -s_cl[k]) : -INFINITY;
        mx = fmaxf(mx, s[k]);
    }
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < 128; ++k) {
        s[k] = (k < m) ? __expf(s[k] - mx) : 0.f;
        sum += s[k];
    }
    const float inv = row_valid ? 1.f / sum : 0.f;
    // L row j -> bf16, SW128 layout, overwriting aL (GEMM 1 has consumed it)
    uint8_t* lt = smem + SM::al;
#pragma unroll
    for (int c8 = 0; c8 < 16; ++c8) {
        uint4 v;
        v.x = pack_bf16(s[8 * c8 + 0] * inv, s[8 * c8 + 1] * inv);
        v.y = pack_bf16(s[8 * c8 + 2] * inv, s[8 * c8 + 3] * inv);
        v.z = pack_bf16(s[8 * c8 + 4] * inv, s[8 * c8 + 5] * inv);
        v.w = pack_bf16(s[8 * c8 + 6] * inv, s[8 * c8 + 7] * inv);
        *reinterpret_cast<uint4*>(lt + (c8 >> 3) * kPanel + sw128_offset(t, (c8 & 7) * 8)) = v;
    }
    fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (leader) {
        if (!FINAL) {
            // aR' = L^T [Qb]: A = L^T (M=k, K=j) MN-major, B = Qb (K=j, N=d) MN-major
            const uint32_t id2 = idesc_bf16(128, 128, 1, 1);
            for (uint32_t kk = 0; kk < n_pad / 16; ++kk)
                umma_ss(tmem, sdesc_sw128(al_addr + kk * 2048, kPanel, 1024),
                        sdesc_sw128(qb_addr + kk * 2048, kPanel, 1024), id2, kk > 0);
        } else {
            // O_i = L Y: A = L (M=j, K=k) K-major, B = Y (K=k, N=d) MN-major
            const uint32_t id2 = idesc_bf16(128, 128, 0, 1);
            for (uint32_t kk = 0; kk < n_pad / 16; ++kk) {
                const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
                umma_ss(tmem, sdesc_sw128(al_addr + off, 16, 1024),
                        sdesc_sw128(y_addr + kk * 2048, kPanel, 1024), id2, kk > 0);
            }
        }
        umma_commit(bar_mma2);
    }
    __syncwarp();

    if (!FINAL && t < m) {
        // cR[k,i] = sum_j L[j,k]  (monarch.hpp:139-143), k = t, from the bf16 copy of L
        float col = 0.f;
        const uint8_t* base = lt + (t >> 6) * kPanel;
        for (int j = 0; j < m; ++j)
            col += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(base + sw128_offset(j, t & 63)));
        a.cR[((int64_t)u * m + t) * a.b + i] = col;
    }

    // ---- epilogue: TMEM row t -> aR[k=t, i] or O[j=t, i]
    mbar_wait(bar_mma2, 0);
    tc_fence_after();
    __nv_bfloat16* dst = nullptr;
    float scale = 1.f;
    bool store = t < m;
    if (!FINAL) {
        dst = a.aR + (((int64_t)u * m + t) * a.b + i) * 128;
        scale = a.ar_scale;
    } else {
        const int64_t ob = u / a.oHn, oh = u % a.oHn;
        dst = a.O + ob * a.oB + oh * a.oH + (int64_t)t * a.oJ + (int64_t)i * a.oI;
        store = store && !(a.skip_j0 && t == 0);
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t orr[32];
        VMB_TMEM_LD32(tmem + lane_base + cc * 32, orr);
        tmem_ld_wait();
        if (store) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                uint4 v;
                v.x = pack_bf16(__uint_as_float(orr[8 * x + 0]) * scale, __uint_as_float(orr[8 * x + 1]) * scale);
                v.y = pack_bf16(__uint_as_float(orr[8 * x + 2]) * scale, __uint_as_float(orr[8 * x + 3]) * scale);
                v.z = pack_bf16(__uint_as_float(orr[8 * x + 4]) * scale, __uint_as_float(orr[8 * x + 5]) * scale);
                v.w = pack_bf16(__uint_as_float(orr[8 * x + 6]) * scale, __uint_as_float(orr[8 * x + 7]) * scale);
                d4[x] = v;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

template <bool FINAL>
void launch(const Params& p, int64_t U, cudaStream_t s) {
    using SM = Smem<FINAL>;
    auto kern = lstep_tc_kernel<FINAL>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    dim3 grid((unsigned)p.a.b, (unsigned)U);
    ProfScope ps(FINAL ? kKLfinal : kKLstep, s);
    kern<<<grid, kThreads, SM::alloc, s>>>(p);
    count_launch();
    check_launch("lstep_tc");
}

}  // namespace

void tc_lstep_launch(const TcLstepArgs& a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.b == 0) return;
    VMB_REQUIRE_DIM(a.m >= 1 && a.m <= 128, "tcgen05 L-step requires m <= 128");
    Params p;
    p.a = a;
    if (a.final_mode) launch<true>(p, U, s);
    else launch<false>(p, U, s);
}

}  // namespace vmb
