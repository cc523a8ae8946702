// lstep_big.cu — tcgen05 L half-step and apply for m > 128 row blocks (bf16, d = 128):
// the general factorizations of SURVEY §8(f) row 4 (overrides with more than 128 frames,
// down to the degenerate b = 1 where the L-step is dense attention over all N tokens).
//
// Per (unit u, position i) the L-step is an m x m attention (monarch.hpp:105-147):
//   S[j,k] = qscale <Qb[i,j], aL[i,k]> - cL[i,k],   L[j,:] = softmax_k S[j,:]
//   ITER : cR[k,i] = sum_j L[j,k],  aR[k,i] = qscale sum_j L[j,k] Qb[i,j]
//   FINAL: O[j*b+i] = sum_k L[j,k] y[k,i]
// With m > 128 a block no longer fits one tile (lstep_tc.cu), so the L-step runs in passes:
//   <kRowStat> CTA = 128 rows j, streams 64-key tiles of aL: online max / sum of S ->
//              lse2[j] (base 2) into the workspace
//   <kIter>    CTA = 128 keys k, streams 64-row tiles of Qb: S^T = aL Qb^T, L^T =
//              exp2(S^T - lse2[j]) (already normalised, no online rescale), cR = row sums,
//              aR += L^T Qb (TS MMA: L^T from TMEM, Qb MN-major)
//   <kFinal>   CTA = 128 rows j, streams 64-key tiles of aL | y: L = exp2(S - lse2[j]),
//              O += L y (TS MMA)
// Warp roles as in fa2_tc.cu: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer, warps
// 2-5 element math / epilogue (TMEM lane = row).  TMEM 256 columns: two 64-column score
// buffers (the next tile's GEMM runs during this tile's math) and the 128-column accumulator;
// under 113 KB of shared memory, so two CTAs share an SM.  Per-column vectors (cL, or lse2)
// of each streamed tile are staged in shared memory by the math warps; indices past m read
// +inf, which zeroes their exponentials -- the TMA zero-fill does the rest of the masking.
#include <cuda_bf16.h>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kPanel128 = 128 * 128;  // 128 rows x 64 bf16 (SW128)
constexpr uint32_t kPanel64 = 64 * 128;    // 64 rows x 64 bf16
enum { kRowStat = 0, kIter = 1, kFinal = 2 };

template <int MODE>
struct BigSmem {
    static constexpr int S = MODE == kFinal ? 2 : 4;                     // streamed stages
    static constexpr uint32_t stage = (MODE == kFinal ? 4 : 2) * kPanel64;  // aL (| y), or Qb
    static constexpr uint32_t stat_off = 0;                              // stationary 128-row tile
    static constexpr uint32_t ring_off = 2 * kPanel128;
    static constexpr uint32_t vec_off = ring_off + S * stage;            // [2][64] column vectors
    static constexpr uint32_t bar_off = vec_off + 2 * 64 * 4;
    static constexpr uint32_t n_bars = 1 + 2 * S + 5;  // st_full, kv_full[S], kv_empty[S], s_full[2], p_full[2], o_full
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t alloc = slot_off + 16 + 1024;
    static_assert(alloc <= 113 * 1024, "two CTAs per SM");
};

__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int c1, int c2, int c3,
                                          int c4, uint32_t panel) {
    tma_load_5d(dst, map, bar, 0, c1, c2, c3, c4);
    tma_load_5d(dst + panel, map, bar, 64, c1, c2, c3, c4);
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) lstep_big_kernel(const __grid_constant__ TcLstepBigArgs a) {
    using SM = BigSmem<MODE>;
    constexpr int S = SM::S;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* st_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = bars + 1 + S;
    uint64_t* s_full = bars + 1 + 2 * S;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_full = s_full + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);
    float* vec = reinterpret_cast<float*>(smem + SM::vec_off);

    const int warp = warp_id();
    const int rt = blockIdx.y;                    // 128-row tile of the stationary operand
    const int ui = blockIdx.x;                    // u * b + i
    const int u = ui / a.b, i = ui % a.b;
    const int qh = u % a.H, qb = u / a.H;
    const int n_tiles = (a.m + 63) / 64;          // streamed 64-row tiles
    const int64_t vbase = (int64_t)ui * a.m;      // cL / lse2 of this (u, i): (U, b, m)

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(MODE == kIter ? &a.tmQ64 : &a.tmQ128);
        tma_prefetch_desc(MODE == kIter ? &a.tmAL128 : &a.tmAL64);
        if (MODE == kFinal) tma_prefetch_desc(&a.tmY64);
        mbar_init(st_full, 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 128);
        }
        mbar_init(o_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tO = tmem + 128;

    if (warp == 0) {
        if (elect_one()) {
            uint8_t* st = smem + SM::stat_off;
            mbar_arrive_expect_tx(st_full, 2 * kPanel128);
            if (MODE == kIter) load_tile(st, &a.tmAL128, st_full, rt * 128, i, 0, u, kPanel128);  // aL rows k
            else load_tile(st, &a.tmQ128, st_full, i, rt * 128, qh, qb, kPanel128);               // Qb rows j
            for (int j = 0; j < n_tiles; ++j) {
                const int s = j % S;
                if (j >= S) mbar_wait_sleep(&kv_empty[s], ((j / S) + 1) & 1);
                uint8_t* d = smem + SM::ring_off + s * SM::stage;
                mbar_arrive_expect_tx(&kv_full[s], SM::stage);
                if (MODE == kIter) {
                    load_tile(d, &a.tmQ64, &kv_full[s], i, j * 64, qh, qb, kPanel64);  // Qb rows j
                } else {
                    load_tile(d, &a.tmAL64, &kv_full[s], j * 64, i, 0, u, kPanel64);   // aL rows k
                    if (MODE == kFinal) load_tile(d + 2 * kPanel64, &a.tmY64, &kv_full[s], i, j * 64, 0, u, kPanel64);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16(128, 64, 0, 0);   // S = A B^T, both K-major
        constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // acc += P B, B MN-major
        const uint32_t st_addr = smem_u32(smem + SM::stat_off), ring = smem_u32(smem + SM::ring_off);
        if (elect_one()) {
            mbar_wait_sleep(st_full, 0);
            for (int j = 0; j <= n_tiles; ++j) {
                if (j < n_tiles) {
                    const int s = j % S;
                    mbar_wait_sleep(&kv_full[s], (j / S) & 1);
                    // RowStat has no second GEMM: wait until the math warps have read S(j-2)
                    if (MODE == kRowStat && j >= 2) mbar_wait_sleep(&p_full[j & 1], ((j - 2) >> 1) & 1);
                    tc_fence_after();
                    const uint32_t ka = ring + s * SM::stage;
                    const uint32_t tS = tmem + (j & 1) * 64;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t ao = (kk >> 2) * kPanel128 + (kk & 3) * 32, bo = (kk >> 2) * kPanel64 + (kk & 3) * 32;
                        umma_ss(tS, sdesc_sw128(st_addr + ao, 16, 1024), sdesc_sw128(ka + bo, 16, 1024), idS, kk > 0);
                    }
                    umma_commit(&s_full[j & 1]);
                    if (MODE == kRowStat) umma_commit(&kv_empty[s]);
                }
                if (MODE != kRowStat && j >= 1) {
                    const int jp = j - 1, s = jp % S;
                    mbar_wait_sleep(&p_full[jp & 1], (jp >> 1) & 1);
                    tc_fence_after();
                    // second operand: Iter -> the Qb tile itself (MN-major view), Final -> y
                    const uint32_t ba = ring + s * SM::stage + (MODE == kFinal ? 2 * kPanel64 : 0);
                    const uint32_t tP = tmem + (jp & 1) * 64;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_ts(tO, tP + kk * 8, sdesc_sw128(ba + kk * 2048, kPanel64, 1024), idO,
                                (jp > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&kv_empty[s]);
                }
            }
            umma_commit(o_full);
        }
    } else {
        const int t = threadIdx.x - 64;                // 0..127
        const int row = (warp & 3) * 32 + lane_id();   // TMEM lane == stationary row
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const int grow = rt * 128 + row;
        const bool valid = grow < a.m;
        // per-row scalar: Final -> lse2[j]; Iter -> cL2[k]
        float rowv = 0.f;
        if (MODE == kFinal) rowv = valid ? a.lse2[vbase + grow] : 0.f;
        if (MODE == kIter) rowv = valid ? a.cL[vbase + grow] * kLog2e : 0.f;
        const float qs2 = a.qscale * kLog2e;
        float m_run = -INFINITY, l_run = 0.f, csum = 0.f;
        for (int j = 0; j < n_tiles; ++j) {
            // stage this tile's per-column vector: cL2 (RowStat, Final) or lse2 (Iter)
            float* sv = vec + (j & 1) * 64;
            if (t < 64) {
                const int c = j * 64 + t;
                float x = INFINITY;
                if (c < a.m) x = MODE == kIter ? a.lse2[vbase + c] : a.cL[vbase + c] * kLog2e;
                sv[t] = x;
            }
            named_bar_sync(1, 128);
            const uint32_t tS = tmem + (j & 1) * 64 + lane_base;
            mbar_wait_sleep(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sr[64];
            VMB_TMEM_LD32(tS + 0, (sr + 0));
            VMB_TMEM_LD32(tS + 32, (sr + 32));
            tmem_ld_wait();
            if (MODE == kRowStat) {
                tc_fence_before();
                mbar_arrive(&p_full[j & 1]);  // S buffer free for S(j+2)
                float mx = m_run;
#pragma unroll
                for (int x = 0; x < 64; ++x) {
                    const float v = fmaf(__uint_as_float(sr[x]), qs2, -sv[x]);
                    sr[x] = __float_as_uint(v);
                    mx = fmaxf(mx, v);
                }
                if (mx > -INFINITY) {
                    float acc = 0.f;
#pragma unroll
                    for (int x = 0; x < 64; ++x) acc += ex2(__uint_as_float(sr[x]) - mx);
                    l_run = l_run * ex2(m_run - mx) + acc;
                    m_run = mx;
                }
            } else {
                uint32_t pk[32];
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    float p[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        p[e] = ex2(fmaf(__uint_as_float(sr[2 * x + e]), qs2, -sv[2 * x + e]) - rowv);
                    if (MODE == kIter) csum += p[0] + p[1];
                    pk[x] = pack_bf16(p[0], p[1]);
                }
                VMB_TMEM_ST16(tS + 0, (pk + 0));
                VMB_TMEM_ST16(tS + 16, (pk + 16));
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[j & 1]);
            }
        }
        if (MODE == kRowStat) {
            if (valid) a.lse2[vbase + grow] = m_run + log2f(l_run);
        } else {
            mbar_wait_sleep(o_full, 0);
            tc_fence_after();
            __nv_bfloat16* dst;
            if (MODE == kIter) {
                // aR (U, m, b, d) row (u, k, i); cR (U, m, b)
                const int64_t r = ((int64_t)u * a.m + grow) * a.b + i;
                dst = a.aR + r * 128;
                if (valid) a.cR[r] = csum;
            } else {
                // O row j*b + i of unit u = (ob, oh)
                const int64_t ob = u / a.oHn, oh = u % a.oHn;
                dst = a.out + ob * a.oB + oh * a.oH + ((int64_t)grow * a.b + i) * a.oT;
            }
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t r[32];
                VMB_TMEM_LD32(tO + lane_base + cc * 32, r);
                tmem_ld_wait();
                if (!valid) continue;
                uint4 v[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    v[x].x = pack_bf16(__uint_as_float(r[8 * x + 0]) * a.out_scale, __uint_as_float(r[8 * x + 1]) * a.out_scale);
                    v[x].y = pack_bf16(__uint_as_float(r[8 * x + 2]) * a.out_scale, __uint_as_float(r[8 * x + 3]) * a.out_scale);
                    v[x].z = pack_bf16(__uint_as_float(r[8 * x + 4]) * a.out_scale, __uint_as_float(r[8 * x + 5]) * a.out_scale);
                    v[x].w = pack_bf16(__uint_as_float(r[8 * x + 6]) * a.out_scale, __uint_as_float(r[8 * x + 7]) * a.out_scale);
                }
                uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
                for (int x = 0; x < 4; ++x) d4[x] = v[x];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

template <int MODE>
void launch(const TcLstepBigArgs& a, int64_t U, cudaStream_t s) {
    using SM = BigSmem<MODE>;
    auto kern = lstep_big_kernel<MODE>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    const dim3 grid((unsigned)(U * a.b), (unsigned)((a.m + 127) / 128));
    kern<<<grid, kThreads, SM::alloc, s>>>(a);
    count_launch();
    check_launch("lstep_big");
}

}  // namespace

void tc_lstep_big_launch(const TcLstepBigArgs& a, int64_t U, bool final_mode, cudaStream_t s) {
    if (U == 0) return;
    VMB_REQUIRE_DIM((a.m + 127) / 128 <= 65535, "large-m L-step: too many row tiles");
    ProfScope ps(final_mode ? kKLfinal : kKLstep, s);
    launch<kRowStat>(a, U, s);
    if (final_mode) launch<kFinal>(a, U, s);
    else launch<kIter>(a, U, s);
}

}  // namespace vmb
