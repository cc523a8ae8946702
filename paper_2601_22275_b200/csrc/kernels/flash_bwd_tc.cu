// flash_bwd_tc.cu — tcgen05 backward of the online-entropy attention (bf16, d = 128):
// flash_entropy.hpp:146-221, the paper's fine-tuning path (Alg. 2), SURVEY §8(f) row 2.
//
// Per unit, with Q pre-scaled by the caller and lse / H from the matching forward:
//   P  = exp(S - lse),  S = Q K^T          D_i = sum_x O[i,x] dO[i,x]
//   dS = P (dP - D) [- dH P (S - lse + H)]  = P (dP - dH S - c),  c = D + dH (H - lse)
//   dV = P^T dO   dK = dS^T Q   dQ = dS K    (dP = dO V^T)
// A row-statistics pass folds D, dH and H into one float4 per query row {lse log2e, c, dH, 0}
// (rows padded to 128 with lse = +inf, so padded queries carry P = dS = 0).  Then two
// deterministic kernels (no atomics; S and dP are recomputed once more than with a dQ
// atomic scheme, 7 instead of 5 GEMMs, in exchange for bitwise-reproducible gradients):
//   bwd_dq_kernel  CTA = 128 query rows; loops over 64-key tiles:
//                  S, dP = Q K_j^T, dO V_j^T (SS) -> thread = query row: dS -> TMEM (bf16)
//                  -> dQ += dS K_j (TS: A = dS from TMEM, B = K_j MN-major).
//   bwd_dkv_kernel CTA = 128 key rows; loops over 64-query tiles:
//                  S^T, dP^T = K Q_j^T, V dO_j^T (SS) -> thread = key row: P^T, dS^T -> TMEM
//                  -> dV += P^T dO_j, dK += dS^T Q_j (TS, B MN-major).
// Ragged edges need no masks: TMA zero-fills rows past the end (zero K rows add nothing to
// dQ, zero Q / dO rows with P = 0 add nothing to dK / dV); only the stores are guarded.
// Warp roles as in fa2_tc.cu: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2-5 element math / epilogue (TMEM lane = row).  TMEM: two (S | dP) buffers of
// 64 + 64 columns (double-buffered: tile j+1's GEMMs run during tile j's element math),
// then the accumulators (dQ; or dV, dK).
#include <cuda_bf16.h>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr int kStages = 3;
constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kPanel128 = 128 * 128;  // 128 rows x 64 bf16 (SW128)
constexpr uint32_t kPanel64 = 64 * 128;    // 64 rows x 64 bf16

struct BwdTcParams {
    CUtensorMap tmQ, tmG, tmK, tmV;  // dq kernel: Q/dO boxes of 128 rows, K/V of 64; dkv: the reverse
    const float4* rowstat;           // (U, nq_pad) {lse*log2e, c, dH, 0}
    __nv_bfloat16 *dq, *dk, *dv;     // (U, n, 128)
    int32_t nq, nk, nq_pad, n_tiles;  // n_tiles: inner-loop tiles (64 rows each)
};

__device__ __forceinline__ void tile_loads(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int row0, int u,
                                           uint32_t panel) {
    tma_load_5d(dst, map, bar, 0, row0, 0, 0, u);
    tma_load_5d(dst + panel, map, bar, 64, row0, 0, 0, u);
}

// TMEM row -> bf16 global row; the TMEM loads are warp-collective, so every lane issues
// them and only the store is predicated
__device__ __forceinline__ void store_row_bf16(__nv_bfloat16* dst, uint32_t tcol, bool valid) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t r[32];
        VMB_TMEM_LD32(tcol + cc * 32, r);
        tmem_ld_wait();
        if (!valid) continue;
        uint4 v[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            v[x].x = pack_bf16(__uint_as_float(r[8 * x + 0]), __uint_as_float(r[8 * x + 1]));
            v[x].y = pack_bf16(__uint_as_float(r[8 * x + 2]), __uint_as_float(r[8 * x + 3]));
            v[x].z = pack_bf16(__uint_as_float(r[8 * x + 4]), __uint_as_float(r[8 * x + 5]));
            v[x].w = pack_bf16(__uint_as_float(r[8 * x + 6]), __uint_as_float(r[8 * x + 7]));
        }
        st_global_256(dst + cc * 32, v[0], v[1]);
        st_global_256(dst + cc * 32 + 16, v[2], v[3]);
    }
}

// ------------------------------------------------------------------------ dQ
struct DqSmem {
    static constexpr uint32_t q_off = 0;                      // Q tile, 2 x 128-row panels
    static constexpr uint32_t g_off = 2 * kPanel128;          // dO tile
    static constexpr uint32_t ring_off = 4 * kPanel128;       // stages of K_j | V_j (64 rows)
    static constexpr uint32_t stage = 4 * kPanel64;
    static constexpr uint32_t bar_off = ring_off + kStages * stage;
    static constexpr uint32_t n_bars = 1 + 2 * kStages + 5;   // q_full, kv_full/empty, s_full[2], p_full[2], o_full
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t alloc = slot_off + 16 + 1024;
};

__global__ void __launch_bounds__(kThreads, 1) bwd_dq_kernel(const __grid_constant__ BwdTcParams p) {
    using SM = DqSmem;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = bars + 1 + kStages;
    uint64_t* s_full = bars + 1 + 2 * kStages;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_full = s_full + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);
    const int warp = warp_id();
    const int qt = blockIdx.x, u = blockIdx.y;
    const int n_kv = p.n_tiles;

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&p.tmQ);
        tma_prefetch_desc(&p.tmG);
        tma_prefetch_desc(&p.tmK);
        tma_prefetch_desc(&p.tmV);
        mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
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
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tDQ = tmem + 256;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(q_full, 4 * kPanel128);
            tile_loads(smem + SM::q_off, &p.tmQ, q_full, qt * 128, u, kPanel128);
            tile_loads(smem + SM::g_off, &p.tmG, q_full, qt * 128, u, kPanel128);
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % kStages;
                if (j >= kStages) mbar_wait_sleep(&kv_empty[st], ((j / kStages) + 1) & 1);
                uint8_t* sk = smem + SM::ring_off + st * SM::stage;
                mbar_arrive_expect_tx(&kv_full[st], SM::stage);
                tile_loads(sk, &p.tmK, &kv_full[st], j * 64, u, kPanel64);
                tile_loads(sk + 2 * kPanel64, &p.tmV, &kv_full[st], j * 64, u, kPanel64);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16(128, 64, 0, 0);   // S = Q K^T, dP = dO V^T
        constexpr uint32_t idQ = idesc_bf16(128, 128, 0, 1);  // dQ += dS K, K MN-major
        const uint32_t q_addr = smem_u32(smem + SM::q_off), g_addr = smem_u32(smem + SM::g_off);
        const uint32_t ring = smem_u32(smem + SM::ring_off);
        if (elect_one()) {
            mbar_wait_sleep(q_full, 0);
            for (int j = 0; j <= n_kv; ++j) {
                if (j < n_kv) {
                    const int st = j % kStages;
                    mbar_wait_sleep(&kv_full[st], (j / kStages) & 1);
                    tc_fence_after();
                    const uint32_t ka = ring + st * SM::stage, va = ka + 2 * kPanel64;
                    const uint32_t tS = tmem + (j & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t ao = (kk >> 2) * kPanel128 + (kk & 3) * 32, bo = (kk >> 2) * kPanel64 + (kk & 3) * 32;
                        umma_ss(tS, sdesc_sw128(q_addr + ao, 16, 1024), sdesc_sw128(ka + bo, 16, 1024), idS, kk > 0);
                    }
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t ao = (kk >> 2) * kPanel128 + (kk & 3) * 32, bo = (kk >> 2) * kPanel64 + (kk & 3) * 32;
                        umma_ss(tS + 64, sdesc_sw128(g_addr + ao, 16, 1024), sdesc_sw128(va + bo, 16, 1024), idS,
                                kk > 0);
                    }
                    umma_commit(&s_full[j & 1]);
                }
                if (j >= 1) {
                    const int jp = j - 1, st = jp % kStages;
                    mbar_wait_sleep(&p_full[jp & 1], (jp >> 1) & 1);
                    tc_fence_after();
                    const uint32_t ka = ring + st * SM::stage;
                    const uint32_t tDS = tmem + (jp & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_ts(tDQ, tDS + kk * 8, sdesc_sw128(ka + kk * 2048, kPanel64, 1024), idQ,
                                (jp > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&kv_empty[st]);
                }
            }
            umma_commit(o_full);
        }
    } else {
        const int row = (warp & 3) * 32 + lane_id();
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const int grow = qt * 128 + row;
        const float4 rs = p.rowstat[(int64_t)u * p.nq_pad + grow];
        const float nlse2 = -rs.x, c = rs.y, ndh = -rs.z;
        for (int j = 0; j < n_kv; ++j) {
            const uint32_t tS = tmem + (j & 1) * 128 + lane_base;
            mbar_wait_sleep(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sr[64], dr[64];
            VMB_TMEM_LD32(tS + 0, (sr + 0));
            VMB_TMEM_LD32(tS + 32, (sr + 32));
            VMB_TMEM_LD32(tS + 64, (dr + 0));
            VMB_TMEM_LD32(tS + 96, (dr + 32));
            tmem_ld_wait();
            uint32_t pk[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                float ds[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float s = __uint_as_float(sr[2 * x + e]), dp = __uint_as_float(dr[2 * x + e]);
                    const float pr = ex2(fmaf(s, kLog2e, nlse2));
                    ds[e] = pr * (fmaf(ndh, s, dp) - c);
                }
                pk[x] = pack_bf16(ds[0], ds[1]);
            }
            VMB_TMEM_ST16(tS + 0, (pk + 0));
            VMB_TMEM_ST16(tS + 16, (pk + 16));
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[j & 1]);
        }
        mbar_wait_sleep(o_full, 0);
        tc_fence_after();
        store_row_bf16(p.dq + ((int64_t)u * p.nq + grow) * 128, tDQ + lane_base, grow < p.nq);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ------------------------------------------------------------------------ dK, dV
struct DkvSmem {
    static constexpr uint32_t k_off = 0;                      // K tile, 2 x 128-row panels
    static constexpr uint32_t v_off = 2 * kPanel128;          // V tile
    static constexpr uint32_t ring_off = 4 * kPanel128;       // stages of Q_j | dO_j (64 rows) | rowstat_j
    static constexpr uint32_t stat_rel = 4 * kPanel64;
    static constexpr uint32_t stage = 4 * kPanel64 + 1024;    // 33 KB, 1024-aligned
    static constexpr uint32_t bar_off = ring_off + kStages * stage;
    static constexpr uint32_t n_bars = 1 + 2 * kStages + 5;   // kv_full, q_full/empty, s_full[2], p_full[2], o_full
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t alloc = slot_off + 16 + 1024;
};

__global__ void __launch_bounds__(kThreads, 1) bwd_dkv_kernel(const __grid_constant__ BwdTcParams p) {
    using SM = DkvSmem;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* kv_full = bars;
    uint64_t* q_full = bars + 1;
    uint64_t* q_empty = bars + 1 + kStages;
    uint64_t* s_full = bars + 1 + 2 * kStages;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_full = s_full + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);
    const int warp = warp_id();
    const int kt = blockIdx.x, u = blockIdx.y;
    const int n_q = p.n_tiles;

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&p.tmQ);
        tma_prefetch_desc(&p.tmG);
        tma_prefetch_desc(&p.tmK);
        tma_prefetch_desc(&p.tmV);
        mbar_init(kv_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 128);
        }
        mbar_init(o_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tDV = tmem + 256, tDK = tmem + 384;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(kv_full, 4 * kPanel128);
            tile_loads(smem + SM::k_off, &p.tmK, kv_full, kt * 128, u, kPanel128);
            tile_loads(smem + SM::v_off, &p.tmV, kv_full, kt * 128, u, kPanel128);
            for (int j = 0; j < n_q; ++j) {
                const int st = j % kStages;
                if (j >= kStages) mbar_wait_sleep(&q_empty[st], ((j / kStages) + 1) & 1);
                uint8_t* sq = smem + SM::ring_off + st * SM::stage;
                mbar_arrive_expect_tx(&q_full[st], SM::stage);
                tile_loads(sq, &p.tmQ, &q_full[st], j * 64, u, kPanel64);
                tile_loads(sq + 2 * kPanel64, &p.tmG, &q_full[st], j * 64, u, kPanel64);
                bulk_load(sq + SM::stat_rel, p.rowstat + (int64_t)u * p.nq_pad + j * 64, 1024, &q_full[st]);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16(128, 64, 0, 0);   // S^T = K Q^T, dP^T = V dO^T
        constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // dV += P^T dO, dK += dS^T Q (B MN-major)
        const uint32_t k_addr = smem_u32(smem + SM::k_off), v_addr = smem_u32(smem + SM::v_off);
        const uint32_t ring = smem_u32(smem + SM::ring_off);
        if (elect_one()) {
            mbar_wait_sleep(kv_full, 0);
            for (int j = 0; j <= n_q; ++j) {
                if (j < n_q) {
                    const int st = j % kStages;
                    mbar_wait_sleep(&q_full[st], (j / kStages) & 1);
                    tc_fence_after();
                    const uint32_t qa = ring + st * SM::stage, ga = qa + 2 * kPanel64;
                    const uint32_t tS = tmem + (j & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t ao = (kk >> 2) * kPanel128 + (kk & 3) * 32, bo = (kk >> 2) * kPanel64 + (kk & 3) * 32;
                        umma_ss(tS, sdesc_sw128(k_addr + ao, 16, 1024), sdesc_sw128(qa + bo, 16, 1024), idS, kk > 0);
                    }
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t ao = (kk >> 2) * kPanel128 + (kk & 3) * 32, bo = (kk >> 2) * kPanel64 + (kk & 3) * 32;
                        umma_ss(tS + 64, sdesc_sw128(v_addr + ao, 16, 1024), sdesc_sw128(ga + bo, 16, 1024), idS,
                                kk > 0);
                    }
                    umma_commit(&s_full[j & 1]);
                }
                if (j >= 1) {
                    const int jp = j - 1, st = jp % kStages;
                    mbar_wait_sleep(&p_full[jp & 1], (jp >> 1) & 1);
                    tc_fence_after();
                    const uint32_t qa = ring + st * SM::stage, ga = qa + 2 * kPanel64;
                    const uint32_t tP = tmem + (jp & 1) * 128, tDS = tP + 64;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_ts(tDV, tP + kk * 8, sdesc_sw128(ga + kk * 2048, kPanel64, 1024), idO,
                                (jp > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_ts(tDK, tDS + kk * 8, sdesc_sw128(qa + kk * 2048, kPanel64, 1024), idO,
                                (jp > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&q_empty[st]);
                }
            }
            umma_commit(o_full);
        }
    } else {
        const int row = (warp & 3) * 32 + lane_id();
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const int grow = kt * 128 + row;
        for (int j = 0; j < n_q; ++j) {
            const int st = j % kStages;
            const uint32_t tS = tmem + (j & 1) * 128 + lane_base;
            mbar_wait_sleep(&q_full[st], (j / kStages) & 1);  // row statistics of this query tile
            mbar_wait_sleep(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            const float4* stat = reinterpret_cast<const float4*>(smem + SM::ring_off + st * SM::stage + SM::stat_rel);
            uint32_t sr[64], dr[64];
            VMB_TMEM_LD32(tS + 0, (sr + 0));
            VMB_TMEM_LD32(tS + 32, (sr + 32));
            VMB_TMEM_LD32(tS + 64, (dr + 0));
            VMB_TMEM_LD32(tS + 96, (dr + 32));
            tmem_ld_wait();
            uint32_t pp[32], pd[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                float pr[2], ds[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float4 rs = stat[2 * x + e];  // broadcast read: every lane the same query
                    const float s = __uint_as_float(sr[2 * x + e]), dp = __uint_as_float(dr[2 * x + e]);
                    pr[e] = ex2(fmaf(s, kLog2e, -rs.x));
                    ds[e] = pr[e] * (fmaf(-rs.z, s, dp) - rs.y);
                }
                pp[x] = pack_bf16(pr[0], pr[1]);
                pd[x] = pack_bf16(ds[0], ds[1]);
            }
            VMB_TMEM_ST16(tS + 0, (pp + 0));
            VMB_TMEM_ST16(tS + 16, (pp + 16));
            VMB_TMEM_ST16(tS + 64, (pd + 0));
            VMB_TMEM_ST16(tS + 80, (pd + 16));
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[j & 1]);
        }
        mbar_wait_sleep(o_full, 0);
        tc_fence_after();
        store_row_bf16(p.dv + ((int64_t)u * p.nk + grow) * 128, tDV + lane_base, grow < p.nk);
        store_row_bf16(p.dk + ((int64_t)u * p.nk + grow) * 128, tDK + lane_base, grow < p.nk);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ------------------------------------------------------------------------ row statistics
// one warp per (unit, padded query row): {lse log2e, c = D + dH (H - lse), dH, 0}
__global__ void __launch_bounds__(256) bwd_rowstat_kernel(const __nv_bfloat16* o, const __nv_bfloat16* g,
                                                          const float* lse, const float* ent, const float* dent,
                                                          int eg, int64_t U, int64_t nq, int64_t nq_pad,
                                                          float4* out) {
    const int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= U * nq_pad) return;
    const int64_t u = w / nq_pad, i = w % nq_pad;
    if (i >= nq) {
        if (lane == 0) out[w] = make_float4(INFINITY, 0.f, 0.f, 0.f);
        return;
    }
    const int64_t r = u * nq + i;
    const uint2 ov = reinterpret_cast<const uint2*>(o + r * 128)[lane];
    const uint2 gv = reinterpret_cast<const uint2*>(g + r * 128)[lane];
    const uint32_t ow[2] = {ov.x, ov.y}, gw[2] = {gv.x, gv.y};
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        acc += (double)__uint_as_float(ow[e] << 16) * (double)__uint_as_float(gw[e] << 16);
        acc += (double)__uint_as_float(ow[e] & 0xFFFF0000u) * (double)__uint_as_float(gw[e] & 0xFFFF0000u);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
        const float l = lse[r];
        const float dh = eg ? dent[r] : 0.f;
        const float c = (float)acc + (eg ? dh * (ent[r] - l) : 0.f);
        out[w] = make_float4(l * kLog2e, c, dh, 0.f);
    }
}

CUtensorMap rows_map(const void* base, int64_t U, int64_t n, uint32_t box_rows) {
    const uint64_t dims[5] = {128, (uint64_t)n, 1, 1, (uint64_t)U};
    const uint64_t row = 256, unit = (uint64_t)n * 256;
    const uint64_t strides[4] = {row, unit, unit, unit};
    const uint32_t box[5] = {64, box_rows, 1, 1, 1};
    return make_tmap_bf16_5d(base, dims, strides, box);
}

}  // namespace

int64_t flash_bwd_tc_rowstat_rows(int64_t nq) { return (nq + 127) / 128 * 128; }

void flash_bwd_tc_launch(int64_t U, int64_t nq, int64_t nk, const void* q, const void* k, const void* v,
                         const void* o, const void* dout, const float* lse, const float* ent, const float* dent,
                         int entropy_grad, void* rowstat, void* dq, void* dk, void* dv, cudaStream_t s) {
    if (U == 0) return;
    const int64_t nq_pad = flash_bwd_tc_rowstat_rows(nq);
    ProfScope ps(kKAttn, s);
    if (nq > 0) {
        const int64_t warps = U * nq_pad;
        bwd_rowstat_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse, ent, dent,
            entropy_grad, U, nq, nq_pad, static_cast<float4*>(rowstat));
        count_launch();
        check_launch("flash_bwd_rowstat");
    }
    BwdTcParams p{};
    p.rowstat = static_cast<const float4*>(rowstat);
    p.dq = static_cast<__nv_bfloat16*>(dq);
    p.dk = static_cast<__nv_bfloat16*>(dk);
    p.dv = static_cast<__nv_bfloat16*>(dv);
    p.nq = (int32_t)nq;
    p.nk = (int32_t)nk;
    p.nq_pad = (int32_t)nq_pad;
    if (nq > 0) {
        // dQ: 128-row Q / dO boxes, 64-row K / V boxes
        p.tmQ = rows_map(q, U, nq, 128);
        p.tmG = rows_map(dout, U, nq, 128);
        p.tmK = rows_map(k, U, nk, 64);
        p.tmV = rows_map(v, U, nk, 64);
        p.n_tiles = (int32_t)((nk + 63) / 64);
        VMB_CHECK_CUDA(cudaFuncSetAttribute(bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)DqSmem::alloc));
        bwd_dq_kernel<<<dim3((unsigned)(nq_pad / 128), (unsigned)U), kThreads, DqSmem::alloc, s>>>(p);
        count_launch();
        check_launch("flash_bwd_dq");
    }
    // dK, dV: 128-row K / V boxes, 64-row Q / dO boxes (nq == 0: dK = dV = 0 from an empty loop)
    p.tmQ = rows_map(q, U, std::max<int64_t>(nq, 1), 64);
    p.tmG = rows_map(dout, U, std::max<int64_t>(nq, 1), 64);
    p.tmK = rows_map(k, U, nk, 128);
    p.tmV = rows_map(v, U, nk, 128);
    p.n_tiles = (int32_t)((nq + 63) / 64);
    VMB_REQUIRE_DIM(p.n_tiles > 0, "flash backward over empty queries needs the CUDA-core path");
    VMB_CHECK_CUDA(cudaFuncSetAttribute(bwd_dkv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)DkvSmem::alloc));
    bwd_dkv_kernel<<<dim3((unsigned)((nk + 127) / 128), (unsigned)U), kThreads, DkvSmem::alloc, s>>>(p);
    count_launch();
    check_launch("flash_bwd_dkv");
}

}  // namespace vmb
