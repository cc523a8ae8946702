// fa_tc.cu — tcgen05 flash-attention kernel with fused online entropy (bf16, d = 128).
//
// One kernel serves three hot-path roles:
//   * R half-step  (monarch.hpp:53-103): query = aR[k] (or Q on the first step), key = value
//     = Kb[k], per-row temperature 1/max(cR, clamp) folded into the softmax scale, outputs
//     aL rows (strided into (b,m,d)) and cL = sum_l R ln R.          <NB=1, NO=1>
//   * last R half-step with the assembly GEMM y[k] = R[k] Vb[k] fused (monarch.hpp:182-185):
//     O = P [K | V], outputs aL and y.                                  <NB=2, NO=2>
//   * first-frame recompute / dense baseline (flash_entropy.hpp:85-139, video.hpp:117-126):
//     query = Q rows, key/value = all keys, outputs O (+ lse, entropy). <NB=2, NO=1>
//
// CTA = one 128-row query tile of one segment.  Warp roles (256 threads):
//   warp 0      TMA producer: Q tile once, then a ring of KV stages (NB tiles of 128x128)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4-7   softmax / statistics / epilogue; thread t owns query row t (TMEM lane t)
// TMEM (512 cols): S0 [0,128), S1 [128,256) double-buffered scores; P (bf16) overwrites
// the first 64 columns of its S buffer; O accumulators at [256, 256 + 128*NO).
// S_{j+1} = Q K_{j+1}^T is issued before waiting for P_j, so the tensor pipe computes the
// next score tile while the softmax warps work on the current one.
//
// Statistics are kept in base 2 with a lazily-updated reference max (rescale O only when
// the running max grows by more than 8, FA4-style); the entropy accumulator uses the
// same reference, so  sum p ln p = ln2 * h / l - ln l  exactly as absorb_stats
// (flash_entropy.hpp:25-51) but without per-tile rescaling.
#include <cuda_bf16.h>

#include <cstdlib>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 256;
constexpr int kTile = 128;                 // query rows per CTA, keys per KV tile
constexpr uint32_t kPanelBytes = 128 * 128;  // 128 rows x 64 bf16
constexpr uint32_t kTileBytes = 2 * kPanelBytes;  // 128 x 128 bf16
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;
constexpr float kMasked = -1.0e30f;

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
// 2^x for an element pair on the FMA/ALU pipes (see fa3_tc.cu)
__device__ __forceinline__ uint64_t ex2_emu2(uint64_t x2) {
    const uint64_t xx = pk2(fmaxf(lo2(x2), -126.f), fmaxf(hi2(x2), -126.f));
    const uint64_t t = fadd2(xx, pk2(12582912.f, 12582912.f));
    const uint64_t f = fadd2(xx, fadd2(pk2(-12582912.f, -12582912.f), t) ^ 0x8000000080000000ull);
    uint64_t p = ffma2(pk2(0.05592203512787819f, 0.05592203512787819f), f,
                       pk2(0.24264007806777954f, 0.24264007806777954f));
    p = ffma2(p, f, pk2(0.6931210160255432f, 0.6931210160255432f));
    p = ffma2(p, f, pk2(0.9999244809150696f, 0.9999244809150696f));
    const uint32_t r0 = (uint32_t)p + ((uint32_t)t << 23);
    const uint32_t r1 = (uint32_t)(p >> 32) + ((uint32_t)(t >> 32) << 23);
    return (uint64_t)r0 | ((uint64_t)r1 << 32);
}

template <int NB>
struct Stages {
    static constexpr int value = NB == 1 ? 4 : 3;
};

struct Params {
    TcFaArgs a;
    int32_t n_kv_tiles;
};

template <int NB, int NO>
struct Smem {
    static constexpr int S = Stages<NB>::value;
    static constexpr uint32_t q_off = 0;
    static constexpr uint32_t kv_off = kTileBytes;
    static constexpr uint32_t bar_off = kv_off + S * NB * kTileBytes;
    // barriers: q_full, kv_full[S], kv_empty[S], s_full[2], p_full[2], pv_done, o_full
    static constexpr uint32_t n_bars = 1 + 2 * S + 2 + 2 + 2;
    static constexpr uint32_t tmem_slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t bytes = tmem_slot_off + 16;
    static constexpr uint32_t alloc = bytes + 1024;  // alignment slack
};

// MC: CTAs of adjacent query tiles form 2-CTA clusters; each K/V stage is loaded once per
// cluster (CTA 0 fetches the K tile, CTA 1 the V tile -- or halves of the K tile when NB == 1)
// and multicast into both CTAs, halving the L2 -> SMEM stream (at one CTA per SM the last
// R-step needs ~11 TB/s of K|V tiles at full MMA rate, the TMA ceiling).  A stage is refilled
// only when both CTAs' MMAs have released it (kv_empty counts 2 multicast commits).
#ifndef VMB_TRACE
#define VMB_TRACE 0
#endif
#if VMB_TRACE
// debug-only timeline probes: [cta][event] globaltimer (ns); read by scripts/trace_fa.py
__device__ unsigned long long g_trace[4096][8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(ev) do { const unsigned cta_ = blockIdx.y * gridDim.x + blockIdx.x; \
    if (cta_ < 4096) g_trace[cta_][ev] = gtimer(); } while (0)
#else
#define TRACE(ev) do { } while (0)
#endif

template <int NB, int NO, bool MC>
__global__ void __launch_bounds__(kThreads, 1) fa_tc_kernel(const __grid_constant__ Params p) {
    using SM = Smem<NB, NO>;
    constexpr int S = SM::S;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = bars + 1 + S;
    uint64_t* s_full = bars + 1 + 2 * S;
    uint64_t* p_full = bars + 3 + 2 * S;
    uint64_t* pv_done = bars + 5 + 2 * S;
    uint64_t* o_full = bars + 6 + 2 * S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::tmem_slot_off);

    const TcFaArgs& a = p.a;
    const int warp = warp_id();
    const int qtile = blockIdx.x;
    const int useg = blockIdx.y;           // u * nseg + s
    const int u = useg / a.nseg, seg = useg % a.nseg;
    const int n_kv = p.n_kv_tiles;

    if (threadIdx.x == 128) TRACE(0);  // CTA start
    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        if (NB == 2) tma_prefetch_desc(&a.tmV);
        mbar_init(q_full, 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], MC ? 2 : 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 128);
        }
        mbar_init(pv_done, 1);
        mbar_init(o_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    if (MC) cluster_sync();  // peers' barriers initialised before any multicast lands
    else __syncthreads();
    tc_fence_after();
    const uint32_t crank = MC ? cluster_ctarank() : 0;
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 128) TRACE(1);  // TMEM allocated, barriers ready
    const uint32_t tS0 = tmem, tO = tmem + 256;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            const int qb = u / a.qH, qh = u % a.qH;
            const int kb = u / a.kH, kh = u % a.kH;
            const int kseg = seg;  // R-step: frame k of K; attention modes have nseg == 1
            uint8_t* sq = smem + SM::q_off;
            mbar_arrive_expect_tx(q_full, kTileBytes);
            tma_load_5d(sq, &a.tmQ, q_full, 0, qtile * kTile, seg, qh, qb);
            tma_load_5d(sq + kPanelBytes, &a.tmQ, q_full, 64, qtile * kTile, seg, qh, qb);
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % S;
                if (j >= S) mbar_wait_sleep(&kv_empty[st], ((j / S) + 1) & 1);
                uint8_t* skv = smem + SM::kv_off + st * NB * kTileBytes;
                mbar_arrive_expect_tx(&kv_full[st], NB * kTileBytes);
                if (MC) {
                    // this CTA fetches one half of the stage (a whole tile when NB == 2, one
                    // 64-column panel of the K tile when NB == 1) for both CTAs
                    if (NB == 2) {
                        const CUtensorMap* map = crank == 0 ? &a.tmK : &a.tmV;
                        uint8_t* dst = skv + crank * kTileBytes;
                        tma_load_5d_mc(dst, map, &kv_full[st], 0x3, 0, j * kTile, kseg, kh, kb);
                        tma_load_5d_mc(dst + kPanelBytes, map, &kv_full[st], 0x3, 64, j * kTile, kseg, kh, kb);
                    } else {
                        tma_load_5d_mc(skv + crank * kPanelBytes, &a.tmK, &kv_full[st], 0x3, 64 * crank, j * kTile,
                                       kseg, kh, kb);
                    }
                    continue;
                }
                tma_load_5d(skv, &a.tmK, &kv_full[st], 0, j * kTile, kseg, kh, kb);
                tma_load_5d(skv + kPanelBytes, &a.tmK, &kv_full[st], 64, j * kTile, kseg, kh, kb);
                if (NB == 2) {
                    tma_load_5d(skv + kTileBytes, &a.tmV, &kv_full[st], 0, j * kTile, kseg, kh, kb);
                    tma_load_5d(skv + kTileBytes + kPanelBytes, &a.tmV, &kv_full[st], 64,
                                j * kTile, kseg, kh, kb);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);   // S = Q K^T, both K-major
        constexpr uint32_t idPV = idesc_bf16(128, 128, 0, 1);  // O += P V, V MN-major
        constexpr uint32_t idPV2 = idesc_bf16(128, 256, 0, 1); // O += P [K | V]
        const uint32_t q_addr = smem_u32(smem + SM::q_off);
        const uint32_t kv_addr = smem_u32(smem + SM::kv_off);
        if (elect_one()) {
            mbar_wait_sleep(q_full, 0);
            for (int j = 0; j <= n_kv; ++j) {
                if (j < n_kv) {
                    const int st = j % S;
                    mbar_wait_sleep(&kv_full[st], (j / S) & 1);
                    tc_fence_after();
                    const uint32_t kaddr = kv_addr + st * NB * kTileBytes;
                    const uint32_t tS = tS0 + (j & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kPanelBytes + (kk & 3) * 32;
                        umma_ss(tS, sdesc_sw128(q_addr + off, 16, 1024),
                                sdesc_sw128(kaddr + off, 16, 1024), idS, kk > 0);
                    }
                    umma_commit(&s_full[j & 1]);
                }
                if (j >= 1) {
                    const int jp = j - 1, st = jp % S;
                    mbar_wait_sleep(&p_full[jp & 1], (jp >> 1) & 1);
                    tc_fence_after();
                    const uint32_t tP = tS0 + (jp & 1) * 128;
                    const uint32_t kaddr = kv_addr + st * NB * kTileBytes;
                    if (NO == 2) {
                        // O[:, 0:256) += P [K | V]: one N = 256 MMA per k-step (the K and V
                        // tiles are adjacent 2-panel tiles, so the four 64-column panels of the
                        // B operand are uniformly strided); N = 256 is the full-rate shape
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            umma_ts(tO, tP + kk * 8, sdesc_sw128(kaddr + kk * 2048, kPanelBytes, 1024), idPV2,
                                    (jp > 0 || kk > 0) ? 1u : 0u);
                    } else {
                        const uint32_t vaddr = kaddr + (NB == 2 ? kTileBytes : 0);
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            umma_ts(tO, tP + kk * 8, sdesc_sw128(vaddr + kk * 2048, kPanelBytes, 1024), idPV,
                                    (jp > 0 || kk > 0) ? 1u : 0u);
                    }
                    if (MC) umma_commit_mc(&kv_empty[st], 0x3);  // release the stage in both CTAs
                    else umma_commit(&kv_empty[st]);
                    umma_commit(pv_done);
                }
            }
            umma_commit(o_full);
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ softmax / epilogue
        const int row = threadIdx.x - 128;            // TMEM lane == query row in tile
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const int grow = qtile * kTile + row;         // row within the segment
        const bool valid = grow < a.q_len;
        float c = 1.f;
        if (a.cR && valid) c = a.cR[((int64_t)u * a.nseg + seg) * a.q_len + grow];
        if (a.clamp_enabled) {
            c = (c < a.clamp_min) ? a.clamp_min : c;
        } else if (!(c > 0.f)) {
            if (valid) atomicExch(a.status, kStatusClampDomain);
            c = 1.f;
        }
        const float scale2 = a.qscale * kLog2e / c;
        const int last_valid = a.kv_len - (n_kv - 1) * kTile;  // valid keys in the last tile

        if (a.check_finite) {
            mbar_wait_sleep(q_full, 0);
            const uint4* q0 = reinterpret_cast<const uint4*>(smem + SM::q_off + row * 128);
            const uint4* q1 = reinterpret_cast<const uint4*>(smem + SM::q_off + kPanelBytes + row * 128);
            bool bad = false;
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                const uint4 v0 = q0[x ^ (row & 7)], v1 = q1[x ^ (row & 7)];
                const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    bad |= ((w[e] & 0x7F80u) == 0x7F80u) || ((w[e] & 0x7F800000u) == 0x7F800000u);
            }
            if (bad && valid) atomicExch(a.status, kStatusNonFiniteQ);
        }

        float m_run = -INFINITY, l_run = 0.f;
        const uint64_t scale2x2 = pk2(scale2, scale2);
        for (int j = 0; j < n_kv; ++j) {
            const uint32_t tS = tS0 + (j & 1) * 128 + lane_base;
            mbar_wait_sleep(&s_full[j & 1], (j >> 1) & 1);
            if (threadIdx.x == 128 && j == 0) TRACE(2);         // first score tile ready
            if (threadIdx.x == 128 && j == n_kv - 1) TRACE(3);  // last score tile ready
            tc_fence_after();
#if VMB_DEBUG_NO_SOFTMAX  // timing experiment only: MMA/TMA pipeline without the softmax
            if (true) {
                mbar_arrive(&p_full[j & 1]);
                continue;
            }
#endif
            uint32_t sr[128];
            VMB_TMEM_LD32(tS + 0, (sr + 0));
            VMB_TMEM_LD32(tS + 32, (sr + 32));
            VMB_TMEM_LD32(tS + 64, (sr + 64));
            VMB_TMEM_LD32(tS + 96, (sr + 96));
            tmem_ld_wait();
            float* s = reinterpret_cast<float*>(sr);
            if (j == n_kv - 1 && last_valid < kTile) {
                asm volatile("");  // keep this a real (rarely taken) branch, not 128 selects
#pragma unroll
                for (int x = 0; x < 128; ++x)
                    if (x >= last_valid) s[x] = kMasked;
            }
            // row max: 4 independent FMNMX3 chains (depth 16) instead of one of depth 127
            float a0 = s[0], a1 = s[1], a2 = s[2], a3 = s[3];
#pragma unroll
            for (int x = 4; x < 124; x += 8) {
                a0 = fmax3(a0, s[x + 0], s[x + 1]);
                a1 = fmax3(a1, s[x + 2], s[x + 3]);
                a2 = fmax3(a2, s[x + 4], s[x + 5]);
                a3 = fmax3(a3, s[x + 6], s[x + 7]);
            }
            a0 = fmax3(a0, s[124], s[125]);
            a1 = fmax3(a1, s[126], s[127]);
            const float m_cand = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)) * scale2;
            bool rescale = false;
            float alpha = 1.f;
            if (j == 0) {
                m_run = m_cand;
            } else {
                const bool need = m_cand > m_run + kRescaleThreshold;
                if (__any_sync(0xffffffffu, need)) {
                    const float m_new = fmaxf(m_run, m_cand);
                    alpha = ex2(m_run - m_new);
                    l_run *= alpha;
                    m_run = m_new;
                    rescale = true;
                }
            }
            // x' - m on the packed FMA pipe; 2^(x' - m) on MUFU (VMB_EMU_PERIOD moves one pair in
            // that many to the FMA-pipe polynomial; off by default, profiles/r1_fa_variants.md);
            // packed row sums; P -> TMEM as bf16
            const uint64_t negm2 = pk2(-m_run, -m_run);
            const uint64_t* s2 = reinterpret_cast<const uint64_t*>(sr);
            uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t pk[16];
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                    const uint64_t t2 = ffma2(s2[cc * 16 + x], scale2x2, negm2);
                    uint64_t pp;
                    if ((x % VMB_EMU_PERIOD) == VMB_EMU_PERIOD - 1) pp = ex2_emu2(t2);
                    else pp = pk2(ex2(lo2(t2)), ex2(hi2(t2)));
                    switch (x & 3) {
                        case 0: acc0 = fadd2(acc0, pp); break;
                        case 1: acc1 = fadd2(acc1, pp); break;
                        case 2: acc2 = fadd2(acc2, pp); break;
                        default: acc3 = fadd2(acc3, pp); break;
                    }
                    pk[x] = pack_bf16(lo2(pp), hi2(pp));
                }
                VMB_TMEM_ST16(tS + cc * 16, pk);
            }
            const uint64_t acc = fadd2(fadd2(acc0, acc1), fadd2(acc2, acc3));
            l_run += lo2(acc) + hi2(acc);
            if (rescale) {
                // O must hold every earlier P V product before it is rescaled; P_j V is not
                // issued before this thread arrives on p_full
                mbar_wait_sleep(pv_done, (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int t = 0; t < NO; ++t) {
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        uint32_t orr[32];
                        const uint32_t ta = tO + t * 128 + cc * 32 + lane_base;
                        VMB_TMEM_LD32(ta, orr);
                        tmem_ld_wait();
#pragma unroll
                        for (int x = 0; x < 32; ++x) orr[x] = __float_as_uint(__uint_as_float(orr[x]) * alpha);
                        VMB_TMEM_ST32(ta, orr);
                    }
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[j & 1]);
        }

        // ------------------------------------------------------------ epilogue
        if (threadIdx.x == 128) TRACE(4);  // last P handed over
        mbar_wait_sleep(o_full, 0);
        if (threadIdx.x == 128) TRACE(5);  // O complete
        tc_fence_after();
        const float inv_l = 1.f / l_run;
        const int64_t ob = u / a.oHn, oh = u % a.oHn;
        float qo = 0.f;  // <q_row, sum_l p_l k_l>  (entropy, see below)
#pragma unroll
        for (int t = 0; t < NO; ++t) {
            __nv_bfloat16* out = static_cast<__nv_bfloat16*>(t == 0 ? a.out0 : a.out1);
            __nv_bfloat16* orow = out + ob * a.oB[t] + oh * a.oH[t] + (int64_t)seg * a.oS[t] +
                                  (int64_t)grow * a.oR[t];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t orr[32];
                VMB_TMEM_LD32(tO + t * 128 + cc * 32 + lane_base, orr);
                tmem_ld_wait();
                if (t == 0 && a.cl_out) {
                    // q row (bf16, SW128 panel cc/2) . O row, 32 columns
                    const uint8_t* qp = smem + SM::q_off + (cc >> 1) * kPanelBytes;
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const uint4 qv = *reinterpret_cast<const uint4*>(qp + sw128_offset(row, (cc & 1) * 32 + 8 * x));
                        const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            qo = fmaf(__uint_as_float(qw[e] << 16), __uint_as_float(orr[8 * x + 2 * e]), qo);
                            qo = fmaf(__uint_as_float(qw[e] & 0xFFFF0000u), __uint_as_float(orr[8 * x + 2 * e + 1]), qo);
                        }
                    }
                }
                uint4 v[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    v[x].x = pack_bf16(__uint_as_float(orr[8 * x + 0]) * inv_l, __uint_as_float(orr[8 * x + 1]) * inv_l);
                    v[x].y = pack_bf16(__uint_as_float(orr[8 * x + 2]) * inv_l, __uint_as_float(orr[8 * x + 3]) * inv_l);
                    v[x].z = pack_bf16(__uint_as_float(orr[8 * x + 4]) * inv_l, __uint_as_float(orr[8 * x + 5]) * inv_l);
                    v[x].w = pack_bf16(__uint_as_float(orr[8 * x + 6]) * inv_l, __uint_as_float(orr[8 * x + 7]) * inv_l);
                }
                if (a.o_tma) {
                    // stage the row in SW128 layout over the drained K/V ring (every MMA has
                    // completed once o_full fired); TMA bulk stores below
                    uint8_t* panel = smem + SM::kv_off + t * kTileBytes + (cc >> 1) * kPanelBytes;
#pragma unroll
                    for (int x = 0; x < 4; ++x)
                        *reinterpret_cast<uint4*>(panel + sw128_offset(row, (cc & 1) * 32 + 8 * x)) = v[x];
                } else if (valid) {
                    uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
                    for (int x = 0; x < 4; ++x) dst[x] = v[x];
                }
            }
        }
        if (threadIdx.x == 128) TRACE(6);  // O read out of TMEM + staged
        if (a.o_tma) {
            // coalesced epilogue: one thread stores the staged (128 x 128) tiles; rows beyond
            // q_len are clipped by the tensor maps (the scattered 16-B row stores of the
            // previous epilogue took 3.3 us per CTA, profiles/r1_fa_variants.md)
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (row == 0) {
#pragma unroll
                for (int t = 0; t < NO; ++t) {
                    const uint8_t* tile = smem + SM::kv_off + t * kTileBytes;
                    // out0 (aL): box (64, 1 frame, 128 rows) at (c, seg, row0);
                    // out1 (y) : box (64, 128 rows, 1 frame) at (c, row0, seg)
                    const int c1 = t == 0 ? seg : qtile * kTile, c2 = t == 0 ? qtile * kTile : seg;
                    tma_store_5d(&a.tmO[t], tile, 0, c1, c2, 0, u);
                    tma_store_5d(&a.tmO[t], tile + kPanelBytes, 64, c1, c2, 0, u);
                }
                tma_store_commit();
                tma_store_wait_read();
            }
        }
        if (valid) {
            const float lse2 = m_run + log2f(l_run);  // base-2 log-sum-exp of x' = s * scale2
            // sum_l R ln R = ln2 * (scale2 * sum_l R_l s_l - lse2), and in the R-step (value
            // operand = the key tile) sum_l R_l s_l = <q, sum_l R_l k_l> = qo / l: the entropy
            // of monarch.hpp:93-98 without a per-element accumulator.
            if (a.cl_out)
                a.cl_out[((int64_t)u * a.q_len + grow) * a.nseg + seg] = kLn2 * (scale2 * qo * inv_l - lse2);
            if (a.lse_out)
                a.lse_out[((int64_t)u * a.nseg + seg) * a.q_len + grow] = kLn2 * lse2;
        }
    }

    tc_fence_before();
    if (MC) cluster_sync();  // no CTA leaves while its peer may still multicast into it
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    if (threadIdx.x == 128) {
        TRACE(7);  // epilogue done, CTA exiting
    }
}

template <int NB, int NO, bool MC>
void launch(const Params& p, int64_t U, cudaStream_t s) {
    using SM = Smem<NB, NO>;
    auto kern = fa_tc_kernel<NB, NO, MC>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    unsigned qt = (unsigned)((p.a.q_len + kTile - 1) / kTile);
    if (MC) qt = (qt + 1) & ~1u;  // whole clusters; a padding CTA computes zero rows, stores nothing
    dim3 grid(qt, (unsigned)(U * p.a.nseg));
    ProfScope ps(NO == 2 ? kKRstepY : (NB == 1 ? kKRstep : kKAttn), s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = SM::alloc;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = MC ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VMB_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
    count_launch();
    check_launch("fa_tc");
}

}  // namespace

void tc_fa_launch(const TcFaArgs& a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.q_len == 0) return;
    VMB_REQUIRE_DIM(a.kv_len >= 1, "attention over empty keys");
    // the entropy output is derived from <q, P K>: the first value operand must be K
    VMB_REQUIRE_DIM(!a.cl_out || a.nv == 2 || a.v_is_k, "entropy output needs the key tile as value operand");
    Params p;
    p.a = a;
    p.n_kv_tiles = (a.kv_len + kTile - 1) / kTile;
    // 2-CTA multicast clusters only with VMB_FA_MC=1: measured slower on B200 (the two CTAs of
    // a cluster advance in lock-step; the L2 -> SMEM stream was not the binding limit),
    // profiles/r1_fa_variants.md
    static const bool mc = [] {
        const char* e = getenv("VMB_FA_MC");
        return e && e[0] == '1';
    }();
    if (a.nv == 2) {
        if (mc) launch<2, 2, true>(p, U, s);
        else launch<2, 2, false>(p, U, s);
    } else if (a.v_is_k) {
        if (mc) launch<1, 1, true>(p, U, s);
        else launch<1, 1, false>(p, U, s);
    }
    else VMB_REQUIRE_DIM(false, "fa_tc serves the R half-steps only");
}

}  // namespace vmb

#if VMB_TRACE
extern "C" int vmb_debug_trace_read(unsigned long long* host, int ctas) {
    const int n = ctas < 4096 ? ctas : 4096;
    return cudaMemcpyFromSymbol(host, vmb::g_trace, sizeof(unsigned long long) * 8 * n) == cudaSuccess ? n : -1;
}
#endif
