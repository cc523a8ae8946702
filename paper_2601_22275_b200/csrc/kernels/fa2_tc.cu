// fa2_tc.cu — tcgen05 flash attention with fused online statistics, two CTAs per SM
// (bf16, d = 128, one value operand).
//
// Serves:
//   * the R half-step (monarch.hpp:53-103): query = aR[k] (or Q on the first step), key =
//     value = Kb[k], per-row temperature 1/max(cR, clamp) folded into the softmax scale;
//     outputs aL rows (strided into (b,m,d)) and cL = sum_l R ln R.                   <NB=1>
//   * the first-frame recompute (flash_entropy.hpp:85-139, video.hpp:117-126) and the
//     dense baseline (oracle.hpp:36-72): query = Q rows, key/value = all keys, split over
//     the key axis (split-KV) with an LSE combine when the query tiles alone do not fill
//     the machine.                                                                     <NB=2>
//
// CTA = one 128-row query tile of one (unit, segment, kv-split).  192 threads:
//   warp 0      TMA producer: Q tile once, then a ring of KV stages
//   warp 1      TMEM allocator (256 columns) + single-thread tcgen05.mma issuer
//   warps 2-5   softmax / statistics / epilogue; thread owns query row (warp%4)*32 + lane
//               (TMEM lane restriction: warp w reaches lanes 32*(w%4) .. +31)
// Key tiles of 64 (BN): TMEM holds two S buffers [0,64) and [64,128) (fp32; P written back
// as bf16 over the first 32 columns of its buffer) and O [128, 256) -- 256 columns, so two
// CTAs share an SM.  S_{j+1} is issued before the issuer waits for P_j (overlap inside the
// CTA), and the SM's tensor pipe is shared by two CTAs whose softmax, prologue and epilogue
// phases interleave (the FA4 ping-pong, across CTAs instead of warpgroups).  The softmax
// uses packed FFMA2/FADD2 for x' - m and the row sum (half the FMA-pipe issue slots).
//
// Statistics: base 2 with a lazily-updated reference max (O and l rescaled only when the
// running max grows by more than 8).  The entropy of the R-step is not accumulated per
// element: with value = key, sum_l R_l s_l = <q, sum_l R_l k_l> = <q, O> / l, so
//   sum_l R ln R = ln2 * (scale2 * <q, O> / l - lse2)            (monarch.hpp:93-98)
// is one 128-term dot product in the epilogue.  Exponentials run on MUFU; the FMA-pipe
// polynomial for one pair in VMB_EMU_PERIOD is compiled in but off by default (measured: MUFU
// is not the binding unit, profiles/r1_fa_variants.md).
#include <cuda_bf16.h>

#include <algorithm>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr int kQTile = 128;
constexpr uint32_t kQPanel = 128 * 128;        // 128 rows x 64 bf16
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;
constexpr float kMasked = -1.0e30f;

#ifndef VMB_TRACE
#define VMB_TRACE 0
#endif
#if VMB_TRACE
// debug-only per-CTA timeline of the first 4096 CTAs of a launch: [cta][event] globaltimer (ns)
__device__ unsigned long long g_trace2[4096][8];
#define TRACE2(ev) do { if (blockIdx.x < 4096) { unsigned long long tt_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt_)); g_trace2[blockIdx.x][ev] = tt_; } } while (0)
#else
#define TRACE2(ev) do { } while (0)
#endif

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// 2^x for an element pair on the FMA/ALU pipes (FADD2/FFMA2 + integer exponent add; see fa3_tc.cu)
__device__ __forceinline__ uint64_t ex2_emu2(uint64_t x2);

struct Params {
    Tc2Args a;
    int32_t n_kv_tiles;   // key tiles per split (the last split may own fewer)
    int32_t total_tiles;  // key tiles of the whole segment
    int32_t q_tiles;
};

// packed fp32 pair arithmetic (FFMA2 / FADD2, sm_100)
__device__ __forceinline__ uint64_t ffma2(uint64_t x, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t x, uint64_t y) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
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
    const float x0 = fmaxf(lo2(x2), -126.f), x1 = fmaxf(hi2(x2), -126.f);
    const uint64_t xx = pk2(x0, x1);
    const uint64_t magic = pk2(12582912.f, 12582912.f), nmagic = pk2(-12582912.f, -12582912.f);
    const uint64_t t = fadd2(xx, magic);
    const uint64_t f = fadd2(xx, fadd2(nmagic, t) ^ 0x8000000080000000ull);  // x - (t - magic)
    uint64_t p = ffma2(pk2(0.05592203512787819f, 0.05592203512787819f), f,
                       pk2(0.24264007806777954f, 0.24264007806777954f));
    p = ffma2(p, f, pk2(0.6931210160255432f, 0.6931210160255432f));
    p = ffma2(p, f, pk2(0.9999244809150696f, 0.9999244809150696f));
    const uint32_t r0 = (uint32_t)p + ((uint32_t)t << 23);
    const uint32_t r1 = (uint32_t)(p >> 32) + ((uint32_t)(t >> 32) << 23);
    return (uint64_t)r0 | ((uint64_t)r1 << 32);
}

constexpr int kBN = 64;  // keys per KV tile (S tile = 128 x 64, double-buffered in TMEM)

// HL (the fp32 parity mode on tensor cores): every operand X arrives as two bf16 tensors
// X = hi + lo (hi = bf16(x), lo = bf16(x - hi): 16 mantissa bits), and each product is three
// bf16 MMA groups into one fp32 accumulator, A B ~ Ah Bh + Ah Bl + Al Bh (the dropped Al Bl is
// 2^-16 relative).  P goes to TMEM as hi (S columns [0,32)) and lo ([32,64)).  The lo tiles
// sit right after their hi tiles in shared memory; 192 KB, so one CTA per SM.
template <int NB, bool HL>
struct Smem {
    static constexpr int S = NB == 1 ? 4 : 2;             // KV stages
    static constexpr uint32_t kv_panel = kBN * 128;       // 64 rows x 64 bf16
    static constexpr uint32_t kv_tile = 2 * kv_panel;     // 64 x 128
    static constexpr uint32_t op_tile = HL ? 2 * kv_tile : kv_tile;  // one operand (hi [+ lo]) per stage
    static constexpr uint32_t q_off = 0;
    static constexpr uint32_t kv_off = (HL ? 4 : 2) * kQPanel;
    static constexpr uint32_t bar_off = kv_off + S * NB * op_tile;
    // q_full, kv_full[S], kv_empty[S], s_full[2], p_full[2], pv_done, o_full
    static constexpr uint32_t n_bars = 1 + 2 * S + 6;
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t bytes = slot_off + 16;
    static constexpr uint32_t alloc = bytes + 1024;
};

template <int NB, bool HL>
__global__ void __launch_bounds__(kThreads, HL ? 1 : 2) fa2_kernel(const __grid_constant__ Params p) {
    using SM = Smem<NB, HL>;
    constexpr int S = SM::S;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = bars + 1 + S;
    uint64_t* s_full = bars + 1 + 2 * S;   // [2]
    uint64_t* p_full = s_full + 2;         // [2]
    uint64_t* pv_done = s_full + 4;
    uint64_t* o_full = s_full + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);

    const Tc2Args& a = p.a;
    const int warp = warp_id();
    // 1-D grid, (useg, split, qtile) with qtile fastest: no 65535 limit on units x segments
    const int per = p.q_tiles * p.a.nsplit;
    const int useg = (int)(blockIdx.x / (unsigned)per);  // u * nseg + seg
    const int qtile = (int)(blockIdx.x % (unsigned)per) % p.q_tiles;
    const int split = (int)(blockIdx.x % (unsigned)per) / p.q_tiles;
    const int u = useg / a.nseg, seg = useg % a.nseg;
    const int kv_tile0 = split * p.n_kv_tiles;
    const int n_kv = min(p.n_kv_tiles, p.total_tiles - kv_tile0);

    if (threadIdx.x == 0 && !HL) TRACE2(0);
    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        if (NB == 2) tma_prefetch_desc(&a.tmV);
        if (HL) {
            tma_prefetch_desc(&a.tmQlo);
            tma_prefetch_desc(&a.tmKlo);
            if (NB == 2) tma_prefetch_desc(&a.tmVlo);
        }
        mbar_init(q_full, 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 128);
        }
        mbar_init(pv_done, 1);
        mbar_init(o_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS0 = tmem, tO = tmem + 128;   // S buffers at [0,64) and [64,128)

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            const int qb = u / a.qH, qh = u % a.qH;
            const int kb = u / a.kH, kh = u % a.kH;
            uint8_t* sq = smem + SM::q_off;
            mbar_arrive_expect_tx(q_full, (HL ? 4 : 2) * kQPanel);
            tma_load_5d(sq, &a.tmQ, q_full, 0, qtile * kQTile, seg, qh, qb);
            tma_load_5d(sq + kQPanel, &a.tmQ, q_full, 64, qtile * kQTile, seg, qh, qb);
            if (HL) {
                tma_load_5d(sq + 2 * kQPanel, &a.tmQlo, q_full, 0, qtile * kQTile, seg, qh, qb);
                tma_load_5d(sq + 3 * kQPanel, &a.tmQlo, q_full, 64, qtile * kQTile, seg, qh, qb);
            }
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % S;
                if (j >= S) mbar_wait_sleep(&kv_empty[st], ((j / S) + 1) & 1);
                uint8_t* skv = smem + SM::kv_off + st * NB * SM::op_tile;
                const int row = (kv_tile0 + j) * kBN;
                mbar_arrive_expect_tx(&kv_full[st], NB * SM::op_tile);
                auto load_op = [&](uint8_t* dst, const CUtensorMap* m) {
                    tma_load_5d(dst, m, &kv_full[st], 0, row, seg, kh, kb);
                    tma_load_5d(dst + SM::kv_panel, m, &kv_full[st], 64, row, seg, kh, kb);
                };
                load_op(skv, &a.tmK);
                if (HL) load_op(skv + SM::kv_tile, &a.tmKlo);
                if (NB == 2) {
                    load_op(skv + SM::op_tile, &a.tmV);
                    if (HL) load_op(skv + SM::op_tile + SM::kv_tile, &a.tmVlo);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // S_j = Q K_j^T into buffer j&1 is issued before waiting for P_{j-1}, so the tensor
        // pipe computes the next score tile while the softmax warps work on the current one.
        constexpr uint32_t idS = idesc_bf16(128, kBN, 0, 0);   // S = Q K^T, both K-major
        constexpr uint32_t idPV = idesc_bf16(128, 128, 0, 1);  // O += P V, V MN-major
        const uint32_t q_addr = smem_u32(smem + SM::q_off);
        const uint32_t kv_addr = smem_u32(smem + SM::kv_off);
        if (elect_one()) {
            mbar_wait_sleep(q_full, 0);
            for (int j = 0; j <= n_kv; ++j) {
                if (j < n_kv) {
                    const int st = j % S;
                    mbar_wait_sleep(&kv_full[st], (j / S) & 1);
                    tc_fence_after();
                    const uint32_t kaddr = kv_addr + st * NB * SM::op_tile;
                    const uint32_t tS = tS0 + (j & 1) * kBN;
                    // HL: Qh Kh + Qh Kl + Ql Kh
#pragma unroll
                    for (int gr = 0; gr < (HL ? 3 : 1); ++gr) {
                        const uint32_t qa = q_addr + (gr == 2 ? 2 * kQPanel : 0);
                        const uint32_t ka = kaddr + (gr == 1 ? SM::kv_tile : 0);
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            umma_ss(tS, sdesc_sw128(qa + (kk >> 2) * kQPanel + (kk & 3) * 32, 16, 1024),
                                    sdesc_sw128(ka + (kk >> 2) * SM::kv_panel + (kk & 3) * 32, 16, 1024), idS,
                                    (gr > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&s_full[j & 1]);
                }
                if (j >= 1) {
                    const int jp = j - 1, st = jp % S;
                    mbar_wait_sleep(&p_full[jp & 1], (jp >> 1) & 1);
                    tc_fence_after();
                    const uint32_t vaddr = kv_addr + st * NB * SM::op_tile + (NB == 2 ? SM::op_tile : 0);
                    const uint32_t tP = tS0 + (jp & 1) * kBN;
                    // HL: Ph Vh + Ph Vl + Pl Vh (P lo in the S buffer's columns [32, 64))
#pragma unroll
                    for (int gr = 0; gr < (HL ? 3 : 1); ++gr) {
                        const uint32_t pa = tP + (gr == 2 ? kBN / 2 : 0);
                        const uint32_t va = vaddr + (gr == 1 ? SM::kv_tile : 0);
#pragma unroll
                        for (int kk = 0; kk < kBN / 16; ++kk) {
                            umma_ts(tO, pa + kk * 8, sdesc_sw128(va + kk * 2048, SM::kv_panel, 1024), idPV,
                                    (jp > 0 || gr > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&kv_empty[st]);
                    umma_commit(pv_done);
                }
            }
            umma_commit(o_full);
        }
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int row = (warp & 3) * 32 + lane_id();  // TMEM lane == query row in tile
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const int grow = qtile * kQTile + row;        // row within the segment
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
        // valid keys in this CTA's last tile (only the globally last tile is ragged)
        const int kv_end = (kv_tile0 + n_kv) * kBN;
        const int last_valid = kBN - (kv_end > a.kv_len ? kv_end - a.kv_len : 0);

        if (a.check_finite) {
            mbar_wait_sleep(q_full, 0);
            bool bad = false;
#pragma unroll
            for (int pnl = 0; pnl < 2; ++pnl) {
                const uint4* q4 = reinterpret_cast<const uint4*>(smem + SM::q_off + pnl * kQPanel + row * 128);
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const uint4 v = q4[x ^ (row & 7)];  // rotate chunks across lanes: no bank conflicts
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        bad |= ((w[e] & 0x7F80u) == 0x7F80u) || ((w[e] & 0x7F800000u) == 0x7F800000u);
                }
            }
            if (bad && valid) atomicExch(a.status, kStatusNonFiniteQ);
            if (a.qn_out) {
                // max |Q row|^2 of the unit (bounds the L-step logits; nonnegative floats order as ints)
                float ss = 0.f;
#pragma unroll
                for (int pnl = 0; pnl < 2; ++pnl) {
                    const uint4* q4 = reinterpret_cast<const uint4*>(smem + SM::q_off + pnl * kQPanel + row * 128);
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        const uint4 v = q4[x ^ (row & 7)];
                        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float lo = __uint_as_float(w[e] << 16), hi = __uint_as_float(w[e] & 0xFFFF0000u);
                            ss = fmaf(lo, lo, fmaf(hi, hi, ss));
                        }
                    }
                }
                // per spatial position i = row: the max over frames of |Q row|^2 (nonnegative floats
                // order as ints); the L-step block of position i has exactly these rows as queries
                if (valid && !bad)
                    atomicMax(reinterpret_cast<unsigned*>(a.qn_out) + (int64_t)u * a.q_len + grow, __float_as_uint(ss));
            }
        }

        float m_run = -INFINITY, l_run = 0.f;
        const uint64_t scale2x2 = pk2(scale2, scale2);
        if (threadIdx.x == 64 && !HL) TRACE2(1);
        for (int j = 0; j < n_kv; ++j) {
            const uint32_t tS = tS0 + (j & 1) * kBN + lane_base;
            mbar_wait_sleep(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 64 && !HL && j == 0) TRACE2(2);
#if VMB_DEBUG_NO_SOFTMAX  // timing experiment only: MMA/TMA pipeline without the softmax
            if (true) {
                mbar_arrive(&p_full[j & 1]);
                continue;
            }
#endif
            uint32_t sr[kBN];
            VMB_TMEM_LD32(tS + 0, (sr + 0));
            VMB_TMEM_LD32(tS + 32, (sr + 32));
            tmem_ld_wait();
            float* s = reinterpret_cast<float*>(sr);
            if (j == n_kv - 1 && last_valid < kBN) {
                asm volatile("");  // keep this a real (rarely taken) branch, not 64 selects
#pragma unroll
                for (int x = 0; x < kBN; ++x)
                    if (x >= last_valid) s[x] = kMasked;
            }
            // row max: 4 independent FMNMX3 chains
            float a0 = s[0], a1 = s[1], a2 = s[2], a3 = s[3];
#pragma unroll
            for (int x = 4; x < kBN - 4; x += 8) {
                a0 = fmax3(a0, s[x + 0], s[x + 1]);
                a1 = fmax3(a1, s[x + 2], s[x + 3]);
                a2 = fmax3(a2, s[x + 4], s[x + 5]);
                a3 = fmax3(a3, s[x + 6], s[x + 7]);
            }
            a0 = fmax3(a0, s[kBN - 4], s[kBN - 3]);
            a1 = fmax3(a1, s[kBN - 2], s[kBN - 1]);
            const float m_cand = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)) * scale2;
            // lazy rescale decision; O itself is rescaled after P is stored (s[] dead by then)
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
            // x' - m for element pairs on the packed FMA pipe, then 2^(x' - m): MUFU for 7 of
            // every 8 pairs, the FMA-pipe polynomial for the 8th
            const uint64_t negm2 = pk2(-m_run, -m_run);
            const uint64_t* s2 = reinterpret_cast<const uint64_t*>(sr);
            uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
            uint32_t pk[kBN / 2];
#pragma unroll
            for (int x = 0; x < kBN / 2; ++x) {
                const uint64_t t2 = ffma2(s2[x], scale2x2, negm2);
                uint64_t pp;
                if ((x % VMB_EMU_PERIOD) == VMB_EMU_PERIOD - 1) pp = ex2_emu2(t2);
                else pp = pk2(ex2(lo2(t2)), ex2(hi2(t2)));
                const float p0 = lo2(pp), p1 = hi2(pp);
                switch (x & 3) {
                    case 0: acc0 = fadd2(acc0, pp); break;
                    case 1: acc1 = fadd2(acc1, pp); break;
                    case 2: acc2 = fadd2(acc2, pp); break;
                    default: acc3 = fadd2(acc3, pp); break;
                }
                pk[x] = pack_bf16(p0, p1);
                if (HL) reinterpret_cast<uint64_t*>(sr)[x] = pp;  // s is dead: keep p for the lo half
            }
            VMB_TMEM_ST16(tS + 0, (pk + 0));
            VMB_TMEM_ST16(tS + 16, (pk + 16));
            if (HL) {
                // P lo = bf16(p - bf16(p)) over the S columns [32, 64) (already in registers)
#pragma unroll
                for (int x = 0; x < kBN / 2; ++x) {
                    const uint64_t pp = reinterpret_cast<const uint64_t*>(sr)[x];
                    pk[x] = pack_bf16_residual(lo2(pp), hi2(pp), pk[x]);
                }
                VMB_TMEM_ST16(tS + 32, (pk + 0));
                VMB_TMEM_ST16(tS + 48, (pk + 16));
            }
            const uint64_t acc = fadd2(fadd2(acc0, acc1), fadd2(acc2, acc3));
            l_run += lo2(acc) + hi2(acc);
            if (rescale) {
                // O must hold P_{j-1} V_{j-1} before it is rescaled; P_j V_j waits for p_full
                mbar_wait_sleep(pv_done, (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t orr[32];
                    const uint32_t ta = tO + cc * 32 + lane_base;
                    VMB_TMEM_LD32(ta, orr);
                    tmem_ld_wait();
#pragma unroll
                    for (int x = 0; x < 32; ++x) orr[x] = __float_as_uint(__uint_as_float(orr[x]) * alpha);
                    VMB_TMEM_ST32(ta, orr);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[j & 1]);
        }

        // ------------------------------------------------------------ epilogue
        if (threadIdx.x == 64 && !HL) TRACE2(3);
        mbar_wait_sleep(o_full, 0);
        tc_fence_after();
        if (threadIdx.x == 64 && !HL) TRACE2(4);
        const float inv_l = 1.f / l_run;
        const float lse2 = m_run + log2f(l_run);  // base-2 log-sum-exp of x' = s * scale2
        float qo = 0.f;                            // <q_row, O_row> (R-step entropy)
        if (a.part_o) {
            // split-KV partial: normalised fp32 O and natural-log lse of this split
            float* prow = a.part_o + (((int64_t)useg * a.nsplit + split) * a.q_len + grow) * 128;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t orr[32];
                VMB_TMEM_LD32(tO + cc * 32 + lane_base, orr);
                tmem_ld_wait();
                if (valid) {
                    // fp32 partial rows (512 B, 32-B aligned workspace): 256-bit stores
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        uint4 lo, hi;
                        lo.x = __float_as_uint(__uint_as_float(orr[8 * x + 0]) * inv_l);
                        lo.y = __float_as_uint(__uint_as_float(orr[8 * x + 1]) * inv_l);
                        lo.z = __float_as_uint(__uint_as_float(orr[8 * x + 2]) * inv_l);
                        lo.w = __float_as_uint(__uint_as_float(orr[8 * x + 3]) * inv_l);
                        hi.x = __float_as_uint(__uint_as_float(orr[8 * x + 4]) * inv_l);
                        hi.y = __float_as_uint(__uint_as_float(orr[8 * x + 5]) * inv_l);
                        hi.z = __float_as_uint(__uint_as_float(orr[8 * x + 6]) * inv_l);
                        hi.w = __float_as_uint(__uint_as_float(orr[8 * x + 7]) * inv_l);
                        st_global_256(prow + cc * 32 + 8 * x, lo, hi);
                    }
                }
            }
            if (valid) a.part_lse[((int64_t)useg * a.nsplit + split) * a.q_len + grow] = kLn2 * lse2;
        } else {
            const int64_t ob = u / a.oHn, oh = u % a.oHn;
            __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + ob * a.oB + oh * a.oH + (int64_t)seg * a.oS +
                                  (int64_t)grow * a.oR;
            float ssa = 0.f;  // |output row|^2 (aln_out)
            // bf16 rows in packed pairs (FMUL2 / FFMA2): the epilogue shares issue slots with the
            // other CTA's softmax warps on the SM
            uint64_t ss2 = 0, qo2 = 0;
            const uint64_t inv2 = pk2(inv_l, inv_l);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t orr[32];
                VMB_TMEM_LD32(tO + cc * 32 + lane_base, orr);
                tmem_ld_wait();
                const uint64_t* o2 = reinterpret_cast<const uint64_t*>(orr);
                if (!HL && a.cl_out) {
                    const uint8_t* qp = smem + SM::q_off + (cc >> 1) * kQPanel;
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const uint4 qv = *reinterpret_cast<const uint4*>(qp + sw128_offset(row, (cc & 1) * 32 + 8 * x));
                        const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            qo2 = ffma2((uint64_t)(qw[e] << 16) | ((uint64_t)(qw[e] & 0xFFFF0000u) << 32), o2[4 * x + e], qo2);
                    }
                } else if (a.cl_out) {
#pragma unroll
                    for (int hl = 0; hl < (HL ? 2 : 1); ++hl) {  // HL: q = q_hi + q_lo
                        const uint8_t* qp = smem + SM::q_off + (2 * hl + (cc >> 1)) * kQPanel;
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
                }
                if (HL && a.out_f32) {
                    // fp32 output rows (element strides in floats)
                    if (valid) {
                        float* frow = static_cast<float*>(a.out) + ob * a.oB + oh * a.oH + (int64_t)seg * a.oS +
                                      (int64_t)grow * a.oR + cc * 32;
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            uint4 lo, hi;
                            lo.x = __float_as_uint(__uint_as_float(orr[8 * x + 0]) * inv_l);
                            lo.y = __float_as_uint(__uint_as_float(orr[8 * x + 1]) * inv_l);
                            lo.z = __float_as_uint(__uint_as_float(orr[8 * x + 2]) * inv_l);
                            lo.w = __float_as_uint(__uint_as_float(orr[8 * x + 3]) * inv_l);
                            hi.x = __float_as_uint(__uint_as_float(orr[8 * x + 4]) * inv_l);
                            hi.y = __float_as_uint(__uint_as_float(orr[8 * x + 5]) * inv_l);
                            hi.z = __float_as_uint(__uint_as_float(orr[8 * x + 6]) * inv_l);
                            hi.w = __float_as_uint(__uint_as_float(orr[8 * x + 7]) * inv_l);
                            if (a.out_align32) {
                                st_global_256(frow + 8 * x, lo, hi);
                            } else {
                                reinterpret_cast<uint4*>(frow + 8 * x)[0] = lo;
                                reinterpret_cast<uint4*>(frow + 8 * x)[1] = hi;
                            }
                        }
                    }
                } else if (valid) {
                    uint64_t nrm[16];
                    uint32_t w16[16];
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        ss2 = ffma2(o2[x], o2[x], ss2);
                        nrm[x] = fmul2(o2[x], inv2);
                        w16[x] = pack_bf16(lo2(nrm[x]), hi2(nrm[x]));
                    }
                    uint4 v[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) v[x] = make_uint4(w16[4 * x], w16[4 * x + 1], w16[4 * x + 2], w16[4 * x + 3]);
                    if (a.out_align32) {  // 256-bit stores: one full sector per instruction
                        st_global_256(orow + cc * 32, v[0], v[1]);
                        st_global_256(orow + cc * 32 + 16, v[2], v[3]);
                    } else {
                        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
                        for (int x = 0; x < 4; ++x) dst[x] = v[x];
                    }
                    if (a.out_lo) {
                        // low half of aL (same layout): bf16(x - bf16(x)), the residual in packed pairs
#pragma unroll
                        for (int x = 0; x < 16; ++x) {
                            const uint64_t hi2v = (uint64_t)(w16[x] << 16) | ((uint64_t)(w16[x] & 0xFFFF0000u) << 32);
                            const uint64_t r2 = fadd2(nrm[x], hi2v ^ 0x8000000080000000ull);
                            w16[x] = pack_bf16(lo2(r2), hi2(r2));
                        }
#pragma unroll
                        for (int x = 0; x < 4; ++x) v[x] = make_uint4(w16[4 * x], w16[4 * x + 1], w16[4 * x + 2], w16[4 * x + 3]);
                        __nv_bfloat16* lrow = static_cast<__nv_bfloat16*>(a.out_lo) + (orow - static_cast<__nv_bfloat16*>(a.out));
                        if (a.out_align32) {
                            st_global_256(lrow + cc * 32, v[0], v[1]);
                            st_global_256(lrow + cc * 32 + 16, v[2], v[3]);
                        } else {
                            uint4* dst = reinterpret_cast<uint4*>(lrow + cc * 32);
#pragma unroll
                            for (int x = 0; x < 4; ++x) dst[x] = v[x];
                        }
                    }
                }
            }
            if (!HL) qo += lo2(qo2) + hi2(qo2);
            ssa = (lo2(ss2) + hi2(ss2)) * (inv_l * inv_l);
            if (valid) {
                if (a.cl_out)
                    a.cl_out[((int64_t)u * a.q_len + grow) * a.nseg + seg] = kLn2 * (scale2 * qo * inv_l - lse2);
                if (a.aln_out) a.aln_out[((int64_t)u * a.q_len + grow) * a.nseg + seg] = sqrtf(ssa);
                if (a.lse_out) a.lse_out[((int64_t)u * a.nseg + seg) * a.q_len + grow] = kLn2 * lse2;
            }
        }
    }

    if (threadIdx.x == 64 && !HL) TRACE2(5);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0 && !HL) TRACE2(6);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

// ---------------------------------------------------------------- split-KV combine
// O[r] = sum_s w_s O_s / sum_s w_s, w_s = exp(lse_s - max lse): one warp per row.
__global__ void __launch_bounds__(256) fa2_combine_kernel(const Tc2Args a) {
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t rows = (int64_t)a.q_len;
    const int64_t useg = gw / rows, r = gw % rows;
    if (useg >= a.n_useg) return;
    const int u = (int)(useg / a.nseg), seg = (int)(useg % a.nseg);
    const float* lse = a.part_lse + (useg * a.nsplit) * rows + r;
    // all split statistics and partial rows are loaded up front (independent loads in flight,
    // registers: nsplit <= kTc2MaxSplit), then reduced in split order
    float ls[kTc2MaxSplit];
    float4 pv[kTc2MaxSplit];
    float mx = -INFINITY;
#pragma unroll
    for (int s = 0; s < kTc2MaxSplit; ++s) {
        ls[s] = s < a.nsplit ? lse[(int64_t)s * rows] : -INFINITY;
        pv[s] = s < a.nsplit
                    ? reinterpret_cast<const float4*>(a.part_o + ((useg * a.nsplit + s) * rows + r) * 128)[lane]
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int s = 0; s < kTc2MaxSplit; ++s) mx = fmaxf(mx, ls[s]);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float wsum = 0.f;
#pragma unroll
    for (int s = 0; s < kTc2MaxSplit; ++s) {
        if (s >= a.nsplit) break;
        const float w = __expf(ls[s] - mx);
        wsum += w;
        acc.x = fmaf(w, pv[s].x, acc.x);
        acc.y = fmaf(w, pv[s].y, acc.y);
        acc.z = fmaf(w, pv[s].z, acc.z);
        acc.w = fmaf(w, pv[s].w, acc.w);
    }
    const float inv = 1.f / wsum;
    if (a.ent_out && lane == 0) {
        // H = sum_s w_s (H_s - ln w_s), w_s = exp(lse_s - lse) (fa3 split-KV with entropy)
        const float lse_all = mx + logf(wsum);
        const float* pe = a.part_ent + (useg * a.nsplit) * rows + r;
        float h = 0.f;
        for (int s = 0; s < a.nsplit; ++s) {
            const float ls = lse[(int64_t)s * rows];
            const float w = __expf(ls - lse_all);
            h += w * (pe[(int64_t)s * rows] - (ls - lse_all));
        }
        a.ent_out[useg * rows + r] = h;
    }
    const int64_t ob = u / a.oHn, oh = u % a.oHn;
    if (a.out_f32) {
        float* frow = static_cast<float*>(a.out) + ob * a.oB + oh * a.oH + (int64_t)seg * a.oS + r * a.oR;
        reinterpret_cast<float4*>(frow)[lane] = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        if (a.lse_out && lane == 0) a.lse_out[useg * rows + r] = mx + logf(wsum);
        return;
    }
    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + ob * a.oB + oh * a.oH + (int64_t)seg * a.oS + r * a.oR;
    uint2 v;
    v.x = pack_bf16(acc.x * inv, acc.y * inv);
    v.y = pack_bf16(acc.z * inv, acc.w * inv);
    reinterpret_cast<uint2*>(orow)[lane] = v;
    if (a.lse_out && lane == 0) a.lse_out[useg * rows + r] = mx + logf(wsum);
}

template <int NB, bool HL>
void launch(const Params& p, int64_t n_useg, int nsplit, cudaStream_t s) {
    using SM = Smem<NB, HL>;
    static_assert(SM::alloc <= 232448, "shared memory budget (227 KB per CTA)");
    auto kern = fa2_kernel<NB, HL>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    VMB_REQUIRE_DIM((int64_t)p.q_tiles * nsplit * n_useg <= (int64_t)INT32_MAX, "attention grid too large");
    const dim3 grid((unsigned)((int64_t)p.q_tiles * nsplit * n_useg));
    ProfScope ps(NB == 1 ? kKRstep : kKAttn, s);
    kern<<<grid, kThreads, SM::alloc, s>>>(p);
    count_launch();
    check_launch("fa2_tc");
}

}  // namespace

int tc2_kv_tile(int) { return kBN; }

int tc2_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int nv, int max_split) {
    if (max_split <= 1 || q_len <= 0 || n_useg <= 0) return 1;
    const int64_t BN = tc2_kv_tile(nv);
    const int64_t total_tiles = (kv_len + BN - 1) / BN;
    // enough CTAs for ~8 waves of 2 CTAs per SM, and at least 8 key tiles per split
    const int64_t base = ((q_len + kQTile - 1) / kQTile) * n_useg;
    const int64_t want = (8 * 2 * 148 + base - 1) / base;
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)max_split, total_tiles / 8}));
    // no empty splits
    while (nsplit > 1 && ((total_tiles + nsplit - 1) / nsplit) * (nsplit - 1) >= total_tiles) --nsplit;
    return nsplit;
}

void tc2_fa_launch(Tc2Args a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.q_len == 0) return;
    VMB_REQUIRE_DIM(a.kv_len >= 1, "attention over empty keys");
    VMB_REQUIRE_DIM(!a.cl_out || a.nv == 1, "entropy output needs the key tile as value operand");
    const int BN = tc2_kv_tile(a.nv);
    Params p;
    p.q_tiles = (a.q_len + kQTile - 1) / kQTile;
    const int total_tiles = (a.kv_len + BN - 1) / BN;
    const int64_t n_useg = U * a.nseg;
    const int nsplit = a.part_o ? tc2_plan_splits(a.q_len, a.kv_len, n_useg, a.nv, a.max_split) : 1;
    p.n_kv_tiles = (total_tiles + nsplit - 1) / nsplit;
    p.total_tiles = total_tiles;
    a.nsplit = nsplit;
    a.n_useg = n_useg;
    // 32-byte rows: 16 bf16 or 8 fp32 elements per stride unit
    a.out_align32 = (a.out_f32 ? (reinterpret_cast<uintptr_t>(a.out) % 32 == 0 && a.oB % 8 == 0 && a.oH % 8 == 0 &&
                                  a.oS % 8 == 0 && a.oR % 8 == 0)
                               : rows_align32(a.out, a.oB, a.oH, a.oS, a.oR)) &&
                    (!a.out_lo || reinterpret_cast<uintptr_t>(a.out_lo) % 32 == 0) ? 1 : 0;
    VMB_REQUIRE_DIM(!a.out_f32 || a.hilo, "fp32 output rows need the hi/lo (fp32 parity) instantiation");
    p.a = a;
    if (nsplit == 1) p.a.part_o = nullptr;
    if (a.hilo) {
        if (a.nv == 1) launch<1, true>(p, n_useg, nsplit, s);
        else launch<2, true>(p, n_useg, nsplit, s);
    } else {
        if (a.nv == 1) launch<1, false>(p, n_useg, nsplit, s);
        else launch<2, false>(p, n_useg, nsplit, s);
    }
    if (nsplit > 1) tc2_combine_launch(p.a, s);
}

void tc2_combine_launch(const Tc2Args& a, cudaStream_t s) {
    const int64_t warps = a.n_useg * a.q_len;
    ProfScope ps(kKCombine, s);
    fa2_combine_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(a);
    count_launch();
    check_launch("fa2_combine");
}

}  // namespace vmb

#if VMB_TRACE
extern "C" int vmb_debug_trace2_read(unsigned long long* host) {
    return cudaMemcpyFromSymbol(host, vmb::g_trace2, sizeof(unsigned long long) * 4096 * 8) == cudaSuccess ? 0 : -1;
}
#endif
