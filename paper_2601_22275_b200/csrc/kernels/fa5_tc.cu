// fa5_tc.cu — persistent FA4-style flash attention: two 128-row query tiles per work item
// with ping-pong softmax warpgroups, one CTA per SM looping over items (bf16, d = 128, one
// value operand).
//
// fa3 (two query tiles per CTA, profiles/r1_fa_variants.md) keeps the MUFU pipe busy --
// while warpgroup A runs tile A's softmax, the tensor pipe works on tile B -- and reaches
// ~74% of the N = 128 tcgen05 rate on long rows, but loses a third of every short R-step row
// (12 key tiles per CTA at C4) to per-CTA prologue/epilogue.  Here one CTA per SM walks a
// flattened stream of items (query-tile pair, unit*segment, kv-split):
//   * the Q pair is double-buffered (R-step: NB = 1), so the next item's Q load overlaps the
//     current item; a Q buffer is released once both warpgroups finished the item's epilogue
//     (their entropy dot reads q from it);
//   * key tiles of consecutive items flow through one TMA ring (flattened tile counter g);
//   * each softmax warpgroup drains its own O after the item's last PV and then starts the
//     next item -- its next P (which the next PV needs) is produced only after the drain, so
//     O needs no extra barrier, while the tensor pipe computes the other tile's last PV and
//     the next item's first S tiles.
// Modes: <NB = 1> R half-step (value = key: aL, cL); <NB = 2> attention (recompute, dense),
// optional split-KV with the fa2 LSE combine.
// TMEM: tile t at column 256*t: S_t [0,128) (P_t as bf16 over its first 64 columns), O_t [128,256).
#include <cuda_bf16.h>

#include <algorithm>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 320;
constexpr int kQTile = 128;
constexpr int kBN = 128;                        // keys per KV tile
constexpr uint32_t kPanel = 128 * 128;          // 128 rows x 64 bf16 (SW128)
constexpr uint32_t kTileBytes = 2 * kPanel;     // 128 x 128 bf16
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
// 2^x for an element pair on the FMA/ALU pipes: n = rint(x) via the 1.5*2^23 magic, 2^(x-n)
// by a degree-3 minimax polynomial on [-0.5, 0.5] (rel. err 1.1e-4, far below the bf16 P
// rounding), n added to the exponent field; x clamped at -126.
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

struct Params {
    Tc2Args a;
    int32_t n_kv_tiles;   // key tiles per split (the last split may own fewer)
    int32_t total_tiles;  // key tiles of the whole segment
    int32_t q_pairs;      // query-tile pairs per segment
    int32_t nsplit;       // key splits per segment
    int32_t n_items;      // q_pairs * nsplit * U * nseg (< 2^31)
};

struct Item {
    int pair, split, useg, u, seg, kv_tile0, n_kv;
};
__device__ __forceinline__ Item decode(const Params& p, uint32_t it) {
    Item r;
    r.pair = (int)(it % (uint32_t)p.q_pairs);
    const uint32_t rest = it / (uint32_t)p.q_pairs;
    r.split = (int)(rest % (uint32_t)p.nsplit);
    r.useg = (int)(rest / (uint32_t)p.nsplit);
    r.u = (int)((uint32_t)r.useg / (uint32_t)p.a.nseg);
    r.seg = (int)((uint32_t)r.useg % (uint32_t)p.a.nseg);
    r.kv_tile0 = r.split * p.n_kv_tiles;
    r.n_kv = min(p.n_kv_tiles, p.total_tiles - r.kv_tile0);
    return r;
}

template <int NB>
struct Smem {
    static constexpr int QB = NB == 1 ? 2 : 1;             // Q-pair buffers
    static constexpr int S = NB == 1 ? 3 : 2;              // KV stages
    static constexpr uint32_t q_off = 0;                   // [QB][Q_A, Q_B]
    static constexpr uint32_t kv_off = QB * 2 * kTileBytes;
    static constexpr uint32_t bar_off = kv_off + S * NB * kTileBytes;
    // q_full[2], q_empty[2], kv_full[S], kv_empty[S], s_full[2], p_full[2], o_full[2]
    static constexpr uint32_t n_bars = 4 + 2 * S + 6;
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t bytes = slot_off + 16;
    static_assert(bytes <= 232448, "shared memory budget (227 KB per CTA)");
    // the dynamic smem window starts 1024-aligned (checked in the kernel): no slack needed
    static constexpr uint32_t alloc = bytes;
};

#ifndef VMB_TRACE
#define VMB_TRACE 0
#endif
#if VMB_TRACE
// debug-only: [cta < 16][item 1..2][tile < 12][event] clock64 of warp 2 lane 0 (tile A row 0)
__device__ long long g_trace5[16][2][12][4];
#define TRACE5(n, j, ev) do { if (threadIdx.x == 64 && blockIdx.x < 16 && (n) >= 1 && (n) <= 2 && (j) < 12) \
    g_trace5[blockIdx.x][(n) - 1][(j)][(ev)] = clock64(); } while (0)
#else
#define TRACE5(n, j, ev) do { } while (0)
#endif

template <int NB>
__global__ void __launch_bounds__(kThreads, 1) fa5_kernel(const __grid_constant__ Params p) {
    using SM = Smem<NB>;
    constexpr int S = SM::S;
    constexpr int QB = SM::QB;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 operand tiles need 1024-B alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* q_full = bars;              // [2]
    uint64_t* q_empty = bars + 2;         // [2]
    uint64_t* kv_full = bars + 4;
    uint64_t* kv_empty = kv_full + S;
    uint64_t* s_full = kv_empty + S;      // [2]
    uint64_t* p_full = s_full + 2;        // [2]
    uint64_t* o_full = s_full + 4;        // [2]: tile t's O complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);

    const Tc2Args& a = p.a;
    const int warp = warp_id();

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        if (NB == 2) tma_prefetch_desc(&a.tmV);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 256);  // both softmax warpgroups, after the item's epilogue
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 128);
        }
        mbar_init(&o_full[0], 1);
        mbar_init(&o_full[1], 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            int64_t g = 0;
            int n = 0;
            for (uint32_t it = blockIdx.x; it < (uint32_t)p.n_items; it += gridDim.x, ++n) {
                const Item w = decode(p, it);
                const int qbuf = n % QB;
                if (n >= QB) mbar_wait_sleep(&q_empty[qbuf], ((n / QB) - 1) & 1);
                const int qb = w.u / a.qH, qh = w.u % a.qH;
                const int kb = w.u / a.kH, kh = w.u % a.kH;
                uint8_t* sq = smem + SM::q_off + qbuf * 2 * kTileBytes;
                mbar_arrive_expect_tx(&q_full[qbuf], 2 * kTileBytes);
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int row = (2 * w.pair + t) * kQTile;
                    tma_load_5d(sq + t * kTileBytes, &a.tmQ, &q_full[qbuf], 0, row, w.seg, qh, qb);
                    tma_load_5d(sq + t * kTileBytes + kPanel, &a.tmQ, &q_full[qbuf], 64, row, w.seg, qh, qb);
                }
                for (int j = 0; j < w.n_kv; ++j, ++g) {
                    const int st = (int)(g % S);
                    if (g >= S) mbar_wait_sleep(&kv_empty[st], ((g / S) + 1) & 1);
                    uint8_t* skv = smem + SM::kv_off + st * NB * kTileBytes;
                    const int row = (w.kv_tile0 + j) * kBN;
                    mbar_arrive_expect_tx(&kv_full[st], NB * kTileBytes);
                    tma_load_5d(skv, &a.tmK, &kv_full[st], 0, row, w.seg, kh, kb);
                    tma_load_5d(skv + kPanel, &a.tmK, &kv_full[st], 64, row, w.seg, kh, kb);
                    if (NB == 2) {
                        tma_load_5d(skv + kTileBytes, &a.tmV, &kv_full[st], 0, row, w.seg, kh, kb);
                        tma_load_5d(skv + kTileBytes + kPanel, &a.tmV, &kv_full[st], 64, row, w.seg, kh, kb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idS = idesc_bf16(128, kBN, 0, 0);   // S = Q K^T, both K-major
        constexpr uint32_t idPV = idesc_bf16(128, 128, 0, 1);  // O += P V, V MN-major
        const uint32_t q_addr0 = smem_u32(smem + SM::q_off);
        const uint32_t kv_addr = smem_u32(smem + SM::kv_off);
        if (elect_one()) {
            int64_t g = 0;  // flattened key-tile counter (stage ring, s_full / p_full phases)
            int n = 0;
            for (uint32_t it = blockIdx.x; it < (uint32_t)p.n_items; it += gridDim.x, ++n) {
                const Item w = decode(p, it);
                const int qbuf = n % QB;
                const uint32_t q_addr = q_addr0 + qbuf * 2 * kTileBytes;
                auto issue_s = [&](int t, int64_t gg) {
                    const uint32_t kaddr = kv_addr + (int)(gg % S) * NB * kTileBytes;
                    const uint32_t qa = q_addr + t * kTileBytes;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
                        umma_ss(tmem + t * 256, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(kaddr + off, 16, 1024),
                                idS, kk > 0);
                    }
                    umma_commit(&s_full[t]);
                };
                auto issue_pv = [&](int t, int64_t gg, bool first) {
                    const uint32_t vaddr = kv_addr + (int)(gg % S) * NB * kTileBytes + (NB == 2 ? kTileBytes : 0);
#pragma unroll
                    for (int kk = 0; kk < kBN / 16; ++kk)
                        umma_ts(tmem + t * 256 + 128, tmem + t * 256 + kk * 8,
                                sdesc_sw128(vaddr + kk * 2048, kPanel, 1024), idPV, (!first || kk > 0) ? 1u : 0u);
                };
                mbar_wait_sleep(&q_full[qbuf], (n / QB) & 1);
                mbar_wait_sleep(&kv_full[g % S], (g / S) & 1);
                tc_fence_after();
                issue_s(0, g);
                issue_s(1, g);
                for (int j = 0; j < w.n_kv; ++j, ++g) {
                    const bool more = j + 1 < w.n_kv;
                    // tile A
                    mbar_wait_sleep(&p_full[0], g & 1);
                    tc_fence_after();
                    issue_pv(0, g, j == 0);
                    if (!more) umma_commit(&o_full[0]);  // tile A's epilogue may start
                    if (more) {
                        mbar_wait_sleep(&kv_full[(g + 1) % S], ((g + 1) / S) & 1);
                        tc_fence_after();
                        issue_s(0, g + 1);
                    }
                    // tile B
                    mbar_wait_sleep(&p_full[1], g & 1);
                    tc_fence_after();
                    issue_pv(1, g, j == 0);
                    umma_commit(&kv_empty[g % S]);
                    if (!more) umma_commit(&o_full[1]);
                    if (more) issue_s(1, g + 1);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int t = (warp - 2) >> 2;                // query tile of this warpgroup
        const int row = (warp & 3) * 32 + lane_id();  // TMEM lane == query row in tile
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + t * 256 + lane_base, tO = tS + 128;
        int64_t g = 0;
        int n = 0;
        // per-row temperature source, loaded one item ahead (its latency hides under an item)
        auto load_c = [&](uint32_t it2) -> float {
            if (!a.cR || it2 >= (uint32_t)p.n_items) return 1.f;
            const Item w2 = decode(p, it2);
            const int gr = (2 * w2.pair + t) * kQTile + row;
            return gr < a.q_len ? __ldg(a.cR + ((int64_t)w2.u * a.nseg + w2.seg) * a.q_len + gr) : 1.f;
        };
        float c_next = load_c(blockIdx.x);
        for (uint32_t it = blockIdx.x; it < (uint32_t)p.n_items; it += gridDim.x, ++n) {
        const Item w = decode(p, it);
        const int u = w.u, seg = w.seg, useg = w.useg, split = w.split, n_kv = w.n_kv, kv_tile0 = w.kv_tile0;
        const int qbuf = n % QB;
        const int grow = (2 * w.pair + t) * kQTile + row;  // row within the segment
        const bool valid = grow < a.q_len;
        float c = c_next;
        c_next = load_c(it + gridDim.x);
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
        const uint8_t* qtile_smem = smem + SM::q_off + (qbuf * 2 + t) * kTileBytes;

        if (a.check_finite) {
            mbar_wait_sleep(&q_full[qbuf], (n / QB) & 1);
            bool bad = false;
#pragma unroll
            for (int pnl = 0; pnl < 2; ++pnl) {
                const uint4* q4 = reinterpret_cast<const uint4*>(qtile_smem + pnl * kPanel + row * 128);
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
        }

        float m_run = -INFINITY, l_run = 0.f;
        const uint64_t scale2x2 = pk2(scale2, scale2);
        for (int j = 0; j < n_kv; ++j, ++g) {
            TRACE5(n, j, 0);
            mbar_wait_sleep(&s_full[t], g & 1);
            TRACE5(n, j, 1);
            tc_fence_after();
#if VMB_DEBUG_NO_SOFTMAX  // timing experiment only: MMA/TMA pipeline without the softmax
            if (true) {
                mbar_arrive(&p_full[t]);
                continue;
            }
#endif
            uint32_t sr[kBN];
#pragma unroll
            for (int cc = 0; cc < kBN / 32; ++cc) VMB_TMEM_LD32(tS + cc * 32, (sr + cc * 32));
            tmem_ld_wait();
            float* s = reinterpret_cast<float*>(sr);
            if (j == n_kv - 1 && last_valid < kBN) {
                asm volatile("");  // keep this a real (rarely taken) branch, not 128 selects
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
            // x' - m on the packed FMA pipe, 2^(x' - m) on MUFU (VMB_EMU_PERIOD: FMA-pipe polynomial,
            // off by default); row sum in packed adds; P -> TMEM as bf16
            const uint64_t negm2 = pk2(-m_run, -m_run);
            const uint64_t* s2 = reinterpret_cast<const uint64_t*>(sr);
            uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
            for (int cc = 0; cc < kBN / 32; ++cc) {
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
                // S_t(j) was issued after PV_t(j-1): O_t is complete here
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t orr[32];
                    VMB_TMEM_LD32(tO + cc * 32, orr);
                    tmem_ld_wait();
#pragma unroll
                    for (int x = 0; x < 32; ++x) orr[x] = __float_as_uint(__uint_as_float(orr[x]) * alpha);
                    VMB_TMEM_ST32(tO + cc * 32, orr);
                }
            }
            TRACE5(n, j, 2);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[t]);
            TRACE5(n, j, 3);
        }

        // ------------------------------------------------------------ epilogue
        mbar_wait_sleep(&o_full[t], n & 1);
        tc_fence_after();
        const float inv_l = 1.f / l_run;
        const float lse2 = m_run + log2f(l_run);  // base-2 log-sum-exp of x' = s * scale2
        if (a.part_o) {
            // split-KV partial: normalised fp32 O and natural-log lse of this split
            float* prow = a.part_o + (((int64_t)useg * a.nsplit + split) * a.q_len + grow) * 128;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t orr[32];
                VMB_TMEM_LD32(tO + cc * 32, orr);
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
            float qo = 0.f;  // <q_row, O_row> (R-step entropy)
            const int64_t ob = u / a.oHn, oh = u % a.oHn;
            __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + ob * a.oB + oh * a.oH + (int64_t)seg * a.oS +
                                  (int64_t)grow * a.oR;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t orr[32];
                VMB_TMEM_LD32(tO + cc * 32, orr);
                tmem_ld_wait();
                if (a.cl_out) {
                    const uint8_t* qp = qtile_smem + (cc >> 1) * kPanel;
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
                if (valid) {
                    uint4 v[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        v[x].x = pack_bf16(__uint_as_float(orr[8 * x + 0]) * inv_l, __uint_as_float(orr[8 * x + 1]) * inv_l);
                        v[x].y = pack_bf16(__uint_as_float(orr[8 * x + 2]) * inv_l, __uint_as_float(orr[8 * x + 3]) * inv_l);
                        v[x].z = pack_bf16(__uint_as_float(orr[8 * x + 4]) * inv_l, __uint_as_float(orr[8 * x + 5]) * inv_l);
                        v[x].w = pack_bf16(__uint_as_float(orr[8 * x + 6]) * inv_l, __uint_as_float(orr[8 * x + 7]) * inv_l);
                    }
                    if (a.out_align32) {  // 256-bit stores: one full sector per instruction
                        st_global_256(orow + cc * 32, v[0], v[1]);
                        st_global_256(orow + cc * 32 + 16, v[2], v[3]);
                    } else {
                        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
                        for (int x = 0; x < 4; ++x) dst[x] = v[x];
                    }
                }
            }
            if (valid) {
                if (a.cl_out)
                    a.cl_out[((int64_t)u * a.q_len + grow) * a.nseg + seg] = kLn2 * (scale2 * qo * inv_l - lse2);
                if (a.lse_out) a.lse_out[((int64_t)u * a.nseg + seg) * a.q_len + grow] = kLn2 * lse2;
            }
        }
        // this item's Q pair may be reloaded (two items ahead) once both warpgroups are done
        mbar_arrive(&q_empty[qbuf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int NB>
void launch(const Params& p, cudaStream_t s) {
    using SM = Smem<NB>;
    auto kern = fa5_kernel<NB>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    int dev = 0, sms = 148;
    VMB_CHECK_CUDA(cudaGetDevice(&dev));
    VMB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::min<int>(p.n_items, sms);
    ProfScope ps(NB == 1 ? kKRstep : kKAttn, s);
    kern<<<(unsigned)grid, kThreads, SM::alloc, s>>>(p);
    count_launch();
    check_launch("fa5_tc");
}

}  // namespace

int tc5_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int max_split) {
    if (max_split <= 1 || q_len <= 0 || n_useg <= 0) return 1;
    const int64_t total_tiles = (kv_len + kBN - 1) / kBN;
    // ~8 items per SM so the persistent CTAs balance, >= 8 key tiles per split
    const int64_t base = ((q_len + 2 * kQTile - 1) / (2 * kQTile)) * n_useg;
    const int64_t want = (8 * 148 + base - 1) / base;
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)max_split, total_tiles / 8}));
    while (nsplit > 1 && ((total_tiles + nsplit - 1) / nsplit) * (nsplit - 1) >= total_tiles) --nsplit;
    return nsplit;
}

void tc5_fa_launch(Tc2Args a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.q_len == 0) return;
    VMB_REQUIRE_DIM(a.kv_len >= 1, "attention over empty keys");
    VMB_REQUIRE_DIM(!a.cl_out || a.nv == 1, "entropy output needs the key tile as value operand");
    Params p;
    p.q_pairs = (a.q_len + 2 * kQTile - 1) / (2 * kQTile);
    p.total_tiles = (a.kv_len + kBN - 1) / kBN;
    const int64_t n_useg = U * a.nseg;
    p.nsplit = a.part_o ? tc5_plan_splits(a.q_len, a.kv_len, n_useg, a.max_split) : 1;
    p.n_kv_tiles = (p.total_tiles + p.nsplit - 1) / p.nsplit;
    const int64_t items = (int64_t)p.q_pairs * p.nsplit * n_useg;
    VMB_REQUIRE_DIM(items < ((int64_t)1 << 31), "too many work items for one launch");
    p.n_items = (int32_t)items;
    a.nsplit = p.nsplit;
    a.n_useg = n_useg;
    a.out_align32 = rows_align32(a.out, a.oB, a.oH, a.oS, a.oR) ? 1 : 0;
    p.a = a;
    if (p.nsplit == 1) p.a.part_o = nullptr;
    if (a.nv == 1) launch<1>(p, s);
    else launch<2>(p, s);
    if (p.nsplit > 1) tc2_combine_launch(p.a, s);
}

}  // namespace vmb

#if VMB_TRACE
extern "C" int vmb_debug_trace5_read(long long* host) {
    return cudaMemcpyFromSymbol(host, vmb::g_trace5, sizeof(long long) * 16 * 2 * 12 * 4) == cudaSuccess ? 0 : -1;
}
#endif
