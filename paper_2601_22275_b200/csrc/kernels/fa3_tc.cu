// fa3_tc.cu — tcgen05 flash attention, two query tiles per CTA with ping-pong softmax
// warpgroups (bf16, d = 128, one value operand).  The main attention kernel of the path.
//
// Serves:
//   * the R half-step (monarch.hpp:53-103): query = aR[k] (or Q on the first step), key =
//     value = Kb[k], per-row temperature 1/max(cR, clamp) folded into the softmax scale;
//     outputs aL rows (strided into (b,m,d)) and cL = sum_l R ln R.                   <NB=1>
//   * the first-frame recompute (flash_entropy.hpp:85-139, video.hpp:117-126) and the
//     dense baseline (oracle.hpp:36-72): query = Q rows, key/value = all keys, split over
//     the key axis with an LSE combine when the query tiles do not fill the machine. <NB=2>
//
// Why this shape (profiles/r1_micro_tcgen05.md): a tcgen05.mma costs >= ~80 cycles whatever
// its N, so score tiles use N = 128 keys (N = 64 runs at half rate); the MUFU pipe gives 16
// exp/clk/SM, i.e. a 128x128 score tile needs 1024 MUFU cycles against 1292 tensor cycles
// for S + PV.  Two 128-row query tiles (A, B) share every K/V stage; while warpgroup A runs
// the softmax of tile A the tensor pipe works on tile B and vice versa (FA4 ping-pong).
//
// CTA = query tiles (2p, 2p+1) of one (unit, segment, kv-split).  320 threads:
//   warp 0      TMA producer: both Q tiles once, then a ring of K (or K,V) stages
//   warp 1      TMEM allocator (512 columns) + single-thread tcgen05.mma issuer
//   warps 2-5   softmax / epilogue of tile A, warps 6-9 of tile B; a thread owns query row
//               (warp%4)*32 + lane (TMEM lane restriction: warp w reaches lanes 32*(w%4)..)
// TMEM: tile t at column 256*t: S_t [0,128) fp32 (P_t written back as bf16 over its first
// 64 columns), O_t [128, 256).
// Issue order per key tile j:  PV_A(j), S_A(j+1), PV_B(j), S_B(j+1).  S_t(j+1) follows
// PV_t(j) in the in-order tcgen05 pipeline, so (i) P_t(j) is consumed before S_t(j+1)
// overwrites it and (ii) once a softmax warp sees S_t(j+1) complete, O_t holds every
// earlier P V product -- the lazy O rescale needs no extra barrier.
//
// Statistics: base 2 with a lazily-updated reference max (O and l rescaled only when the
// running max grows by more than 8).  The R-step entropy uses value = key:
//   sum_l R ln R = ln2 * (scale2 * <q, O> / l - lse2)            (monarch.hpp:93-98)
// one 128-term dot product in the epilogue instead of a per-element accumulator.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

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
    int32_t q_pairs;      // CTAs (tile pairs) per segment
};

template <int NB>
struct Smem {
    static constexpr int S = NB == 1 ? 3 : 2;              // KV stages
    static constexpr uint32_t q_off = 0;                   // Q_A, Q_B
    static constexpr uint32_t kv_off = 2 * kTileBytes;
    static constexpr uint32_t bar_off = kv_off + S * NB * kTileBytes;
    // q_full, kv_full[S], kv_empty[S], s_full[2], p_full[2], o_full
    static constexpr uint32_t n_bars = 1 + 2 * S + 5;
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    static constexpr uint32_t bytes = slot_off + 16;
    static constexpr uint32_t alloc = bytes + 1024;
};

// ENT: also the row entropy H = -sum P ln P = ln2 (lse2 - sum_l 2^(x'_l - m) x'_l / l) in
// base-2 units x' (flash_entropy.hpp:30-45, 137): one more packed FMA per element pair.
template <int NB, bool ENT>
__global__ void __launch_bounds__(kThreads, 1) fa3_kernel(const __grid_constant__ Params p) {
    using SM = Smem<NB>;
    constexpr int S = SM::S;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = bars + 1 + S;
    uint64_t* s_full = bars + 1 + 2 * S;  // [2]
    uint64_t* p_full = s_full + 2;        // [2]
    uint64_t* o_full = s_full + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);

    const Tc2Args& a = p.a;
    const int warp = warp_id();
    const int pair = blockIdx.x % p.q_pairs;
    const int split = blockIdx.x / p.q_pairs;
    const int useg = blockIdx.y;  // u * nseg + seg
    const int u = useg / a.nseg, seg = useg % a.nseg;
    const int kv_tile0 = split * p.n_kv_tiles;
    const int n_kv = min(p.n_kv_tiles, p.total_tiles - kv_tile0);

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        if (NB == 2) tma_prefetch_desc(&a.tmV);
        mbar_init(q_full, 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 128);
        }
        mbar_init(o_full, 1);
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
            const int qb = u / a.qH, qh = u % a.qH;
            const int kb = u / a.kH, kh = u % a.kH;
            uint8_t* sq = smem + SM::q_off;
            mbar_arrive_expect_tx(q_full, 2 * kTileBytes);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int row = (2 * pair + t) * kQTile;
                tma_load_5d(sq + t * kTileBytes, &a.tmQ, q_full, 0, row, seg, qh, qb);
                tma_load_5d(sq + t * kTileBytes + kPanel, &a.tmQ, q_full, 64, row, seg, qh, qb);
            }
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % S;
                if (j >= S) mbar_wait_sleep(&kv_empty[st], ((j / S) + 1) & 1);
                uint8_t* skv = smem + SM::kv_off + st * NB * kTileBytes;
                const int row = (kv_tile0 + j) * kBN;
                mbar_arrive_expect_tx(&kv_full[st], NB * kTileBytes);
                tma_load_5d(skv, &a.tmK, &kv_full[st], 0, row, seg, kh, kb);
                tma_load_5d(skv + kPanel, &a.tmK, &kv_full[st], 64, row, seg, kh, kb);
                if (NB == 2) {
                    tma_load_5d(skv + kTileBytes, &a.tmV, &kv_full[st], 0, row, seg, kh, kb);
                    tma_load_5d(skv + kTileBytes + kPanel, &a.tmV, &kv_full[st], 64, row, seg, kh, kb);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idS = idesc_bf16(128, kBN, 0, 0);   // S = Q K^T, both K-major
        constexpr uint32_t idPV = idesc_bf16(128, 128, 0, 1);  // O += P V, V MN-major
        const uint32_t q_addr = smem_u32(smem + SM::q_off);
        const uint32_t kv_addr = smem_u32(smem + SM::kv_off);
        if (elect_one()) {
            auto issue_s = [&](int t, int j) {
                const uint32_t kaddr = kv_addr + (j % S) * NB * kTileBytes;
                const uint32_t qa = q_addr + t * kTileBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
                    umma_ss(tmem + t * 256, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(kaddr + off, 16, 1024), idS,
                            kk > 0);
                }
                umma_commit(&s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {
                const uint32_t vaddr = kv_addr + (j % S) * NB * kTileBytes + (NB == 2 ? kTileBytes : 0);
#pragma unroll
                for (int kk = 0; kk < kBN / 16; ++kk)
                    umma_ts(tmem + t * 256 + 128, tmem + t * 256 + kk * 8, sdesc_sw128(vaddr + kk * 2048, kPanel, 1024),
                            idPV, (j > 0 || kk > 0) ? 1u : 0u);
            };
            mbar_wait_sleep(q_full, 0);
            mbar_wait_sleep(&kv_full[0], 0);
            tc_fence_after();
            issue_s(0, 0);
            issue_s(1, 0);
            for (int j = 0; j < n_kv; ++j) {
                const bool more = j + 1 < n_kv;
                // tile A
                mbar_wait_sleep(&p_full[0], j & 1);
                tc_fence_after();
                issue_pv(0, j);
                if (more) {
                    mbar_wait_sleep(&kv_full[(j + 1) % S], ((j + 1) / S) & 1);
                    tc_fence_after();
                    issue_s(0, j + 1);
                }
                // tile B
                mbar_wait_sleep(&p_full[1], j & 1);
                tc_fence_after();
                issue_pv(1, j);
                umma_commit(&kv_empty[j % S]);
                if (more) issue_s(1, j + 1);
            }
            umma_commit(o_full);
        }
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int t = (warp - 2) >> 2;                // query tile of this warpgroup
        const int row = (warp & 3) * 32 + lane_id();  // TMEM lane == query row in tile
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + t * 256 + lane_base, tO = tS + 128;
        const int grow = (2 * pair + t) * kQTile + row;  // row within the segment
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
        const uint8_t* qtile_smem = smem + SM::q_off + t * kTileBytes;

        if (a.check_finite) {
            mbar_wait_sleep(q_full, 0);
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
        float a_run = 0.f;  // ENT: sum_l 2^(x'_l - m_run) x'_l
        const uint64_t scale2x2 = pk2(scale2, scale2);
        for (int j = 0; j < n_kv; ++j) {
            mbar_wait_sleep(&s_full[t], j & 1);
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
                    if (ENT) a_run *= alpha;
                    m_run = m_new;
                    rescale = true;
                }
            }
            // x' - m on the packed FMA pipe, 2^(x' - m) on MUFU (one pair in VMB_EMU_PERIOD on the
            // FMA-pipe polynomial; off by default); row sum in packed adds; P -> TMEM as bf16
            const uint64_t negm2 = pk2(-m_run, -m_run);
            const uint64_t* s2 = reinterpret_cast<const uint64_t*>(sr);
            uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, acce = 0;
#pragma unroll
            for (int cc = 0; cc < kBN / 32; ++cc) {
                uint32_t pk[16];
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                    const uint64_t t2 = ffma2(s2[cc * 16 + x], scale2x2, negm2);
                    uint64_t pp;
                    if ((x % VMB_EMU_PERIOD) == VMB_EMU_PERIOD - 1) pp = ex2_emu2(t2);
                    else pp = pk2(ex2(lo2(t2)), ex2(hi2(t2)));
                    if (ENT) acce = ffma2(pp, t2, acce);  // sum p (x' - m)
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
            const float tile_l = lo2(acc) + hi2(acc);
            l_run += tile_l;
            if (ENT) a_run += (lo2(acce) + hi2(acce)) + m_run * tile_l;  // sum p x' = sum p (x' - m) + m sum p
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
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[t]);
        }

        // ------------------------------------------------------------ epilogue
        mbar_wait_sleep(o_full, 0);
        tc_fence_after();
        const float inv_l = 1.f / l_run;
        const float lse2 = m_run + log2f(l_run);  // base-2 log-sum-exp of x' = s * scale2
        const float ent = ENT ? kLn2 * (lse2 - a_run * inv_l) : 0.f;
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
            if (ENT && valid) a.part_ent[((int64_t)useg * a.nsplit + split) * a.q_len + grow] = ent;
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
                if (ENT) a.ent_out[((int64_t)u * a.nseg + seg) * a.q_len + grow] = ent;
            }
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
void launch(const Params& p, int64_t n_useg, int nsplit, cudaStream_t s) {
    using SM = Smem<NB>;
    auto kern = (NB == 2 && p.a.ent_out) ? fa3_kernel<NB, NB == 2> : fa3_kernel<NB, false>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    dim3 grid((unsigned)(p.q_pairs * nsplit), (unsigned)n_useg);
    ProfScope ps(NB == 1 ? kKRstep : kKAttn, s);
    kern<<<grid, kThreads, SM::alloc, s>>>(p);
    count_launch();
    check_launch("fa3_tc");
}

}  // namespace

int tc3_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int max_split) {
    if (max_split <= 1 || q_len <= 0 || n_useg <= 0) return 1;
#ifdef VMB_FORCE_SPLITS  // experiment builds only (make EXTRA=-DVMB_FORCE_SPLITS=n)
    return std::min(VMB_FORCE_SPLITS, max_split);
#endif
    const int64_t total_tiles = (kv_len + kBN - 1) / kBN;
    // The split count depends on the per-unit shape only, never on the number of units in
    // the call: a unit's output is then bitwise the same whether it runs alone, in a batch or
    // on another GPU of a head-sharded job (test_video.cpp:197-216).  ~84 CTAs per unit
    // (C4: 6 tile pairs x 14 splits) keep 5-heads-per-GPU loads at 2.84 waves and cost ~1% at
    // 40 heads against the best per-U choice (profiles/r1_fa_variants.md).
    const int64_t pairs = (q_len + 2 * kQTile - 1) / (2 * kQTile);
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>({(int64_t)max_split, 14, total_tiles / 8}));
    int nsplit = (int)std::min<int64_t>(cap, (84 + pairs - 1) / pairs);
    while (nsplit > 1 && ((total_tiles + nsplit - 1) / nsplit) * (nsplit - 1) >= total_tiles) --nsplit;
    return nsplit;
}

Tc2Args tc3_fa_launch(Tc2Args a, int64_t U, cudaStream_t s, bool do_combine) {
    if (U == 0 || a.q_len == 0) return a;
    VMB_REQUIRE_DIM(a.kv_len >= 1, "attention over empty keys");
    VMB_REQUIRE_DIM(!a.cl_out || a.nv == 1, "entropy output needs the key tile as value operand");
    Params p;
    p.q_pairs = (a.q_len + 2 * kQTile - 1) / (2 * kQTile);
    const int total_tiles = (a.kv_len + kBN - 1) / kBN;
    const int64_t n_useg = U * a.nseg;
    const int nsplit = a.part_o ? tc3_plan_splits(a.q_len, a.kv_len, n_useg, a.max_split) : 1;
    p.n_kv_tiles = (total_tiles + nsplit - 1) / nsplit;
    p.total_tiles = total_tiles;
    a.nsplit = nsplit;
    a.n_useg = n_useg;
    a.out_align32 = rows_align32(a.out, a.oB, a.oH, a.oS, a.oR) ? 1 : 0;
    p.a = a;
    if (nsplit == 1) p.a.part_o = nullptr;
    if (a.nv == 1) launch<1>(p, n_useg, nsplit, s);
    else launch<2>(p, n_useg, nsplit, s);
    if (nsplit > 1 && do_combine) tc2_combine_launch(p.a, s);
    return p.a;
}

}  // namespace vmb
