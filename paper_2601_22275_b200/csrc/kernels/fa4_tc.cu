// fa4_tc.cu — persistent tcgen05 flash attention with fused online statistics (bf16, d = 128).
//
// One CTA per SM loops over work items (128-row query tile, unit*segment, kv-split); the
// key/value tiles of consecutive items form one continuous stream through the TMA ring, so
// an item's prologue (Q load, first S MMAs) and epilogue (O read-out, output stores)
// overlap its neighbours' main loops.  This is what the short rows of the R half-step need
// (12 key tiles per item at C4): a non-persistent CTA spends a third of its life in
// prologue/epilogue latency.
//
// Modes:
//   <NB=1, NO=1>  R half-step (monarch.hpp:53-103): value = key; outputs aL, cL
//   <NB=2, NO=2>  last R half-step with y = R V fused (monarch.hpp:182-185): O = P [K | V],
//                 one N = 256 MMA per k-step (the full-rate tcgen05 shape,
//                 profiles/r1_micro_tcgen05.md)
//   <NB=2, NO=1>  attention: first-frame recompute / dense baseline (flash_entropy.hpp:85-139)
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA
// issuer, warps 2-5 the softmax (a thread owns one whole query row (warp%4)*32 + lane: row
// max, exponentials and row sum stay in registers, no cross-thread exchange per key tile),
// warps 6-9 the epilogue: they read an item's O out of TMEM, normalise it with the row
// statistics handed over in shared memory and store it, while the softmax warpgroup already
// runs the next item (a non-persistent CTA spends ~5 of its ~18 us in prologue/epilogue with
// the tensor pipe idle, profiles/r1_fa_variants.md).  One softmax warp per SM sub-partition:
// the MUFU pipe of each SMSP serves 32 rows x 128 keys = 1024 cycles per tile, under the
// 1536 tensor cycles of S + P [K | V] (tcgen05: 64 cycles per 128x128x16, 128 per
// 128x256x16, profiles/r2_micro_tcgen05.md).
// TMEM (512 columns): S0 [0,128), S1 [128,256) double-buffered scores (P written back as
// bf16 over the first 64 columns); NO=1: O0 [256,384), O1 [384,512) double-buffered over
// items; NO=2: O [256,512) = [P K | P V].
// Shared memory: one Q tile (released by the MMA warp after the item's last S MMA, so the
// next item's Q load overlaps the last tile's softmax / PV) + a 6-stage K (or 3-stage K|V)
// ring.  The epilogue's entropy dot reads the q row from global memory (L2).
//
// Issue order (flattened tile index g over this CTA's items): S(g), PV(g-1), S(g+1), ...
// S(g) goes to buffer g&1 after PV(g-2) has been issued (in-order tcgen05 pipeline), and
// an item's first PV waits for the epilogue to have drained that O buffer (o_empty).
//
// Statistics: base 2, lazily rescaled reference max (threshold 8).  With value = key the
// entropy is  sum_l R ln R = ln2 * (scale2 * <q, O_K> / l - lse2)  (monarch.hpp:93-98): one
// dot product in the epilogue, with the q row prefetched from L2.
#include <cuda_bf16.h>

#include <algorithm>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 320;
constexpr int kTile = 128;                      // query rows per item, keys per KV tile
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
__device__ __forceinline__ uint64_t fmul2(uint64_t x, uint64_t y) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
    return d;
}
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
// 2^x for an element pair on the FMA/ALU pipes (degree-3 minimax on [-0.5,0.5], rel. err
// 1.1e-4; see fa3_tc.cu)
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
    Tc4Args a;
    int32_t q_tiles;      // query tiles per segment
    int32_t nsplit;       // key splits per segment
    int32_t n_kv_tiles;   // key tiles per split (the last split may own fewer)
    int32_t total_tiles;  // key tiles of the whole segment
    int64_t n_items;      // q_tiles * nsplit * U * nseg
};

struct Item {
    int qtile, split, useg, u, seg, kv_tile0, n_kv;
};
__device__ __forceinline__ Item decode(const Params& p, int64_t it64) {
    // 32-bit index arithmetic (n_items < 2^31, checked at launch): 64-bit divisions are
    // software routines and sat on the per-item critical path
    const uint32_t it = (uint32_t)it64;
    Item r;
    const uint32_t qt = (uint32_t)p.q_tiles, ns = (uint32_t)p.nsplit, sg = (uint32_t)p.a.nseg;
    r.qtile = (int)(it % qt);
    const uint32_t rest = it / qt;
    r.split = (int)(rest % ns);
    r.useg = (int)(rest / ns);
    r.u = (int)((uint32_t)r.useg / sg);
    r.seg = (int)((uint32_t)r.useg % sg);
    r.kv_tile0 = r.split * p.n_kv_tiles;
    r.n_kv = min(p.n_kv_tiles, p.total_tiles - r.kv_tile0);
    return r;
}

template <int NB, int NO>
struct Smem {
    static constexpr int NOB = NO == 1 ? 2 : 1;           // O buffers (TMEM) / stats buffers
    static constexpr int S = NB == 1 ? 5 : (NO == 2 ? 3 : 2);  // KV stages (32 KB K or 64 KB K|V)
    static constexpr uint32_t q_off = 0;                  // one Q buffer, released by the MMA warp
    static constexpr uint32_t kv_off = kTileBytes;        // after the item's last S
    static constexpr uint32_t bar_off = kv_off + S * NB * kTileBytes;
    // q_full, q_empty, kv_full[S], kv_empty[S], s_full[2], p_full[2], pv_done, o_full[2],
    // o_empty[2], stat_full[2], stat_empty[2]
    static constexpr uint32_t n_bars = 2 + 2 * S + 5 + 4 + 4;
    static constexpr uint32_t slot_off = bar_off + n_bars * 8;
    // float [O buffers][2][128 rows]: the row sum and the running max of an item, handed
    // from the softmax warpgroup to the epilogue warpgroup
    static constexpr uint32_t stat_off = slot_off + 16;
    static constexpr uint32_t bytes = stat_off + NOB * 2 * 128 * 4;
    static_assert(bytes <= 232448, "shared memory budget (227 KB per CTA)");
    // the dynamic smem window starts 1024-aligned (checked in the kernel): no slack needed
    static constexpr uint32_t alloc = bytes;
};

#ifndef VMB_TRACE
#define VMB_TRACE 0
#endif
// timing experiment only: the epilogue computes but does not store aL / y
#ifndef VMB_DEBUG_NO_STORE
#define VMB_DEBUG_NO_STORE 0
#endif
#if VMB_TRACE
// debug-only per-item timeline: [cta < 64][item < 16][event] globaltimer (ns)
__device__ unsigned long long g_trace4[64][16][8];
__device__ __forceinline__ void trace4(int n, int ev) {
    if (blockIdx.x < 64 && n < 16) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace4[blockIdx.x][n][ev] = t;
    }
}
#define TRACE4(n, ev) trace4(n, ev)
__device__ long long g_trace4t[16][2][12][6];
#define TRACE4T(n, j, ev) do { if (threadIdx.x == 64 && blockIdx.x < 16 && (n) >= 1 && (n) <= 2 && (j) < 12) \
    g_trace4t[blockIdx.x][(n) - 1][(j)][(ev)] = clock64(); } while (0)
#else
#define TRACE4(n, ev) do { } while (0)
#define TRACE4T(n, j, ev) do { } while (0)
#endif

template <int NB, int NO>
__global__ void __launch_bounds__(kThreads, 1) fa4_kernel(const __grid_constant__ Params p) {
    using SM = Smem<NB, NO>;
    constexpr int S = SM::S;
    constexpr int NOB = SM::NOB;  // O buffers
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 operand tiles need 1024-B alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bar_off);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* kv_full = bars + 2;         // [S]
    uint64_t* kv_empty = kv_full + S;     // [S]
    uint64_t* s_full = kv_empty + S;      // [2]
    uint64_t* p_full = s_full + 2;        // [2]
    uint64_t* pv_done = p_full + 2;
    uint64_t* o_full = pv_done + 1;       // [2]
    uint64_t* o_empty = o_full + 2;       // [2]
    uint64_t* stat_full = o_empty + 2;    // [2]
    uint64_t* stat_empty = stat_full + 2; // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::slot_off);

    const Tc4Args& a = p.a;
    const int warp = warp_id();

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        if (NB == 2) tma_prefetch_desc(&a.tmV);
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 128);
            mbar_init(&stat_full[i], 128);
            mbar_init(&stat_empty[i], 128);
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        mbar_init(pv_done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS0 = tmem, tO0 = tmem + 256;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            int64_t g = 0;
            int n = 0;
            for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++n) {
                const Item w = decode(p, it);
                // the Q buffer frees once the previous item's last S MMA has completed
                if (n >= 1) mbar_wait_sleep(q_empty, (n - 1) & 1);
                const int qb = w.u / a.qH, qh = w.u % a.qH;
                const int kb = w.u / a.kH, kh = w.u % a.kH;
                uint8_t* sq = smem + SM::q_off;
                mbar_arrive_expect_tx(q_full, kTileBytes);
                tma_load_5d(sq, &a.tmQ, q_full, 0, w.qtile * kTile, w.seg, qh, qb);
                tma_load_5d(sq + kPanel, &a.tmQ, q_full, 64, w.qtile * kTile, w.seg, qh, qb);
                for (int j = 0; j < w.n_kv; ++j, ++g) {
                    const int st = (int)(g % S);
                    if (g >= S) mbar_wait_sleep(&kv_empty[st], ((g / S) - 1) & 1);
                    uint8_t* skv = smem + SM::kv_off + st * NB * kTileBytes;
                    const int row = (w.kv_tile0 + j) * kTile;
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
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);            // S = Q K^T, both K-major
        constexpr uint32_t idPV = idesc_bf16(128, NO == 2 ? 256 : 128, 0, 1);  // O += P [K|]V, MN-major
        const uint32_t q_addr = smem_u32(smem + SM::q_off);
        const uint32_t kv_addr = smem_u32(smem + SM::kv_off);
        if (elect_one()) {
            // the PV of tile g-1 is issued after S(g): remember what it needs
            int64_t pg = -1;   // flattened index of the pending PV
            int pst = 0, pob = 0, pn = 0;
            bool pfirst = false, plast = false;
            auto issue_pv = [&]() {
                mbar_wait_sleep(&p_full[pg & 1], (pg >> 1) & 1);
                if (pfirst && pn >= NOB) mbar_wait_sleep(&o_empty[pob], ((pn / NOB) - 1) & 1);
                tc_fence_after();
                const uint32_t tP = tS0 + (uint32_t)(pg & 1) * 128;
                const uint32_t vaddr = kv_addr + pst * NB * kTileBytes + ((NB == 2 && NO == 1) ? kTileBytes : 0);
                const uint32_t tO = tO0 + (uint32_t)pob * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_ts(tO, tP + kk * 8, sdesc_sw128(vaddr + kk * 2048, kPanel, 1024), idPV,
                            (!pfirst || kk > 0) ? 1u : 0u);
                umma_commit(&kv_empty[pst]);
                umma_commit(pv_done);
                if (plast) umma_commit(&o_full[pob]);
            };
            int64_t g = 0;
            int n = 0;
            for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++n) {
                const Item w = decode(p, it);
                mbar_wait_sleep(q_full, n & 1);
                const uint32_t qa = q_addr;
                for (int j = 0; j < w.n_kv; ++j, ++g) {
                    const int st = (int)(g % S);
                    mbar_wait_sleep(&kv_full[st], (g / S) & 1);
                    tc_fence_after();
                    const uint32_t kaddr = kv_addr + st * NB * kTileBytes;
                    const uint32_t tS = tS0 + (uint32_t)(g & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
                        umma_ss(tS, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(kaddr + off, 16, 1024), idS, kk > 0);
                    }
                    umma_commit(&s_full[g & 1]);
                    if (j == w.n_kv - 1) umma_commit(q_empty);  // last read of this item's Q
                    if (pg >= 0) issue_pv();
                    pg = g;
                    pst = st;
                    pob = n % NOB;
                    pn = n;
                    pfirst = j == 0;
                    plast = j == w.n_kv - 1;
                }
            }
            if (pg >= 0) issue_pv();
        }
    } else if (warp >= 2 && warp < 6) {
        // ------------------------------------------------------------ softmax (one warpgroup)
        // thread = one whole query row: no cross-thread reduction anywhere in the softmax
        const int row = (warp & 3) * 32 + lane_id();  // TMEM lane == query row in tile
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        float* stats = reinterpret_cast<float*>(smem + SM::stat_off);  // [ob][2][row]
        int64_t g = 0;
        int n = 0;
        // per-row temperature source, loaded one item ahead (its latency hides under a whole item)
        auto load_c = [&](int64_t it2) -> float {
            if (!a.cR || it2 >= p.n_items) return 1.f;
            const Item w2 = decode(p, it2);
            const int gr = w2.qtile * kTile + row;
            return gr < a.q_len ? __ldg(a.cR + ((int64_t)w2.u * a.nseg + w2.seg) * a.q_len + gr) : 1.f;
        };
        float c_next = load_c(blockIdx.x);
        for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++n) {
            const Item w = decode(p, it);
            const int ob = n % NOB;
            const uint32_t tO = tO0 + (uint32_t)ob * 128 + lane_base;
            const uint8_t* qsm = smem + SM::q_off;
            const int grow = w.qtile * kTile + row;  // row within the segment
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
            const int kv_end = (w.kv_tile0 + w.n_kv) * kTile;
            const int last_valid = kTile - (kv_end > a.kv_len ? kv_end - a.kv_len : 0);

            if (a.check_finite) {
                mbar_wait_sleep(q_full, n & 1);
                bool bad = false;
#pragma unroll
                for (int pnl = 0; pnl < 2; ++pnl) {
                    const uint4* q4 = reinterpret_cast<const uint4*>(qsm + pnl * kPanel + row * 128);
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        const uint4 v = q4[x ^ (row & 7)];  // rotate chunks across lanes: no bank conflicts
                        const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            bad |= ((wd[e] & 0x7F80u) == 0x7F80u) || ((wd[e] & 0x7F800000u) == 0x7F800000u);
                    }
                }
                if (bad && valid) atomicExch(a.status, kStatusNonFiniteQ);
                if (a.qn_out) {
                    // max |Q row|^2 of the unit (bounds the L-step logits; nonnegative floats order as ints)
                    float ss = 0.f;
#pragma unroll
                    for (int pnl = 0; pnl < 2; ++pnl) {
                        const uint4* q4 = reinterpret_cast<const uint4*>(qsm + pnl * kPanel + row * 128);
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            const uint4 v = q4[x ^ (row & 7)];
                            const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float lo = __uint_as_float(wd[e] << 16), hi = __uint_as_float(wd[e] & 0xFFFF0000u);
                                ss = fmaf(lo, lo, fmaf(hi, hi, ss));
                            }
                        }
                    }
                    if (valid && !bad)
                        atomicMax(reinterpret_cast<unsigned*>(a.qn_out) + (int64_t)w.u * a.q_len + grow, __float_as_uint(ss));
                }
            }

            float m_run = -INFINITY, l_run = 0.f;
            const uint64_t scale2x2 = pk2(scale2, scale2);
            if (threadIdx.x == 64) TRACE4(n, 0);
            for (int j = 0; j < w.n_kv; ++j, ++g) {
                const uint32_t tS = tS0 + (uint32_t)(g & 1) * 128 + lane_base;
                TRACE4T(n, j, 0);
                mbar_wait_sleep(&s_full[g & 1], (g >> 1) & 1);
                TRACE4T(n, j, 1);
                if (threadIdx.x == 64 && j == 0) TRACE4(n, 1);
                tc_fence_after();
                uint32_t sr[kTile];
#pragma unroll
                for (int cc = 0; cc < kTile / 32; ++cc) VMB_TMEM_LD32(tS + cc * 32, (sr + cc * 32));
                tmem_ld_wait();
                TRACE4T(n, j, 2);
                float* s = reinterpret_cast<float*>(sr);
                if (j == w.n_kv - 1 && last_valid < kTile) {
                    asm volatile("");  // keep this a real (rarely taken) branch, not 128 selects
#pragma unroll
                    for (int x = 0; x < kTile; ++x)
                        if (x >= last_valid) s[x] = kMasked;
                }
                // row max: 4 independent FMNMX3 chains
                float a0 = s[0], a1 = s[1], a2 = s[2], a3 = s[3];
#pragma unroll
                for (int x = 4; x < kTile - 4; x += 8) {
                    a0 = fmax3(a0, s[x + 0], s[x + 1]);
                    a1 = fmax3(a1, s[x + 2], s[x + 3]);
                    a2 = fmax3(a2, s[x + 4], s[x + 5]);
                    a3 = fmax3(a3, s[x + 6], s[x + 7]);
                }
                a0 = fmax3(a0, s[kTile - 4], s[kTile - 3]);
                a1 = fmax3(a1, s[kTile - 2], s[kTile - 1]);
                TRACE4T(n, j, 3);
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
                const uint64_t negm2 = pk2(-m_run, -m_run);
                const uint64_t* s2 = reinterpret_cast<const uint64_t*>(sr);
                uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
                for (int cc = 0; cc < kTile / 32; ++cc) {
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
                    // O must hold every earlier P V product of this item before it is rescaled
                    mbar_wait_sleep(pv_done, (uint32_t)((g - 1) & 1));
                    tc_fence_after();
#pragma unroll
                    for (int cc = 0; cc < 4 * NO; ++cc) {
                        uint32_t orr[32];
                        const uint32_t ta = tO + cc * 32;
                        VMB_TMEM_LD32(ta, orr);
                        tmem_ld_wait();
#pragma unroll
                        for (int x = 0; x < 32; ++x) orr[x] = __float_as_uint(__uint_as_float(orr[x]) * alpha);
                        VMB_TMEM_ST32(ta, orr);
                    }
                }
                TRACE4T(n, j, 4);
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[g & 1]);
                TRACE4T(n, j, 5);
            }
            if (threadIdx.x == 64) TRACE4(n, 2);
            // hand the item's row statistics to the epilogue warpgroup and move on
            if (n >= NOB) mbar_wait_sleep(&stat_empty[ob], ((n / NOB) - 1) & 1);
            float* st = stats + ob * 256;
            st[row] = l_run;
            st[128 + row] = m_run;
            mbar_arrive(&stat_full[ob]);
        }
    } else if (warp >= 6) {
        // ------------------------------------------------------------ epilogue warpgroup
        // drains O of item n while the softmax warpgroups already work on item n+1
        const int row = (warp & 3) * 32 + lane_id();
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const float* stats = reinterpret_cast<const float*>(smem + SM::stat_off);
        int n = 0;
        for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++n) {
            const Item w = decode(p, it);
            const int ob = n % NOB;
            const uint32_t tO = tO0 + (uint32_t)ob * 128 + lane_base;
            const int grow = w.qtile * kTile + row;
            const bool valid = grow < a.q_len;
            // the per-row temperature and the q row (entropy dot) are fetched before the item's
            // statistics arrive, so their latency hides under the item's last tiles
            float c = 1.f;
            if (a.cR && valid) c = __ldg(a.cR + ((int64_t)w.u * a.nseg + w.seg) * a.q_len + grow);
            uint4 qv[16];
            if (a.cl_out) {
                const uint4* qp = reinterpret_cast<const uint4*>(
                    static_cast<const __nv_bfloat16*>(a.q_rows) + (w.u / a.qrHn) * a.qrB + (w.u % a.qrHn) * a.qrH +
                    (int64_t)w.seg * a.qrS + (int64_t)grow * a.qrR);
#pragma unroll
                for (int x = 0; x < 16; ++x) qv[x] = valid ? __ldg(qp + x) : make_uint4(0, 0, 0, 0);
            }
            if (a.clamp_enabled) c = (c < a.clamp_min) ? a.clamp_min : c;
            else if (!(c > 0.f)) c = 1.f;
            const float scale2 = a.qscale * kLog2e / c;
            mbar_wait_sleep(&stat_full[ob], (n / NOB) & 1);
            const float* st = stats + ob * 256;
            const float l_tot = st[row];
            const float m_run = st[128 + row];
            mbar_arrive(&stat_empty[ob]);
            if (threadIdx.x == 192) TRACE4(n, 3);
            const float inv_l = 1.f / l_tot;
            const float lse2 = m_run + log2f(l_tot);  // base-2 log-sum-exp of x' = s * scale2
            mbar_wait_sleep(&o_full[ob], (n / NOB) & 1);
            if (threadIdx.x == 192) TRACE4(n, 4);
            tc_fence_after();
            if (a.part_o) {
                // split-KV partial: normalised fp32 O and natural-log lse of this split
                float* prow = a.part_o + (((int64_t)w.useg * a.nsplit + w.split) * a.q_len + grow) * 128;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t orr[32];
                    VMB_TMEM_LD32(tO + cc * 32, orr);
                    tmem_ld_wait();
                    if (valid) {
                        float4* dst = reinterpret_cast<float4*>(prow + cc * 32);
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            dst[x] = make_float4(__uint_as_float(orr[4 * x + 0]) * inv_l, __uint_as_float(orr[4 * x + 1]) * inv_l,
                                                 __uint_as_float(orr[4 * x + 2]) * inv_l, __uint_as_float(orr[4 * x + 3]) * inv_l);
                    }
                }
                tc_fence_before();
                mbar_arrive(&o_empty[ob]);
                if (valid) a.part_lse[((int64_t)w.useg * a.nsplit + w.split) * a.q_len + grow] = kLn2 * lse2;
            } else {
                // packed pairs throughout: the epilogue shares each SMSP's issue slots with the
                // next item's softmax warp, so its instruction count is the drain time
                uint64_t qo2 = 0;   // <q_row, (P K)_row> (R-step entropy), lane pairs
                uint64_t ss2 = 0;   // |(P K)_row|^2 before normalisation, lane pairs
                const uint64_t inv2 = pk2(inv_l, inv_l);
                float ssa = 0.f;    // |aL row|^2: decides its low half and feeds aln_out
                const int64_t obh = w.u / a.oHn, ohh = w.u % a.oHn;
#pragma unroll
                for (int t = 0; t < NO; ++t) {
                    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(t == 0 ? a.out0 : a.out1) + obh * a.oB[t] +
                                          ohh * a.oH[t] + (int64_t)w.seg * a.oS[t] + (int64_t)grow * a.oR[t];
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        uint32_t orr[32];
                        VMB_TMEM_LD32(tO + t * 128 + cc * 32, orr);
                        tmem_ld_wait();
                        if (t == NO - 1 && cc == 3 && !(NO == 1 && a.out0_lo)) {
                            // all of O is in registers or stored: the next item's PV may start
                            tc_fence_before();
                            mbar_arrive(&o_empty[ob]);
                            if (threadIdx.x == 192) TRACE4(n, 5);
                        }
                        const uint64_t* o2 = reinterpret_cast<const uint64_t*>(orr);
                        if (t == 0 && a.cl_out) {
#pragma unroll
                            for (int x = 0; x < 4; ++x) {
                                const uint4 q4 = qv[cc * 4 + x];
                                const uint32_t qw[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    qo2 = ffma2((uint64_t)(qw[e] << 16) | ((uint64_t)(qw[e] & 0xFFFF0000u) << 32), o2[4 * x + e], qo2);
                            }
                        }
                        if (valid) {
                            uint32_t w16[16];
#pragma unroll
                            for (int x = 0; x < 16; ++x) {
                                if (t == 0) ss2 = ffma2(o2[x], o2[x], ss2);
                                const uint64_t nrm = fmul2(o2[x], inv2);
                                w16[x] = pack_bf16(lo2(nrm), hi2(nrm));
                            }
                            uint4 v[4];
#pragma unroll
                            for (int x = 0; x < 4; ++x) v[x] = make_uint4(w16[4 * x], w16[4 * x + 1], w16[4 * x + 2], w16[4 * x + 3]);
                            if (VMB_DEBUG_NO_STORE) {
                                asm volatile("" ::"r"(v[0].x), "r"(v[1].y), "r"(v[2].z), "r"(v[3].w));
                            } else if (a.out_align32) {
                                st_global_256(orow + cc * 32, v[0], v[1]);
                                st_global_256(orow + cc * 32 + 16, v[2], v[3]);
                            } else {
                                uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
                                for (int x = 0; x < 4; ++x) dst[x] = v[x];
                            }
                        }
                    }
                    // low half of aL (same layout): bf16(x - bf16(x)), only for rows whose L-step
                    // logits could move by more than the bound (qn: Qmax^2 of the unit; nullptr:
                    // not known yet -> every row), a second TMEM pass so the entropy dot's
                    // prefetched q row is dead by then (register budget).  tcgen05.ld is
                    // warp-collective: a warp with any such row loads, only those rows store.
                    if (t == 0) ssa = (lo2(ss2) + hi2(ss2)) * (inv_l * inv_l);
                    const bool need_lo =
                        valid && (a.qn == nullptr || a.qn[(int64_t)w.u * a.q_len + grow] * ssa > a.lo_thresh2);
                    if (t == 0 && a.out0_lo && NO == 1 && !__any_sync(0xffffffffu, need_lo)) {
                        tc_fence_before();
                        mbar_arrive(&o_empty[ob]);
                    }
                    if (t == 0 && a.out0_lo && __any_sync(0xffffffffu, need_lo)) {
                        __nv_bfloat16* lrow = static_cast<__nv_bfloat16*>(a.out0_lo) + obh * a.oB[0] + ohh * a.oH[0] +
                                              (int64_t)w.seg * a.oS[0] + (int64_t)grow * a.oR[0];
#pragma unroll 1
                        for (int cc = 0; cc < 4; ++cc) {
                            uint32_t orr[32];
                            VMB_TMEM_LD32(tO + cc * 32, orr);
                            tmem_ld_wait();
                            if (NO == 1 && cc == 3) {
                                tc_fence_before();
                                mbar_arrive(&o_empty[ob]);
                            }
                            if (need_lo) {
                                uint4 v[4];
#pragma unroll
                                for (int x = 0; x < 4; ++x) {
                                    uint32_t h[4];
#pragma unroll
                                    for (int e = 0; e < 4; ++e) {
                                        const float f0 = __uint_as_float(orr[8 * x + 2 * e]) * inv_l;
                                        const float f1 = __uint_as_float(orr[8 * x + 2 * e + 1]) * inv_l;
                                        h[e] = pack_bf16_residual(f0, f1, pack_bf16(f0, f1));
                                    }
                                    v[x] = make_uint4(h[0], h[1], h[2], h[3]);
                                }
                                if (VMB_DEBUG_NO_STORE) {
                                    asm volatile("" ::"r"(v[0].x), "r"(v[1].y), "r"(v[2].z), "r"(v[3].w));
                                } else if (a.out_align32) {
                                    st_global_256(lrow + cc * 32, v[0], v[1]);
                                    st_global_256(lrow + cc * 32 + 16, v[2], v[3]);
                                } else {
                                    uint4* dst = reinterpret_cast<uint4*>(lrow + cc * 32);
#pragma unroll
                                    for (int x = 0; x < 4; ++x) dst[x] = v[x];
                                }
                            }
                            __syncwarp();
                        }
                    }
                }
                if (valid) {
                    if (a.cl_out)
                        a.cl_out[((int64_t)w.u * a.q_len + grow) * a.nseg + w.seg] = kLn2 * (scale2 * (lo2(qo2) + hi2(qo2)) * inv_l - lse2);
                    if (a.aln_out) a.aln_out[((int64_t)w.u * a.q_len + grow) * a.nseg + w.seg] = sqrtf(ssa);
                    if (a.lse_out) a.lse_out[((int64_t)w.u * a.nseg + w.seg) * a.q_len + grow] = kLn2 * lse2;
                }
                if (threadIdx.x == 192) TRACE4(n, 6);
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

template <int NB, int NO>
void launch(const Params& p, cudaStream_t s) {
    using SM = Smem<NB, NO>;
    auto kern = fa4_kernel<NB, NO>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::alloc));
    int dev = 0, sms = 148;
    VMB_CHECK_CUDA(cudaGetDevice(&dev));
    VMB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t grid = std::min<int64_t>(p.n_items, sms);
    ProfScope ps(NO == 2 ? kKRstepY : (NB == 1 ? kKRstep : kKAttn), s);
    kern<<<(unsigned)grid, kThreads, SM::alloc, s>>>(p);
    count_launch();
    check_launch("fa4_tc");
}

}  // namespace

int tc4_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int max_split) {
    if (max_split <= 1 || q_len <= 0 || n_useg <= 0) return 1;
    const int64_t total_tiles = (kv_len + kTile - 1) / kTile;
    // ~16 items per SM so the persistent CTAs balance, >= 8 key tiles per split
    const int64_t base = ((q_len + kTile - 1) / kTile) * n_useg;
    const int64_t want = (16 * 148 + base - 1) / base;
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)max_split, total_tiles / 8}));
    while (nsplit > 1 && ((total_tiles + nsplit - 1) / nsplit) * (nsplit - 1) >= total_tiles) --nsplit;
    return nsplit;
}

void tc4_fa_launch(Tc4Args a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.q_len == 0) return;
    VMB_REQUIRE_DIM(a.kv_len >= 1, "attention over empty keys");
    VMB_REQUIRE_DIM(a.nv == 1 || a.nv == 2, "value operand count");
    VMB_REQUIRE_DIM(!a.cl_out || a.v_is_k || a.nv == 2, "entropy output needs the key tile as first value operand");
    Params p;
    p.q_tiles = (a.q_len + kTile - 1) / kTile;
    p.total_tiles = (a.kv_len + kTile - 1) / kTile;
    const int64_t n_useg = U * a.nseg;
    p.nsplit = (a.part_o && a.nv == 1 && !a.v_is_k) ? tc4_plan_splits(a.q_len, a.kv_len, n_useg, a.max_split) : 1;
    p.n_kv_tiles = (p.total_tiles + p.nsplit - 1) / p.nsplit;
    p.n_items = (int64_t)p.q_tiles * p.nsplit * n_useg;
    {
        // 256-bit stores need every output row 32-byte aligned
        bool al = true;
        for (int t = 0; t < a.nv && t < 2; ++t) {
            void* base = t == 0 ? a.out0 : a.out1;
            al = al && (reinterpret_cast<uintptr_t>(base) % 32 == 0) && a.oB[t] % 16 == 0 && a.oH[t] % 16 == 0 &&
                 a.oS[t] % 16 == 0 && a.oR[t] % 16 == 0;
        }
        if (a.out0_lo) al = al && reinterpret_cast<uintptr_t>(a.out0_lo) % 32 == 0;
        a.out_align32 = al ? 1 : 0;
    }
    VMB_REQUIRE_DIM(p.n_items < ((int64_t)1 << 31), "too many work items for one launch");
    a.nsplit = p.nsplit;
    if (p.nsplit == 1) a.part_o = nullptr;
    p.a = a;
    if (a.nv == 2) launch<2, 2>(p, s);
    else if (a.v_is_k) launch<1, 1>(p, s);
    else launch<2, 1>(p, s);
    if (p.nsplit > 1) {
        Tc2Args c{};
        c.q_len = a.q_len;
        c.nseg = a.nseg;
        c.oHn = a.oHn;
        c.out = a.out0;
        c.oB = a.oB[0]; c.oH = a.oH[0]; c.oS = a.oS[0]; c.oR = a.oR[0];
        c.lse_out = a.lse_out;
        c.part_o = a.part_o;
        c.part_lse = a.part_lse;
        c.nsplit = p.nsplit;
        c.n_useg = n_useg;
        tc2_combine_launch(c, s);
    }
}

}  // namespace vmb

#if VMB_TRACE
extern "C" int vmb_debug_trace4t_read(long long* host) {
    return cudaMemcpyFromSymbol(host, vmb::g_trace4t, sizeof(long long) * 16 * 2 * 12 * 6) == cudaSuccess ? 0 : -1;
}
extern "C" int vmb_debug_trace4_read(unsigned long long* host) {
    return cudaMemcpyFromSymbol(host, vmb::g_trace4, sizeof(unsigned long long) * 64 * 16 * 8) == cudaSuccess ? 0 : -1;
}
#endif
