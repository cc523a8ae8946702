// lstep_tc.cu — tcgen05 L half-step and the permutation-folded Monarch apply (bf16, d = 128,
// m <= 128).  HBM-bound stage.
//
// One CTA per (unit u, spatial position i); 128 threads; up to 4 CTAs per SM so that the
// TMA loads of some CTAs overlap the tensor-core / softmax work of the others.
// Reference semantics (monarch.hpp:105-147):
//   S[j,k]  = <Qb[i,j], aL[i,k]> * qscale - cL[i,k]        GEMM 1 (M=j, N=k, K=d)
//   L[j,:]  = softmax_k(S[j,:])                             thread j owns row j (TMEM lane j)
//   ITER : cR[k,i] = sum_j L[j,k]                           column sums of the smem copy of L
//          aR[k,i] = sum_j L[j,k] Qb[i,j]                   GEMM 2 (M=k, N=d, K=j): A = L^T
//                                                           read MN-major from the same tile
//   FINAL: O[j*b+i] = sum_k L[j,k] y[k,i]                   GEMM 2 (M=j, N=d, K=k), the
//          assembly of monarch.hpp:187-190 with the reshape-transpose permutation folded
//          into the TMA coordinates of Qb / y / O.
// Qb[i] rows are the tokens j*b+i of Q (stride b*d): a (d, i, j) box of a 5-D TMA map, so
// no permuted copy of Q ever exists (mat.hpp:99-113 / perm.hpp:19-50 are addressing only).
//
// Shared memory (R = m rounded up to 16 rows, P = R*128 bytes per 64-column panel):
//   [Qb: 2P][aL -> L: 2P][y: 2P (FINAL)][cL: R floats][barriers]
// L (bf16, SW128, K-major in k) overwrites aL once GEMM 1 has consumed it; the output tile
// (aR or O, bf16 SW128) is staged over Qb once GEMM 2 has consumed it and leaves through a
// TMA store.  TMEM: 128 columns; GEMM 2's accumulator reuses the S columns.
#include <cuda_bf16.h>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 128;
constexpr float kLog2e = 1.4426950408889634f;

// packed fp32 pairs (FFMA2 / FADD2 / FMUL2): half the issue slots of the scalar softmax
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
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
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

#ifndef VMB_TRACE
#define VMB_TRACE 0
#endif
#if VMB_TRACE
// debug-only per-CTA timeline of unit 0, positions < 1456: [final][pos][event] globaltimer (ns)
__device__ unsigned long long g_tracel[2][1456][8];
__device__ int g_tracel_lo[2][1456];
#define TRACEL(ev) do { if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 1456) { \
    unsigned long long tt_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt_)); \
    g_tracel[FINAL ? 1 : 0][blockIdx.x][ev] = tt_; } } while (0)
#else
#define TRACEL(ev) do { } while (0)
#endif

struct Params {
    TcLstepArgs a;
    int32_t rows;  // R
};

struct Layout {
    uint32_t panel, qb, al, y, cl, bars, slot, ones, bytes;
    __host__ __device__ Layout(int rows, bool final_mode) {
        panel = (uint32_t)rows * 128u;
        qb = 0;
        al = 2 * panel;
        // FINAL: y lands over Qb once GEMM 1 has consumed it (four CTAs per SM instead of three)
        y = 0;
        cl = 4 * panel;
        bars = cl + 512;
        slot = bars + 56;
        // ITER: 16 K-major rows of bf16 ones (the B operand of the column-sum MMA), 1024-aligned
        ones = (slot + 16 + 1023u) & ~1023u;
        bytes = final_mode ? slot + 16 : ones + 4096u;
        // M = 128 MMAs read 128 rows of every K-major A panel (rows >= R are don't-care
        // rows of the accumulator) -- keep those reads inside the allocation.
        const uint32_t a_end = (final_mode ? 3 * panel : panel) + 128u * 128u;
        bytes = bytes > a_end ? bytes : a_end;
    }
};

// P positions per CTA (m <= 32: 4, m <= 64: 2, else 1).  With P > 1 the positions' tiles are
// stacked in the 128 tile rows (position p in rows [p R, p R + R), R = 128 / P) and the
// products are block-diagonal: GEMM 1 computes every cross-position block as well (the
// softmax reads only its own), L is written with zeros outside its diagonal block, so GEMM 2
// and the column sums need no masking.  Small m then keeps the tensor tiles and the bytes in
// flight per CTA as large as at m = 128.
template <bool FINAL, int NCH, int P>
__global__ void __launch_bounds__(kThreads, NCH == 4 ? 2 : 4) lstep_tc_kernel(const __grid_constant__ Params p) {
    const TcLstepArgs& a = p.a;
    const int R = p.rows;                       // rows per position
    const int RT = P * R;                       // stacked rows (P > 1: 128)
    const Layout L(RT, FINAL);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bar_load = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* bar_mma1 = bar_load + 1;
    uint64_t* bar_mma2 = bar_load + 2;
    uint64_t* bar_lo = bar_load + 3;      // aL low half loaded
    uint64_t* bar_mma1b = bar_load + 4;   // S += Qb aL_lo^T done
    uint64_t* bar_cr = bar_load + 5;      // ITER: column sums L^T 1 done
    uint64_t* bar_y = bar_load + 6;       // FINAL: y loaded (over Qb, after GEMM 1)
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + L.slot);
    float* s_cl = reinterpret_cast<float*>(smem + L.cl);

    const int i = blockIdx.x * P, u = blockIdx.y;  // first position of this CTA
    const int m = a.m;
    const int warp = warp_id();
    const int t = threadIdx.x;
    // thread t = stacked row t: position pi (i + pi), row rr within it
    const int pi = P == 1 ? 0 : t / R;
    const int rr = P == 1 ? t : t % R;
    const bool pos_ok = i + pi < a.b;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t qb_addr = smem_u32(smem + L.qb);
    const uint32_t al_addr = smem_u32(smem + L.al);
    const uint32_t y_addr = smem_u32(smem + L.y);
    // the per-position scalars first: their global-load latency overlaps the barrier setup,
    // the TMA issue and the TMEM allocation below
    TRACEL(0);
    const int64_t pos = (int64_t)u * a.b + i + pi;
    const bool row_ok = rr < m && pos_ok;
    const float clv = row_ok ? __ldg(a.cL + pos * m + rr) : 0.f;
    float qnv = 0.f, alnv = 0.f;
    if (a.use_lo && row_ok) {
        qnv = __ldg(a.qn + pos);
        alnv = __ldg(a.aln + pos * m + rr);
    }

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch_desc(&a.tmQ);
            tma_prefetch_desc(&a.tmAL);
            if (FINAL) tma_prefetch_desc(&a.tmY);
            if (a.use_lo) tma_prefetch_desc(&a.tmALlo);
            tma_prefetch_desc(&a.tmOut);
            mbar_init(bar_load, 1);
            mbar_init(bar_mma1, 1);
            mbar_init(bar_mma2, 1);
            mbar_init(bar_lo, 1);
            mbar_init(bar_mma1b, 1);
            mbar_init(bar_cr, 1);
            mbar_init(bar_y, 1);
            fence_mbar_init();
            // loads first: their latency overlaps the TMEM allocation
            const int qbb = u / a.H, qh = u % a.H;
            mbar_arrive_expect_tx(bar_load, 4u * L.panel);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const uint32_t o = (uint32_t)(q * R) * 128u;
                tma_load_5d(smem + L.qb + o, &a.tmQ, bar_load, 0, i + q, 0, qh, qbb);
                tma_load_5d(smem + L.qb + L.panel + o, &a.tmQ, bar_load, 64, i + q, 0, qh, qbb);
                tma_load_5d(smem + L.al + o, &a.tmAL, bar_load, 0, 0, i + q, 0, u);
                tma_load_5d(smem + L.al + L.panel + o, &a.tmAL, bar_load, 64, 0, i + q, 0, u);
            }
        }
        __syncwarp();
        tmem_alloc<128>(slot);
    }
    // -cL[i, k] * log2(e) -> smem (all rows of this block share it); columns k >= m get -inf,
    // so their logits are -inf and their exponentials 0 with no per-element select
    s_cl[t] = row_ok ? -clv * kLog2e : -INFINITY;
    if (!FINAL) {
        // bf16 ones for the column-sum MMA (read by the tensor core after the L-tile fence)
        uint4* o4 = reinterpret_cast<uint4*>(smem + L.ones);
        o4[2 * t] = o4[2 * t + 1] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    }
    // row k = t of aL needs its low half iff the hi half alone could move an L-step logit by more
    // than kLoBound * 2^-9: qscale Qmax |aL_k| > kLoBound (Cauchy-Schwarz over the block's queries)
    const bool need_lo = a.use_lo && row_ok && qnv * (alnv * alnv) > a.lo_thresh2;
    tc_fence_before();
    const int any_lo = __syncthreads_or(need_lo);
    tc_fence_after();
    TRACEL(1);
#if VMB_TRACE
    if (t == 0 && u == 0 && i < 1456) g_tracel_lo[FINAL ? 1 : 0][i] = any_lo;
#endif
    const uint32_t tmem = *slot;
    const bool leader = (warp == 0) && elect_one();

    if (leader) {
        mbar_wait(bar_load, 0);
        tc_fence_after();
        const uint32_t id1 = idesc_bf16(128, (uint32_t)RT, 0, 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * L.panel + (kk & 3) * 32;
            umma_ss(tmem, sdesc_sw128(qb_addr + off, 16, 1024), sdesc_sw128(al_addr + off, 16, 1024), id1, kk > 0);
        }
        umma_commit(bar_mma1);
    }
    __syncwarp();

    // ---- softmax of row j = t over k < m   (monarch.hpp:124-138)
    mbar_wait(bar_mma1, 0);
    tc_fence_after();
    TRACEL(2);
    // FINAL: Qb is consumed (unless the low-half pass still reads it): y goes over it
    auto load_y = [&]() {
        if (FINAL && leader) {
            mbar_arrive_expect_tx(bar_y, 2u * L.panel);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const uint32_t o = (uint32_t)(q * R) * 128u;
                tma_load_5d(smem + L.y + o, &a.tmY, bar_y, 0, i + q, 0, 0, u);
                tma_load_5d(smem + L.y + L.panel + o, &a.tmY, bar_y, 64, i + q, 0, 0, u);
            }
        }
    };
    if (!any_lo) load_y();
    uint32_t sr[NCH * 32];
    if (any_lo) {
        // aL = hi + lo: S += Qb aL_lo^T for the rows that need it.  GEMM 1 has finished reading
        // aL hi (bar_mma1): the low half lands in its place; rows whose low half the R half-step
        // did not write (or does not matter) are zeroed before the MMA reads the tile.
        if (leader) {
            mbar_arrive_expect_tx(bar_lo, 2u * L.panel);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const uint32_t o = (uint32_t)(q * R) * 128u;
                tma_load_5d(smem + L.al + o, &a.tmALlo, bar_lo, 0, 0, i + q, 0, u);
                tma_load_5d(smem + L.al + L.panel + o, &a.tmALlo, bar_lo, 64, 0, i + q, 0, u);
            }
        }
        __syncwarp();
        mbar_wait(bar_lo, 0);
        if (t < RT && !need_lo) {
            uint4* r0 = reinterpret_cast<uint4*>(smem + L.al + t * 128);
            uint4* r1 = reinterpret_cast<uint4*>(smem + L.al + L.panel + t * 128);
#pragma unroll
            for (int x = 0; x < 8; ++x) r0[x] = r1[x] = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (leader) {
            const uint32_t id1 = idesc_bf16(128, (uint32_t)RT, 0, 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * L.panel + (kk & 3) * 32;
                umma_ss(tmem, sdesc_sw128(qb_addr + off, 16, 1024), sdesc_sw128(al_addr + off, 16, 1024), id1, 1u);
            }
            umma_commit(bar_mma1b);
        }
        __syncwarp();
        mbar_wait(bar_mma1b, 0);
        tc_fence_after();
        load_y();
    }
    float inv_row = 0.f;  // 1 / row sum of row j = t
    if (warp * 32 < RT) {  // (a warp past the R rows holds no row of L)
        // this row's own block of the score tile: columns [pi R, pi R + R)
        const uint32_t tcol = tmem + lane_base + (uint32_t)(pi * R);
#pragma unroll
        for (int c = 0; c < NCH; ++c) VMB_TMEM_LD32(tcol + c * 32, (sr + c * 32));
        tmem_ld_wait();
        float* s = reinterpret_cast<float*>(sr);
        // R = NCH*32 - 16: TMEM columns [R, NCH*32) are not written by GEMM 1 (don't-care data)
        if (R < NCH * 32) {
#pragma unroll
            for (int k = NCH * 32 - 16; k < NCH * 32; ++k) s[k] = 0.f;
        }
        // base-2 logits x' = S * qscale * log2e - cL * log2e (k >= m: -inf), in packed pairs;
        // four independent max / sum chains
        const uint64_t sc2x2 = pk2(a.qscale * kLog2e, a.qscale * kLog2e);
        uint64_t* s2 = reinterpret_cast<uint64_t*>(sr);
        const ulonglong2* ncl = reinterpret_cast<const ulonglong2*>(s_cl + pi * R);
#pragma unroll
        for (int k4 = 0; k4 < NCH * 8; ++k4) {
            const ulonglong2 c = ncl[k4];
            s2[2 * k4] = ffma2(s2[2 * k4], sc2x2, c.x);
            s2[2 * k4 + 1] = ffma2(s2[2 * k4 + 1], sc2x2, c.y);
        }
        float m4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
        for (int k = 4; k < NCH * 32; k += 8) {
            m4[0] = fmax3(m4[0], s[k + 0], s[k + 1]);
            m4[1] = fmax3(m4[1], s[k + 2], s[k + 3]);
            m4[2] = fmax3(m4[2], s[k + 4], s[k + 5]);
            m4[3] = fmax3(m4[3], s[k + 6], s[k + 7]);
        }
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        const uint64_t negm2 = pk2(-mx, -mx);
        uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int x = 0; x < NCH * 16; ++x) {
            const uint64_t t2 = fadd2(s2[x], negm2);
            s2[x] = pk2(ex2(lo2(t2)), ex2(hi2(t2)));
            acc[x & 3] = fadd2(acc[x & 3], s2[x]);
        }
        const uint64_t accs = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        // rows j >= m are zeros: they are part of GEMM 2's K extent (ITER).  FINAL leaves the
        // rows unnormalised (E = exp) and scales row j of O = E y by 1/sum in the epilogue.
        inv_row = row_ok ? 1.f / (lo2(accs) + hi2(accs)) : 0.f;
        const uint64_t inv2 = FINAL ? pk2(1.f, 1.f) : pk2(inv_row, inv_row);
        // L row j -> bf16, SW128, over the consumed aL tile
        if (P > 1) {
            // stacked: the own block at columns [pi R, pi R + R), zeros in the other blocks
            uint8_t* lt = smem + L.al;
#pragma unroll
            for (int c8 = 0; c8 < 16; ++c8) {
                const int col = c8 * 8;
                if (col < pi * R || col >= pi * R + R)
                    *reinterpret_cast<uint4*>(lt + (col >> 6) * L.panel + sw128_offset(t, col & 63)) =
                        make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int c8 = 0; c8 < NCH * 4; ++c8) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint64_t q2 = FINAL ? s2[4 * c8 + e] : fmul2(s2[4 * c8 + e], inv2);
                    w[e] = pack_bf16(lo2(q2), hi2(q2));
                }
                const int col = pi * R + c8 * 8;
                *reinterpret_cast<uint4*>(lt + (col >> 6) * L.panel + sw128_offset(t, col & 63)) =
                    make_uint4(w[0], w[1], w[2], w[3]);
            }
        } else if (t < R) {
            uint8_t* lt = smem + L.al;
#pragma unroll
            for (int c8 = 0; c8 < NCH * 4; ++c8) {
                if (c8 * 8 < R) {
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint64_t q2 = FINAL ? s2[4 * c8 + e] : fmul2(s2[4 * c8 + e], inv2);
                        w[e] = pack_bf16(lo2(q2), hi2(q2));
                    }
                    *reinterpret_cast<uint4*>(lt + (c8 >> 3) * L.panel + sw128_offset(t, (c8 & 7) * 8)) =
                        make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    TRACEL(3);

    const uint32_t nk = (uint32_t)RT / 16;
    if (!FINAL) {
        // cR[k,i] = sum_j L[j,k]  (monarch.hpp:139-143) on the tensor core: L^T 1 with
        // A = L^T (M=k, K=j) MN-major, B = 16 columns of ones, into TMEM columns [0, 16); read
        // (lane k = thread t) before GEMM 2 overwrites them
        if (leader) {
            const uint32_t ones_addr = smem_u32(smem + L.ones);
            const uint32_t idc = idesc_bf16(128, 16, 1, 0);
            for (uint32_t kk = 0; kk < nk; ++kk)
                umma_ss(tmem, sdesc_sw128(al_addr + kk * 2048, L.panel, 1024),
                        sdesc_sw128(ones_addr + (kk & 3) * 32, 16, 1024), idc, kk > 0);
            umma_commit(bar_cr);
        }
        __syncwarp();
        mbar_wait(bar_cr, 0);
        tc_fence_after();
        if (warp * 32 < (P == 1 ? m : RT)) {
            uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + lane_base));
            tmem_ld_wait();
            if (row_ok) a.cR[((int64_t)u * m + rr) * a.b + i + pi] = __uint_as_float(v);
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }

    if (leader) {
        if (!FINAL) {
            // aR' = L^T [Qb]: A = L^T (M=k, K=j) MN-major, B = Qb (K=j, N=d) MN-major
            const uint32_t id2 = idesc_bf16(128, 128, 1, 1);
            for (uint32_t kk = 0; kk < nk; ++kk)
                umma_ss(tmem, sdesc_sw128(al_addr + kk * 2048, L.panel, 1024),
                        sdesc_sw128(qb_addr + kk * 2048, L.panel, 1024), id2, kk > 0);
        } else {
            // O_i = E Y (E: unnormalised rows of L): A = E (M=j, K=k) K-major, B = Y (K=k, N=d)
            // MN-major
            mbar_wait(bar_y, 0);
            tc_fence_after();
            const uint32_t id2 = idesc_bf16(128, 128, 0, 1);
            for (uint32_t kk = 0; kk < nk; ++kk) {
                const uint32_t off = (kk >> 2) * L.panel + (kk & 3) * 32;
                umma_ss(tmem, sdesc_sw128(al_addr + off, 16, 1024), sdesc_sw128(y_addr + kk * 2048, L.panel, 1024),
                        id2, kk > 0);
            }
        }
        umma_commit(bar_mma2);
    }
    __syncwarp();

    // ---- epilogue: TMEM row t -> bf16 SW128 staging tile over Qb -> TMA store
    TRACEL(4);
    mbar_wait(bar_mma2, 0);
    tc_fence_after();
    TRACEL(5);
    const float scale = FINAL ? a.out_scale * inv_row : a.out_scale;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        if (warp * 32 >= RT) break;  // no output row in this warp
        uint32_t orr[32];
        VMB_TMEM_LD32(tmem + lane_base + cc * 32, orr);
        tmem_ld_wait();
        if (t < RT) {
            uint8_t* panel = smem + L.qb + (cc >> 1) * L.panel;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                uint4 v;
                v.x = pack_bf16(__uint_as_float(orr[8 * x + 0]) * scale, __uint_as_float(orr[8 * x + 1]) * scale);
                v.y = pack_bf16(__uint_as_float(orr[8 * x + 2]) * scale, __uint_as_float(orr[8 * x + 3]) * scale);
                v.z = pack_bf16(__uint_as_float(orr[8 * x + 4]) * scale, __uint_as_float(orr[8 * x + 5]) * scale);
                v.w = pack_bf16(__uint_as_float(orr[8 * x + 6]) * scale, __uint_as_float(orr[8 * x + 7]) * scale);
                *reinterpret_cast<uint4*>(panel + sw128_offset(t, (cc & 1) * 32 + 8 * x)) = v;
            }
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    TRACEL(6);
    if (t == 0) {
        // one store box per position (a position past b is clipped by the map)
        const int ob = FINAL ? u / a.oHn : u, oh = FINAL ? u % a.oHn : 0;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const uint32_t o = (uint32_t)(q * R) * 128u;
            tma_store_5d(&a.tmOut, smem + L.qb + o, 0, i + q, 0, oh, ob);
            tma_store_5d(&a.tmOut, smem + L.qb + L.panel + o, 64, i + q, 0, oh, ob);
        }
        tma_store_commit();
        tma_store_wait_read();
        TRACEL(7);
    }
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
    __syncthreads();
}

// ------------------------------------------------------------------ fp32 parity mode (hi/lo)
// The same half-step with every operand a bf16 hi/lo pair (x = hi + lo) and each product
// three MMA groups, A B ~ Ah Bh + Ah Bl + Al Bh, into the fp32 accumulator (the dropped Al Bl
// is 2^-16 relative).  Shared memory (P = R*128 bytes per 64-column panel):
//   [Qb hi: 2P][Qb lo: 2P][aL hi -> L hi: 2P][aL lo -> L lo: 2P][y hi: 2P][y lo: 2P (FINAL)][cL]
// Outputs leave from registers (thread = row): ITER aR*qscale as hi/lo bf16 rows and cR;
// FINAL O as fp32 rows.
struct HlLayout {
    uint32_t panel, cl, bars, slot, bytes;
    __host__ __device__ HlLayout(int rows, bool final_mode) {
        panel = (uint32_t)rows * 128u;
        cl = (final_mode ? 12 : 8) * panel;
        bars = cl + 512;
        slot = bars + 32;
        bytes = slot + 16;
        // M = 128 A reads from the last A panel (Qb lo panel 1, or L lo panel 1) stay inside
        const uint32_t a_end = 7 * panel + 128u * 128u;
        bytes = bytes > a_end ? bytes : a_end;
    }
};
struct HlParams {
    TcLstepHlArgs a;
    int32_t rows;
};

template <bool FINAL, int NCH>
__global__ void __launch_bounds__(kThreads, FINAL ? 1 : 2) lstep_hl_kernel(const __grid_constant__ HlParams p) {
    const TcLstepHlArgs& a = p.a;
    const int R = p.rows;
    const HlLayout L(R, FINAL);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar_load = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* bar_mma1 = bar_load + 1;
    uint64_t* bar_mma2 = bar_load + 2;
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + L.slot);
    float* s_cl = reinterpret_cast<float*>(smem + L.cl);
    const uint32_t P = L.panel;
    // operand tiles: q (hi, lo), l (aL -> L; hi, lo), y (hi, lo); each 2 panels
    const uint32_t base = smem_u32(smem);
    const uint32_t q_hi = base, q_lo = base + 2 * P, l_hi = base + 4 * P, l_lo = base + 6 * P;
    const uint32_t y_hi = base + 8 * P, y_lo = base + 10 * P;

    const int i = blockIdx.x, u = blockIdx.y;
    const int m = a.m;
    const int warp = warp_id();
    const int t = threadIdx.x;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;

    if (warp == 0) {
        if (elect_one()) {
            mbar_init(bar_load, 1);
            mbar_init(bar_mma1, 1);
            mbar_init(bar_mma2, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(bar_load, (FINAL ? 12u : 8u) * P);
            const CUtensorMap* qm[2] = {&a.tmQ, &a.tmQlo};
            const CUtensorMap* lm[2] = {&a.tmAL, &a.tmALlo};
            const CUtensorMap* ym[2] = {&a.tmY, &a.tmYlo};
            for (int h = 0; h < 2; ++h) {
                tma_load_5d(smem + 2 * h * P, qm[h], bar_load, 0, i, 0, 0, u);
                tma_load_5d(smem + (2 * h + 1) * P, qm[h], bar_load, 64, i, 0, 0, u);
                tma_load_5d(smem + (4 + 2 * h) * P, lm[h], bar_load, 0, 0, i, 0, u);
                tma_load_5d(smem + (5 + 2 * h) * P, lm[h], bar_load, 64, 0, i, 0, u);
                if (FINAL) {
                    tma_load_5d(smem + (8 + 2 * h) * P, ym[h], bar_load, 0, i, 0, 0, u);
                    tma_load_5d(smem + (9 + 2 * h) * P, ym[h], bar_load, 64, i, 0, 0, u);
                }
            }
        }
        __syncwarp();
        tmem_alloc<128>(slot);
    }
    const float* cl = a.cL + ((int64_t)u * a.b + i) * m;
    if (t < R) s_cl[t] = (t < m) ? cl[t] : 0.f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const bool leader = (warp == 0) && elect_one();

    if (leader) {
        // GEMM 1: S = Qb aL^T  (Qh aLh + Qh aLl + Ql aLh)
        mbar_wait(bar_load, 0);
        tc_fence_after();
        const uint32_t id1 = idesc_bf16(128, (uint32_t)R, 0, 0);
        const uint32_t qa[3] = {q_hi, q_hi, q_lo}, la[3] = {l_hi, l_lo, l_hi};
#pragma unroll
        for (int gr = 0; gr < 3; ++gr) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * P + (kk & 3) * 32;
                umma_ss(tmem, sdesc_sw128(qa[gr] + off, 16, 1024), sdesc_sw128(la[gr] + off, 16, 1024), id1,
                        (gr > 0 || kk > 0) ? 1u : 0u);
            }
        }
        umma_commit(bar_mma1);
    }
    __syncwarp();

    // ---- softmax of row j = t over k < m   (monarch.hpp:124-138)
    mbar_wait(bar_mma1, 0);
    tc_fence_after();
    uint32_t sr[NCH * 32];
#pragma unroll
    for (int c = 0; c < NCH; ++c) VMB_TMEM_LD32(tmem + lane_base + c * 32, (sr + c * 32));
    tmem_ld_wait();
    float* s = reinterpret_cast<float*>(sr);
    const float sc2 = a.qscale * kLog2e;
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < NCH * 32; ++k) {
        s[k] = (k < m) ? (s[k] * sc2 - s_cl[k] * kLog2e) : -INFINITY;
        mx = fmaxf(mx, s[k]);
    }
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < NCH * 32; ++k) {
        s[k] = (k < m) ? ex2(s[k] - mx) : 0.f;
        sum += s[k];
    }
    // rows j >= m are written as zeros: they are part of GEMM 2's K extent (ITER)
    const float inv = (t < m) ? 1.f / sum : 0.f;
    // L row j -> hi/lo bf16, SW128, over the consumed aL hi/lo tiles
    if (t < R) {
#pragma unroll
        for (int c8 = 0; c8 < NCH * 4; ++c8) {
            if (c8 * 8 < R) {
                uint4 h, l;
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = s[8 * c8 + e] * inv;
                h.x = pack_bf16(f[0], f[1]);
                h.y = pack_bf16(f[2], f[3]);
                h.z = pack_bf16(f[4], f[5]);
                h.w = pack_bf16(f[6], f[7]);
                l.x = pack_bf16_residual(f[0], f[1], h.x);
                l.y = pack_bf16_residual(f[2], f[3], h.y);
                l.z = pack_bf16_residual(f[4], f[5], h.z);
                l.w = pack_bf16_residual(f[6], f[7], h.w);
                const uint32_t off = (c8 >> 3) * P + sw128_offset(t, (c8 & 7) * 8);
                *reinterpret_cast<uint4*>(smem + 4 * P + off) = h;
                *reinterpret_cast<uint4*>(smem + 6 * P + off) = l;
            }
        }
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (leader) {
        const uint32_t nk = (uint32_t)R / 16;
        if (!FINAL) {
            // aR' = L^T Qb: A = L^T (M=k, K=j) MN-major, B = Qb (K=j, N=d) MN-major
            const uint32_t id2 = idesc_bf16(128, 128, 1, 1);
            const uint32_t aa[3] = {l_hi, l_hi, l_lo}, bb[3] = {q_hi, q_lo, q_hi};
#pragma unroll
            for (int gr = 0; gr < 3; ++gr)
                for (uint32_t kk = 0; kk < nk; ++kk)
                    umma_ss(tmem, sdesc_sw128(aa[gr] + kk * 2048, P, 1024), sdesc_sw128(bb[gr] + kk * 2048, P, 1024), id2,
                            (gr > 0 || kk > 0) ? 1u : 0u);
        } else {
            // O_i = L Y: A = L (M=j, K=k) K-major, B = Y (K=k, N=d) MN-major
            const uint32_t id2 = idesc_bf16(128, 128, 0, 1);
            const uint32_t aa[3] = {l_hi, l_hi, l_lo}, bb[3] = {y_hi, y_lo, y_hi};
#pragma unroll
            for (int gr = 0; gr < 3; ++gr)
                for (uint32_t kk = 0; kk < nk; ++kk) {
                    const uint32_t off = (kk >> 2) * P + (kk & 3) * 32;
                    umma_ss(tmem, sdesc_sw128(aa[gr] + off, 16, 1024), sdesc_sw128(bb[gr] + kk * 2048, P, 1024), id2,
                            (gr > 0 || kk > 0) ? 1u : 0u);
                }
        }
        umma_commit(bar_mma2);
    }
    __syncwarp();

    if (!FINAL && t < m) {
        // cR[k,i] = sum_j L[j,k]  (monarch.hpp:139-143), k = t, from L hi + lo
        float col[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const uint8_t* bh = smem + 4 * P + (t >> 6) * P;
        const uint8_t* bl = smem + 6 * P + (t >> 6) * P;
        auto lj = [&](int j) {
            const uint32_t off = sw128_offset(j, t & 63);
            return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(bh + off)) +
                   __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(bl + off));
        };
        int j = 0;
        for (; j + 8 <= m; j += 8) {
#pragma unroll
            for (int e = 0; e < 8; ++e) col[e] += lj(j + e);
        }
        for (; j < m; ++j) col[0] += lj(j);
        a.cR[((int64_t)u * m + t) * a.b + i] = ((col[0] + col[1]) + (col[2] + col[3])) + ((col[4] + col[5]) + (col[6] + col[7]));
    }

    // ---- epilogue: TMEM row t -> global (ITER: aR hi/lo bf16 rows (u, k=t, i); FINAL: O fp32
    // row (u, token t*b + i))
    mbar_wait(bar_mma2, 0);
    tc_fence_after();
    const bool store = t < m;
    __nv_bfloat16* rh = nullptr;
    __nv_bfloat16* rl = nullptr;
    float* orow = nullptr;
    if (!FINAL) {
        const int64_t r = ((int64_t)u * m + t) * a.b + i;
        rh = static_cast<__nv_bfloat16*>(a.ar_hi) + r * 128;
        rl = static_cast<__nv_bfloat16*>(a.ar_lo) + r * 128;
    } else {
        orow = a.out + (int64_t)(u / a.oHn) * a.oB + (int64_t)(u % a.oHn) * a.oH + ((int64_t)t * a.b + i) * a.oT;
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t orr[32];
        VMB_TMEM_LD32(tmem + lane_base + cc * 32, orr);
        tmem_ld_wait();
        if (!store) continue;
        if (!FINAL) {
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                uint4 h, l;
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(orr[8 * x + e]) * a.qscale;
                h.x = pack_bf16(f[0], f[1]);
                h.y = pack_bf16(f[2], f[3]);
                h.z = pack_bf16(f[4], f[5]);
                h.w = pack_bf16(f[6], f[7]);
                l.x = pack_bf16_residual(f[0], f[1], h.x);
                l.y = pack_bf16_residual(f[2], f[3], h.y);
                l.z = pack_bf16_residual(f[4], f[5], h.z);
                l.w = pack_bf16_residual(f[6], f[7], h.w);
                reinterpret_cast<uint4*>(rh + cc * 32)[x] = h;
                reinterpret_cast<uint4*>(rl + cc * 32)[x] = l;
            }
        } else {
#pragma unroll
            for (int x = 0; x < 8; ++x)
                reinterpret_cast<float4*>(orow + cc * 32)[x] =
                    make_float4(__uint_as_float(orr[4 * x + 0]), __uint_as_float(orr[4 * x + 1]),
                                __uint_as_float(orr[4 * x + 2]), __uint_as_float(orr[4 * x + 3]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

template <bool FINAL, int NCH>
void launch_hl_nch(const HlParams& p, int64_t U, cudaStream_t s) {
    const HlLayout L(p.rows, FINAL);
    const int smem = (int)L.bytes + 1024;
    auto kern = lstep_hl_kernel<FINAL, NCH>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid((unsigned)p.a.b, (unsigned)U);
    ProfScope ps(FINAL ? kKLfinal : kKLstep, s);
    kern<<<grid, kThreads, smem, s>>>(p);
    count_launch();
    check_launch("lstep_hl");
}

template <bool FINAL>
void launch_hl(const HlParams& p, int64_t U, cudaStream_t s) {
    switch ((p.rows + 31) / 32) {
        case 1: launch_hl_nch<FINAL, 1>(p, U, s); break;
        case 2: launch_hl_nch<FINAL, 2>(p, U, s); break;
        case 3: launch_hl_nch<FINAL, 3>(p, U, s); break;
        default: launch_hl_nch<FINAL, 4>(p, U, s); break;
    }
}

template <bool FINAL, int NCH, int P>
void launch_nch(const Params& p, int64_t U, cudaStream_t s) {
    const Layout L(P * p.rows, FINAL);
    const int smem = (int)L.bytes + 1024;
    auto kern = lstep_tc_kernel<FINAL, NCH, P>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid((unsigned)((p.a.b + P - 1) / P), (unsigned)U);
    ProfScope ps(FINAL ? kKLfinal : kKLstep, s);
    kern<<<grid, kThreads, smem, s>>>(p);
    count_launch();
    check_launch("lstep_tc");
}

template <bool FINAL>
void launch(const Params& p, int64_t U, cudaStream_t s) {
    switch (lstep_positions(p.a.m)) {
        case 4: launch_nch<FINAL, 1, 4>(p, U, s); return;  // rows per position 32
        case 2: launch_nch<FINAL, 2, 2>(p, U, s); return;  // 64
        default: break;
    }
    switch ((p.rows + 31) / 32) {
        case 1: launch_nch<FINAL, 1, 1>(p, U, s); break;
        case 2: launch_nch<FINAL, 2, 1>(p, U, s); break;
        case 3: launch_nch<FINAL, 3, 1>(p, U, s); break;
        default: launch_nch<FINAL, 4, 1>(p, U, s); break;
    }
}

}  // namespace

#if VMB_TRACE
extern "C" int vmb_debug_tracel_read(unsigned long long* host) {
    return cudaMemcpyFromSymbol(host, g_tracel, sizeof(unsigned long long) * 2 * 1456 * 8) == cudaSuccess ? 0 : -1;
}
extern "C" int vmb_debug_tracel_lo_read(int* host) {
    return cudaMemcpyFromSymbol(host, g_tracel_lo, sizeof(int) * 2 * 1456) == cudaSuccess ? 0 : -1;
}
#endif

void tc_lstep_hl_launch(const TcLstepHlArgs& a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.b == 0) return;
    VMB_REQUIRE_DIM(a.m >= 1 && a.m <= 128, "tcgen05 L-step requires m <= 128");
    VMB_REQUIRE_DIM(a.b <= 2147483647 && U <= 65535, "tcgen05 L-step grid limits");
    HlParams p;
    p.a = a;
    p.rows = lstep_rows(a.m);
    if (a.final_mode) launch_hl<true>(p, U, s);
    else launch_hl<false>(p, U, s);
}

void tc_lstep_launch(const TcLstepArgs& a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.b == 0) return;
    VMB_REQUIRE_DIM(a.m >= 1 && a.m <= 128, "tcgen05 L-step requires m <= 128");
    VMB_REQUIRE_DIM(a.b <= 2147483647 && U <= 65535, "tcgen05 L-step grid limits");
    Params p;
    p.a = a;
    p.rows = lstep_box_rows(a.m);
    if (a.final_mode) launch<true>(p, U, s);
    else launch<false>(p, U, s);
}

}  // namespace vmb
