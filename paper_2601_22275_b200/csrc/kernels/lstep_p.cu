// lstep_p.cu — persistent, pipelined L half-step / permutation-folded apply (bf16, d = 128,
// m <= 128).  Same math as lstep_tc.cu (monarch.hpp:105-147, 187-190); different schedule.
//
// The L-step is HBM-bound: per position i it moves Qb[i], aL[i] (+ y[:, i]) in and
// aR[:, i] (or O rows j*b+i) out.  A one-position-per-CTA kernel has no loads in flight while
// it computes, so only about half of the smem it occupies carries traffic (measured 4.1 / 4.8
// TB/s, profiles/r1final_ncu_summary.md).  Here one CTA per SM walks the positions u*b + i:
//   warp 0      TMA producer: a ring of S stages [Qb | aL | (y)] kept full
//   warp 1      TMEM allocator + single-thread MMA issuer (GEMM 1 of item n+1 is issued before
//               waiting for L of item n, so the tensor pipe never blocks the ring)
//   warps 4-7,  two consumer warpgroups taking alternate items: softmax of S -> L (bf16, over
//   warps 8-11  the consumed aL tile), column sums cR (ITER), GEMM-2 read-out -> bf16 staging
//               over the consumed Qb tile -> TMA store, then the stage returns to the producer
// TMEM: 4 buffers of 128 columns (2 per warpgroup); S and the GEMM-2 accumulator share a buffer.
#include <cuda_bf16.h>

#include <algorithm>

#include "../internal.hpp"
#include "sm100_ptx.cuh"

namespace vmb {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr float kLog2e = 1.4426950408889634f;

struct Params {
    TcLstepArgs a;
    int32_t rows;     // R = m rounded up to 16
    int32_t n_items;  // U * b
};

template <bool FINAL>
struct Layout {
    int S;
    uint32_t panel, stage, qb, al, y, bars, slot, cl, bytes;
    __host__ __device__ Layout(int rows) {
        panel = (uint32_t)rows * 128u;
        stage = (FINAL ? 6u : 4u) * panel;
        // as many stages as fit next to the barriers (<= 6)
        const uint32_t budget = 232448u - 2048u;
        S = (int)(budget / stage);
        S = S > 6 ? 6 : S;
        qb = 0;
        al = 2 * panel;
        y = 4 * panel;
        bars = (uint32_t)S * stage;
        // full[S], empty[S], mma1[4], lrdy[4], mma2[4], bufempty[4]
        slot = bars + (uint32_t)(2 * S + 16) * 8;
        cl = slot + 16;               // float [2 warpgroups][128]: cL row of the current item
        bytes = cl + 2 * 128 * 4;
        // M = 128 MMAs read 128 rows of each K-major A panel (rows >= R are don't-care rows of
        // the accumulator): the last stage's reads must stay inside the allocation
        const uint32_t a_end = (uint32_t)(S - 1) * stage + (FINAL ? 3 * panel : panel) + 128u * 128u;
        bytes = bytes > a_end ? bytes : a_end;
    }
};

template <bool FINAL, int NCH>
__global__ void __launch_bounds__(kThreads, 1) lstep_p_kernel(const __grid_constant__ Params p) {
    const TcLstepArgs& a = p.a;
    const int R = p.rows;
    const Layout<FINAL> L(R);
    const int S = L.S;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 tiles need 1024-B alignment
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + S;
    uint64_t* mma1 = empty + S;      // [4]
    uint64_t* lrdy = mma1 + 4;       // [4]
    uint64_t* mma2 = lrdy + 4;       // [4]
    uint64_t* bufempty = mma2 + 4;   // [4]
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + L.slot);
    const int m = a.m;
    const int warp = warp_id();

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmAL);
        if (FINAL) tma_prefetch_desc(&a.tmY);
        tma_prefetch_desc(&a.tmOut);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(&mma1[b], 1);
            mbar_init(&lrdy[b], 128);
            mbar_init(&mma2[b], 1);
            mbar_init(&bufempty[b], 128);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            int n = 0;
            for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++n) {
                const int u = it / a.b, i = it % a.b;
                const int st = n % S;
                if (n >= S) mbar_wait(&empty[st], ((n / S) - 1) & 1);
                uint8_t* sb = smem + st * L.stage;
                const int qbb = u / a.H, qh = u % a.H;
                mbar_arrive_expect_tx(&full[st], (FINAL ? 6u : 4u) * L.panel);
                tma_load_5d(sb + L.qb, &a.tmQ, &full[st], 0, i, 0, qh, qbb);
                tma_load_5d(sb + L.qb + L.panel, &a.tmQ, &full[st], 64, i, 0, qh, qbb);
                tma_load_5d(sb + L.al, &a.tmAL, &full[st], 0, 0, i, 0, u);
                tma_load_5d(sb + L.al + L.panel, &a.tmAL, &full[st], 64, 0, i, 0, u);
                if (FINAL) {
                    tma_load_5d(sb + L.y, &a.tmY, &full[st], 0, i, 0, 0, u);
                    tma_load_5d(sb + L.y + L.panel, &a.tmY, &full[st], 64, i, 0, 0, u);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (elect_one()) {
            const uint32_t id1 = idesc_bf16(128, (uint32_t)R, 0, 0);
            const uint32_t id2 = FINAL ? idesc_bf16(128, 128, 0, 1) : idesc_bf16(128, 128, 1, 1);
            const uint32_t nk = (uint32_t)R / 16;
            auto gemm2 = [&](int n2) {
                const int st = n2 % S, buf = (n2 & 1) * 2 + ((n2 >> 1) & 1);
                const uint32_t sb = smem_u32(smem + st * L.stage);
                mbar_wait(&lrdy[buf], (n2 >> 2) & 1);
                tc_fence_after();
                const uint32_t d = tmem + buf * 128;
                if (!FINAL) {
                    // aR' = L^T [Qb]: A = L^T (M=k, K=j) MN-major, B = Qb (K=j, N=d) MN-major
                    for (uint32_t kk = 0; kk < nk; ++kk)
                        umma_ss(d, sdesc_sw128(sb + L.al + kk * 2048, L.panel, 1024),
                                sdesc_sw128(sb + L.qb + kk * 2048, L.panel, 1024), id2, kk > 0);
                } else {
                    // O_i = L Y: A = L (M=j, K=k) K-major, B = Y (K=k, N=d) MN-major
                    for (uint32_t kk = 0; kk < nk; ++kk) {
                        const uint32_t off = (kk >> 2) * L.panel + (kk & 3) * 32;
                        umma_ss(d, sdesc_sw128(sb + L.al + off, 16, 1024),
                                sdesc_sw128(sb + L.y + kk * 2048, L.panel, 1024), id2, kk > 0);
                    }
                }
                umma_commit(&mma2[buf]);
            };
            int n = 0;
            for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++n) {
                const int st = n % S, buf = (n & 1) * 2 + ((n >> 1) & 1);
                mbar_wait(&full[st], (n / S) & 1);
                // the TMEM buffer was last used by item n-4: its epilogue must have read it
                if (n >= 4) mbar_wait(&bufempty[buf], ((n >> 2) - 1) & 1);
                tc_fence_after();
                const uint32_t sb = smem_u32(smem + st * L.stage);
                const uint32_t d = tmem + buf * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * L.panel + (kk & 3) * 32;
                    umma_ss(d, sdesc_sw128(sb + L.qb + off, 16, 1024), sdesc_sw128(sb + L.al + off, 16, 1024), id1,
                            kk > 0);
                }
                umma_commit(&mma1[buf]);
                if (n >= 1) gemm2(n - 1);
            }
            if (n >= 1) gemm2(n - 1);
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ consumer warpgroups
        const int wg = (warp - 4) >> 2;
        const int t = (warp & 3) * 32 + lane_id();  // TMEM lane == row j (GEMM 1) / k or j (GEMM 2)
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const float sc2 = a.qscale * kLog2e;
        // cL of this warpgroup's next item, loaded one item ahead (row t holds cL[t])
        auto load_cl = [&](int it2) -> float {
            if (it2 >= p.n_items || t >= m) return 0.f;
            const int u2 = it2 / a.b, i2 = it2 % a.b;
            return __ldg(a.cL + ((int64_t)u2 * a.b + i2) * m + t);
        };
        int n = wg;
        int it = blockIdx.x + wg * gridDim.x;
        float cl_next = load_cl(it);
        for (; it < p.n_items; it += 2 * gridDim.x, n += 2) {
            const int u = it / a.b, i = it % a.b;
            const int st = n % S, buf = (n & 1) * 2 + ((n >> 1) & 1);
            uint8_t* sb = smem + st * L.stage;
            const uint32_t d = tmem + buf * 128 + lane_base;
            // this item's cL row -> the warpgroup's smem row (all rows j of the block share it)
            float* s_cl = reinterpret_cast<float*>(smem + L.cl) + wg * 128;
            s_cl[t] = cl_next;
            cl_next = load_cl(it + 2 * gridDim.x);
            named_bar_sync(1 + wg, 128);
            // ---- softmax of row j = t over k < m   (monarch.hpp:124-138)
            mbar_wait(&mma1[buf], (n >> 2) & 1);
            tc_fence_after();
            uint32_t sr[NCH * 32];
#pragma unroll
            for (int c = 0; c < NCH; ++c) VMB_TMEM_LD32(d + c * 32, (sr + c * 32));
            tmem_ld_wait();
            float* s = reinterpret_cast<float*>(sr);
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
            const float inv = (t < m) ? 1.f / sum : 0.f;  // rows j >= m are zeros (GEMM-2 K extent)
            if (t < R) {
                uint8_t* lt = sb + L.al;
#pragma unroll
                for (int c8 = 0; c8 < NCH * 4; ++c8) {
                    if (c8 * 8 < R) {
                        uint4 v;
                        v.x = pack_bf16(s[8 * c8 + 0] * inv, s[8 * c8 + 1] * inv);
                        v.y = pack_bf16(s[8 * c8 + 2] * inv, s[8 * c8 + 3] * inv);
                        v.z = pack_bf16(s[8 * c8 + 4] * inv, s[8 * c8 + 5] * inv);
                        v.w = pack_bf16(s[8 * c8 + 6] * inv, s[8 * c8 + 7] * inv);
                        *reinterpret_cast<uint4*>(lt + (c8 >> 3) * L.panel + sw128_offset(t, (c8 & 7) * 8)) = v;
                    }
                }
            }
            fence_proxy_async_smem();  // generic smem writes -> visible to the tensor core
            tc_fence_before();
            mbar_arrive(&lrdy[buf]);
            named_bar_sync(1 + wg, 128);  // the whole L tile is written
            if (!FINAL && t < m) {
                // cR[k,i] = sum_j L[j,k]  (monarch.hpp:139-143), k = t, from the bf16 copy of L:
                // 8 independent loads / accumulators per step (the loop is on the warpgroup's
                // critical path)
                const uint8_t* base = sb + L.al + (t >> 6) * L.panel + (t & 7) * 2;
                const uint32_t chunk = (uint32_t)((t & 63) >> 3);
                float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                int j = 0;
                for (; j + 8 <= m; j += 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int jj = j + q;  // row jj: chunk index XOR (jj & 7) == q ^ (j & 7) == q
                        acc[q] += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                            base + jj * 128 + ((chunk ^ (uint32_t)q) << 4)));
                    }
                }
                for (; j < m; ++j)
                    acc[0] += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                        base + j * 128 + ((chunk ^ (uint32_t)(j & 7)) << 4)));
                const float col0 = (acc[0] + acc[1]) + (acc[2] + acc[3]), col1 = (acc[4] + acc[5]) + (acc[6] + acc[7]);
                a.cR[((int64_t)u * m + t) * a.b + i] = col0 + col1;
            }
            // ---- epilogue: TMEM row t -> bf16 SW128 staging over the consumed Qb tile -> TMA store
            mbar_wait(&mma2[buf], (n >> 2) & 1);
            tc_fence_after();
            const float scale = a.out_scale;
            uint32_t packed[64];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t orr[32];
                VMB_TMEM_LD32(d + cc * 32, orr);
                tmem_ld_wait();
#pragma unroll
                for (int x = 0; x < 16; ++x)
                    packed[cc * 16 + x] = pack_bf16(__uint_as_float(orr[2 * x]) * scale, __uint_as_float(orr[2 * x + 1]) * scale);
            }
            tc_fence_before();
            mbar_arrive(&bufempty[buf]);  // TMEM buffer free for item n+4
            if (t < R) {
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint8_t* panel = sb + L.qb + (cc >> 1) * L.panel;
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const uint4 v = make_uint4(packed[cc * 16 + 4 * x], packed[cc * 16 + 4 * x + 1],
                                                   packed[cc * 16 + 4 * x + 2], packed[cc * 16 + 4 * x + 3]);
                        *reinterpret_cast<uint4*>(panel + sw128_offset(t, (cc & 1) * 32 + 8 * x)) = v;
                    }
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1 + wg, 128);
            if (t == 0) {
                if (!FINAL) {
                    tma_store_5d(&a.tmOut, sb + L.qb, 0, i, 0, 0, u);
                    tma_store_5d(&a.tmOut, sb + L.qb + L.panel, 64, i, 0, 0, u);
                } else {
                    const int ob = u / a.oHn, oh = u % a.oHn;
                    tma_store_5d(&a.tmOut, sb + L.qb, 0, i, 0, oh, ob);
                    tma_store_5d(&a.tmOut, sb + L.qb + L.panel, 64, i, 0, oh, ob);
                }
                tma_store_commit();
                tma_store_wait_read();  // the stage's smem is read: hand it back to the producer
                mbar_arrive(&empty[st]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) tma_store_wait_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <bool FINAL, int NCH>
void launch_nch(const Params& p, cudaStream_t s) {
    const Layout<FINAL> L(p.rows);
    VMB_REQUIRE_DIM(L.S >= 2, "L-step stage does not fit shared memory");
    auto kern = lstep_p_kernel<FINAL, NCH>;
    VMB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes));
    int dev = 0, sms = 148;
    VMB_CHECK_CUDA(cudaGetDevice(&dev));
    VMB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::min<int>(p.n_items, sms);
    ProfScope ps(FINAL ? kKLfinal : kKLstep, s);
    kern<<<(unsigned)grid, kThreads, L.bytes, s>>>(p);
    count_launch();
    check_launch("lstep_p");
}

template <bool FINAL>
void launch(const Params& p, cudaStream_t s) {
    switch ((p.rows + 31) / 32) {
        case 1: launch_nch<FINAL, 1>(p, s); break;
        case 2: launch_nch<FINAL, 2>(p, s); break;
        case 3: launch_nch<FINAL, 3>(p, s); break;
        default: launch_nch<FINAL, 4>(p, s); break;
    }
}

}  // namespace

void tc_lstep_p_launch(const TcLstepArgs& a, int64_t U, cudaStream_t s) {
    if (U == 0 || a.b == 0) return;
    VMB_REQUIRE_DIM(a.m >= 1 && a.m <= 128, "tcgen05 L-step requires m <= 128");
    VMB_REQUIRE_DIM(U * (int64_t)a.b < ((int64_t)1 << 31), "too many L-step items for one launch");
    Params p;
    p.a = a;
    p.rows = lstep_rows(a.m);
    p.n_items = (int32_t)(U * a.b);
    if (a.final_mode) launch<true>(p, s);
    else launch<false>(p, s);
}

}  // namespace vmb
