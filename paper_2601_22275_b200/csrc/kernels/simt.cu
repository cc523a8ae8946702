// simt.cu — general-shape CUDA-core kernels for the VMonarch forward.
//
// These serve (1) the fp32 parity mode (VMB_F32: fp32 storage, fp32 dot products,
// double row sums / entropy exactly where the reference uses double) and (2) any
// bf16 shape the tcgen05 kernels do not cover (d > 128).  They are
// GPU kernels, not a CPU fallback.
//
// Thread mapping: G threads cooperate on one row, each owning 32 consecutive
// head-dim elements (d <= 32*G); dot products are reduced with xor-shuffles inside
// the G-lane group, so per-thread state is 32 floats regardless of d.
//
// Reference semantics followed:
//   simt_rstep_kernel  monarch.hpp:53-103  (logits, clamp, softmax, plogp -> cL, R*K)
//   simt_lstep_kernel  monarch.hpp:105-147 (logits - cL, softmax, col sums, L^T*Qb)
//                      + the assembly O[j*b+i] = sum_k L[i,j,k] y[k,i]  (monarch.hpp:187-190)
//   simt_flash_kernel  flash_entropy.hpp:85-139 (online max/sum/entropy, double stats)
#include <cuda_bf16.h>

#include <algorithm>

#include "../internal.hpp"

namespace vmb {
namespace {

constexpr int DPT = 32;          // head-dim elements per thread
constexpr int BLOCK = 128;       // threads per block
constexpr int KTILE = 32;        // key rows staged per smem tile

template <typename T>
__device__ __forceinline__ float ld1(const T* p);
template <>
__device__ __forceinline__ float ld1<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st1(T* p, float v);
template <>
__device__ __forceinline__ void st1<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st1<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}

__device__ __forceinline__ int64_t row_off(const View& v, int64_t u, int64_t a, int64_t c) {
    return (u / v.H) * v.sB + (u % v.H) * v.sH + a * v.sa + c * v.sc;
}

template <int G>
__device__ __forceinline__ float group_sum(float x) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Load this thread's 32-element slice of row `p` (scaled) into regs.
template <typename T>
__device__ __forceinline__ void load_slice(const T* p, int d0, int d, float scale, float* r) {
#pragma unroll
    for (int x = 0; x < DPT; ++x) r[x] = (d0 + x < d) ? ld1(p + d0 + x) * scale : 0.f;
}

// Stage KTILE rows (u, a, l0..l0+KTILE) of view `v` into smem as float [KTILE][d].
template <typename T>
__device__ __forceinline__ void stage_rows(float* sm, const View& v, int64_t u, int64_t a,
                                           int64_t l0, int64_t nrows, int d) {
    const T* base = static_cast<const T*>(v.base);
    for (int e = threadIdx.x; e < KTILE * d; e += blockDim.x) {
        const int r = e / d, x = e % d;
        const int64_t l = l0 + r;
        sm[r * d + x] = (l < nrows) ? ld1(base + row_off(v, u, a, l) + x) : 0.f;
    }
}

template <int G>
__device__ __forceinline__ float dot_smem(const float* q, const float* krow, int d0, int d) {
    float acc = 0.f;
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) acc = fmaf(q[x], krow[d0 + x], acc);
    return group_sum<G>(acc);
}

// ------------------------------------------------------------------ R half-step
// grid: (ceil(b / rows_per_block), m, U); one query row (u, k, i) per G-lane group.
template <typename T, int G>
__global__ void __launch_bounds__(BLOCK) simt_rstep_kernel(SimtRstepArgs a) {
    extern __shared__ float sm[];
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t k = blockIdx.y, u = blockIdx.z;
    const int64_t i = (int64_t)blockIdx.x * RPB + rloc;
    const bool valid = i < a.b;
    const int d = (int)a.d, d0 = g * DPT;

    float q[DPT];
    float inv_c = 1.f;
    if (valid) {
        load_slice(static_cast<const T*>(a.A.base) + row_off(a.A, u, k, i), d0, d, 1.f, q);
        float c = a.cR ? a.cR[(u * a.m + k) * a.b + i] : 1.f;
        if (a.clamp_enabled) {
            c = (c < a.clamp_min) ? a.clamp_min : c;
        } else if (!(c > 0.f)) {
            if (g == 0) atomicExch(a.status, kStatusClampDomain);
            c = 1.f;
        }
        inv_c = 1.f / c;
    } else {
#pragma unroll
        for (int x = 0; x < DPT; ++x) q[x] = 0.f;
    }
    const float qs = a.qscale;

    if (!a.R) {
        // One pass with running statistics (no R export requested): max m, sum l and
        // A = sum e s in double (monarch.hpp:87-98 accumulate in double), acc = sum e V in fp32,
        // rescaled whenever the row max grows.  Then aL = acc / l and
        // cL = sum p ln p = A / l - m - ln l.  Same quantities as the three passes below, a
        // third of the dot products.
        float m_run = -INFINITY;
        double l_run = 0.0, a_run = 0.0;
        float acc[DPT];
#pragma unroll
        for (int x = 0; x < DPT; ++x) acc[x] = 0.f;
        float* smv = sm + KTILE * d;
        for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
            __syncthreads();
            stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
            stage_rows<T>(smv, a.V, u, k, l0, a.b, d);
            __syncthreads();
            const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
            for (int r = 0; r < nl; ++r) {
                const float sv = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
                if (sv > m_run) {
                    const float sc = expf(m_run - sv);  // 0 on the first key
                    l_run *= sc;
                    a_run *= sc;
#pragma unroll
                    for (int x = 0; x < DPT; ++x) acc[x] *= sc;
                    m_run = sv;
                }
                const float e = expf(sv - m_run);
                l_run += (double)e;
                a_run += (double)e * (double)sv;
                const float* vr = smv + r * d;
#pragma unroll
                for (int x = 0; x < DPT; ++x)
                    if (d0 + x < d) acc[x] = fmaf(e, vr[d0 + x], acc[x]);
            }
        }
        if (!valid) return;
        const float inv_l = (float)(1.0 / l_run);
        T* out = static_cast<T*>(const_cast<void*>(a.Out.base)) + row_off(a.Out, u, k, i);
#pragma unroll
        for (int x = 0; x < DPT; ++x)
            if (d0 + x < d) st1(out + d0 + x, acc[x] * inv_l);
        if (a.cL && g == 0) a.cL[(u * a.b + i) * a.m + k] = (float)(a_run / l_run - (double)m_run - log(l_run));
        return;
    }

    // R export: the reference's three passes (the exported R rows need the final max and sum)
    // pass 1: row max of logits * inv_c   (monarch.hpp:81-86)
    float mx = -INFINITY;
    for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
        __syncthreads();
        const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
        for (int r = 0; r < nl; ++r) {
            const float s = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
            mx = fmaxf(mx, s);
        }
    }
    // pass 2: sum of exp in double   (monarch.hpp:87-91)
    double sum = 0.0;
    for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
        __syncthreads();
        const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
        for (int r = 0; r < nl; ++r) {
            const float s = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
            sum += (double)expf(s - mx);
        }
    }
    const float inv_sum = (float)(1.0 / sum);
    // pass 3: p, entropy (double), P * V   (monarch.hpp:92-101)
    double ent = 0.0;
    float acc[DPT];
#pragma unroll
    for (int x = 0; x < DPT; ++x) acc[x] = 0.f;
    float* smv = sm + KTILE * d;
    for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
        stage_rows<T>(smv, a.V, u, k, l0, a.b, d);
        __syncthreads();
        const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
        for (int r = 0; r < nl; ++r) {
            const float s = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
            const float p = expf(s - mx) * inv_sum;
            ent += (p > 0.f) ? (double)(p * logf(p)) : 0.0;
            if (a.R && valid && g == 0) a.R[((u * a.m + k) * a.b + i) * a.b + l0 + r] = p;
            const float* vr = smv + r * d;
#pragma unroll
            for (int x = 0; x < DPT; ++x)
                if (d0 + x < d) acc[x] = fmaf(p, vr[d0 + x], acc[x]);
        }
    }
    if (!valid) return;
    T* out = static_cast<T*>(const_cast<void*>(a.Out.base)) + row_off(a.Out, u, k, i);
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) st1(out + d0 + x, acc[x]);
    if (a.cL && g == 0) a.cL[(u * a.b + i) * a.m + k] = (float)ent;
}

// ------------------------------------------------------------------ L half-step
// grid: (b, U); block handles spatial position i.  Phase 1: row stats per j.
// Phase 2 (ITER): per column k -> cR[k,i], aR[k,i].  Phase 2 (FINAL): per row j -> O.
template <typename T, int G>
__global__ void __launch_bounds__(BLOCK) simt_lstep_kernel(SimtLstepArgs a) {
    extern __shared__ float sm[];
    float* s_mx = sm;              // [m]
    float* s_isum = sm + a.m;      // [m]
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t i = blockIdx.x, u = blockIdx.y;
    const int d = (int)a.d, d0 = g * DPT;
    const T* Qbase = static_cast<const T*>(a.Q.base);
    const T* Lbase = static_cast<const T*>(a.aL.base);
    const float* cl = a.cL + (u * a.b + i) * a.m;

    // phase 1  (monarch.hpp:121-138).  Loops are warp-uniform (shuffles need all lanes).
    for (int64_t j0 = 0; j0 < a.m; j0 += RPB) {
        const int64_t j = j0 + rloc;
        const bool valid = j < a.m;
        float q[DPT];
        if (valid) load_slice(Qbase + row_off(a.Q, u, i, j), d0, d, 1.f, q);
        else
#pragma unroll
            for (int x = 0; x < DPT; ++x) q[x] = 0.f;
        float mx = -INFINITY;
        for (int64_t k = 0; k < a.m; ++k) {
            float kr[DPT];
            load_slice(Lbase + row_off(a.aL, u, i, k), d0, d, 1.f, kr);
            float acc = 0.f;
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc = fmaf(q[x], kr[x], acc);
            const float s = group_sum<G>(acc) * a.qscale - cl[k];
            mx = fmaxf(mx, s);
        }
        double sum = 0.0;
        for (int64_t k = 0; k < a.m; ++k) {
            float kr[DPT];
            load_slice(Lbase + row_off(a.aL, u, i, k), d0, d, 1.f, kr);
            float acc = 0.f;
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc = fmaf(q[x], kr[x], acc);
            const float s = group_sum<G>(acc) * a.qscale - cl[k];
            sum += (double)expf(s - mx);
        }
        if (valid && g == 0) {
            s_mx[j] = mx;
            s_isum[j] = (float)(1.0 / sum);
        }
    }
    __syncthreads();

    if (!a.final_mode) {
        // phase 2 (ITER): column k  (monarch.hpp:139-145)
        for (int64_t k0 = 0; k0 < a.m; k0 += RPB) {
            const int64_t k = k0 + rloc;
            const bool valid = k < a.m;
            const int64_t kk = valid ? k : 0;
            float kr[DPT], acc[DPT];
            load_slice(Lbase + row_off(a.aL, u, i, kk), d0, d, 1.f, kr);
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc[x] = 0.f;
            double col = 0.0;
            for (int64_t j = 0; j < a.m; ++j) {
                float q[DPT];
                load_slice(Qbase + row_off(a.Q, u, i, j), d0, d, 1.f, q);
                float dd = 0.f;
#pragma unroll
                for (int x = 0; x < DPT; ++x) dd = fmaf(q[x], kr[x], dd);
                const float s = group_sum<G>(dd) * a.qscale - cl[kk];
                const float l = expf(s - s_mx[j]) * s_isum[j];
                col += (double)l;
                if (valid && a.L && g == 0) a.L[((u * a.b + i) * a.m + j) * a.m + k] = l;
#pragma unroll
                for (int x = 0; x < DPT; ++x) acc[x] = fmaf(l, q[x], acc[x]);
            }
            if (!valid) continue;
            T* out = static_cast<T*>(const_cast<void*>(a.aR.base)) + row_off(a.aR, u, k, i);
#pragma unroll
            for (int x = 0; x < DPT; ++x)
                if (d0 + x < d) st1(out + d0 + x, acc[x] * a.qscale);
            if (g == 0) a.cR[(u * a.m + k) * a.b + i] = (float)col;
        }
    } else {
        // phase 2 (FINAL): row j of O  (monarch.hpp:187-190)
        const T* Ybase = static_cast<const T*>(a.Y.base);
        for (int64_t j0 = 0; j0 < a.m; j0 += RPB) {
            const int64_t j = j0 + rloc;
            const bool valid = j < a.m;
            const int64_t jj = valid ? j : 0;
            float q[DPT], acc[DPT];
            load_slice(Qbase + row_off(a.Q, u, i, jj), d0, d, 1.f, q);
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc[x] = 0.f;
            for (int64_t k = 0; k < a.m; ++k) {
                float kr[DPT];
                load_slice(Lbase + row_off(a.aL, u, i, k), d0, d, 1.f, kr);
                float dd = 0.f;
#pragma unroll
                for (int x = 0; x < DPT; ++x) dd = fmaf(q[x], kr[x], dd);
                const float s = group_sum<G>(dd) * a.qscale - cl[k];
                const float l = expf(s - s_mx[jj]) * s_isum[jj];
                if (valid && a.L && g == 0) a.L[((u * a.b + i) * a.m + j) * a.m + k] = l;
                float yr[DPT];
                load_slice(Ybase + row_off(a.Y, u, k, i), d0, d, 1.f, yr);
#pragma unroll
                for (int x = 0; x < DPT; ++x) acc[x] = fmaf(l, yr[x], acc[x]);
            }
            if (!valid || (a.skip_j0 && j == 0)) continue;
            T* out = static_cast<T*>(const_cast<void*>(a.O.base)) + row_off(a.O, u, j, i);
#pragma unroll
            for (int x = 0; x < DPT; ++x)
                if (d0 + x < d) st1(out + d0 + x, acc[x]);
        }
    }
}

// ------------------------------------------------------------------ online-entropy attention
// grid: (ceil(nq / rows_per_block), U).  flash_entropy.hpp:107-137 / absorb_stats 20-51.
template <typename T, int G>
__global__ void __launch_bounds__(BLOCK) simt_flash_kernel(SimtFlashArgs a) {
    extern __shared__ float sm[];
    float* smk = sm;
    float* smv = sm + KTILE * a.d;
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t u = blockIdx.y;
    const int64_t r = (int64_t)blockIdx.x * RPB + rloc;
    const bool valid = r < a.nq;
    const int d = (int)a.d, d0 = g * DPT;
    // key range of this split
    const int64_t chunk = (a.nk + a.nsplit - 1) / a.nsplit;
    const int64_t kb = (int64_t)blockIdx.z * chunk, ke = kb + chunk < a.nk ? kb + chunk : a.nk;
    float q[DPT], acc[DPT];
    if (valid) {
        load_slice(static_cast<const T*>(a.Q.base) + row_off(a.Q, u, 0, r), d0, d, a.qscale, q);
    } else {
#pragma unroll
        for (int x = 0; x < DPT; ++x) q[x] = 0.f;
    }
#pragma unroll
    for (int x = 0; x < DPT; ++x) acc[x] = 0.f;
    double run_max = -INFINITY, norm = 0.0, ent = 0.0;
    for (int64_t l0 = kb; l0 < ke; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(smk, a.K, u, 0, l0, ke, d);
        stage_rows<T>(smv, a.V, u, 0, l0, ke, d);
        __syncthreads();
        const int nl = (int)((ke - l0) < KTILE ? (ke - l0) : KTILE);
        float s[KTILE];
        double tmax = -INFINITY;
#pragma unroll
        for (int rr = 0; rr < KTILE; ++rr) {
            s[rr] = (rr < nl) ? dot_smem<G>(q, smk + rr * d, d0, d) : -INFINITY;
            tmax = fmax(tmax, (double)s[rr]);
        }
        const double m_new = fmax(run_max, tmax);
        if (!isinf(run_max)) {
            const double delta = run_max - m_new;
            const double alpha = exp(delta);
            ent = alpha * ent + alpha * delta * norm;
            norm *= alpha;
            if (alpha != 1.0) {
                const float af = (float)alpha;
#pragma unroll
                for (int x = 0; x < DPT; ++x) acc[x] *= af;
            }
        }
#pragma unroll
        for (int rr = 0; rr < KTILE; ++rr) {
            if (rr < nl) {
                const double x = (double)s[rr];
                const double p = exp(x - m_new);
                norm += p;
                ent += p * (x - m_new);
                const float pf = (float)p;
                const float* vr = smv + rr * d;
#pragma unroll
                for (int xx = 0; xx < DPT; ++xx)
                    if (d0 + xx < d) acc[xx] = fmaf(pf, vr[d0 + xx], acc[xx]);
            }
        }
        run_max = m_new;
    }
    if (!valid) return;
    if (a.nsplit > 1) {
        // split-KV partial: unnormalised acc and (max, sum, entropy accumulator)
        const int64_t pr = ((int64_t)blockIdx.z * a.U + u) * a.nq + r;
        float* pa = a.part_acc + pr * d;
#pragma unroll
        for (int x = 0; x < DPT; ++x)
            if (d0 + x < d) pa[d0 + x] = acc[x];
        if (g == 0) {
            a.part_stat[pr * 3 + 0] = run_max;
            a.part_stat[pr * 3 + 1] = norm;
            a.part_stat[pr * 3 + 2] = ent;
        }
        return;
    }
    const float inv = (float)(1.0 / norm);
    T* out = static_cast<T*>(const_cast<void*>(a.O.base)) + row_off(a.O, u, 0, r);
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) st1(out + d0 + x, acc[x] * inv);
    if (g == 0) {
        if (a.lse) a.lse[u * a.nq + r] = (float)(run_max + log(norm));
        if (a.ent) a.ent[u * a.nq + r] = (float)(log(norm) - ent / norm);
    }
}

// Merge of the split-KV partials (same statistics as the single pass, flash_entropy.hpp:30-45):
// m = max m_s, l = sum l_s e^(m_s - m), E = sum e^(m_s - m) (E_s + (m_s - m) l_s), O = acc / l.
template <typename T, int G>
__global__ void __launch_bounds__(BLOCK) simt_flash_combine_kernel(SimtFlashArgs a) {
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t u = blockIdx.y;
    const int64_t r = (int64_t)blockIdx.x * RPB + rloc;
    if (r >= a.nq) return;
    const int d = (int)a.d, d0 = g * DPT;
    double m = -INFINITY;
    for (int s = 0; s < a.nsplit; ++s) m = fmax(m, a.part_stat[(((int64_t)s * a.U + u) * a.nq + r) * 3]);
    double norm = 0.0, ent = 0.0;
    float acc[DPT];
#pragma unroll
    for (int x = 0; x < DPT; ++x) acc[x] = 0.f;
    for (int s = 0; s < a.nsplit; ++s) {
        const int64_t pr = ((int64_t)s * a.U + u) * a.nq + r;
        const double ms = a.part_stat[pr * 3 + 0], ls = a.part_stat[pr * 3 + 1], es = a.part_stat[pr * 3 + 2];
        if (isinf(ms)) continue;  // empty split
        const double w = exp(ms - m);
        norm += w * ls;
        ent += w * (es + (ms - m) * ls);
        const float wf = (float)w;
        const float* pa = a.part_acc + pr * d;
#pragma unroll
        for (int x = 0; x < DPT; ++x)
            if (d0 + x < d) acc[x] = fmaf(wf, pa[d0 + x], acc[x]);
    }
    const float inv = (float)(1.0 / norm);
    T* out = static_cast<T*>(const_cast<void*>(a.O.base)) + row_off(a.O, u, 0, r);
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) st1(out + d0 + x, acc[x] * inv);
    if (g == 0) {
        if (a.lse) a.lse[u * a.nq + r] = (float)(m + log(norm));
        if (a.ent) a.ent[u * a.nq + r] = (float)(log(norm) - ent / norm);
    }
}

template <typename T>
__global__ void finite_rows_kernel(View q, int64_t U, int64_t rows, int64_t d, int32_t* status) {
    const int64_t total = U * rows * d;
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = e % d, rr = (e / d) % rows, u = e / (d * rows);
        const float v = ld1(static_cast<const T*>(q.base) + row_off(q, u, 0, rr) + x);
        bad |= !isfinite(v);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicExch(status, kStatusNonFiniteQ);
}

__global__ void clamp_domain_kernel(const float* cR, int64_t n, int32_t* status) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= !(cR[e] > 0.f);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicExch(status, kStatusClampDomain);
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        VMB_CHECK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)bytes));
}

int pick_g(int64_t d) {
    VMB_REQUIRE_DIM(d >= 1 && d <= 8 * DPT, "head dim must be in [1, 256]");
    return d <= 32 ? 1 : d <= 64 ? 2 : d <= 128 ? 4 : 8;
}

template <typename T, int G>
void rstep_launch(const SimtRstepArgs& a, cudaStream_t s) {
    constexpr int RPB = BLOCK / G;
    dim3 grid((unsigned)((a.b + RPB - 1) / RPB), (unsigned)a.m, (unsigned)a.U);
    const size_t smem = 2 * KTILE * a.d * sizeof(float);
    set_smem(simt_rstep_kernel<T, G>, smem);
    ProfScope ps(kKSimt, s);
    simt_rstep_kernel<T, G><<<grid, BLOCK, smem, s>>>(a);
    count_launch();
    check_launch("simt_rstep");
}
template <typename T, int G>
void lstep_launch(const SimtLstepArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)a.b, (unsigned)a.U);
    const size_t smem = 2 * a.m * sizeof(float);
    set_smem(simt_lstep_kernel<T, G>, smem);
    ProfScope ps(kKSimt, s);
    simt_lstep_kernel<T, G><<<grid, BLOCK, smem, s>>>(a);
    count_launch();
    check_launch("simt_lstep");
}
template <typename T, int G>
void flash_launch(const SimtFlashArgs& a0, cudaStream_t s) {
    constexpr int RPB = BLOCK / G;
    SimtFlashArgs a = a0;
    const int64_t row_blocks = (a.nq + RPB - 1) / RPB;
    // split the keys when the row blocks of one unit fill less than two waves; the split count
    // depends on the per-unit shape only (bitwise-identical results for any unit count)
    a.nsplit = (int32_t)std::max<int64_t>(1, std::min<int64_t>({(2 * 148 + row_blocks - 1) / row_blocks, 32,
                                                                 a.nk / (8 * KTILE)}));
    if (a.nsplit > 1) {
        scratch_alloc(reinterpret_cast<void**>(&a.part_acc),
                                       sizeof(float) * a.nsplit * a.U * a.nq * a.d, s);
        scratch_alloc(reinterpret_cast<void**>(&a.part_stat),
                                       sizeof(double) * 3 * a.nsplit * a.U * a.nq, s);
    }
    const dim3 grid((unsigned)row_blocks, (unsigned)a.U, (unsigned)a.nsplit);
    const size_t smem = 2 * KTILE * a.d * sizeof(float);
    set_smem(simt_flash_kernel<T, G>, smem);
    ProfScope ps(kKSimt, s);
    simt_flash_kernel<T, G><<<grid, BLOCK, smem, s>>>(a);
    count_launch();
    check_launch("simt_flash");
    if (a.nsplit > 1) {
        simt_flash_combine_kernel<T, G><<<dim3((unsigned)row_blocks, (unsigned)a.U), BLOCK, 0, s>>>(a);
        count_launch();
        check_launch("simt_flash_combine");
        VMB_CHECK_CUDA(cudaFreeAsync(a.part_acc, s));
        VMB_CHECK_CUDA(cudaFreeAsync(a.part_stat, s));
    }
}

#define VMB_DISPATCH_G(G_, FN, T_, ...)                                  \
    switch (G_) {                                                        \
        case 1: FN<T_, 1>(__VA_ARGS__); break;                           \
        case 2: FN<T_, 2>(__VA_ARGS__); break;                           \
        case 4: FN<T_, 4>(__VA_ARGS__); break;                           \
        default: FN<T_, 8>(__VA_ARGS__); break;                          \
    }

}  // namespace

void simt_rstep(const SimtRstepArgs& a, bool bf16, cudaStream_t s) {
    const int G = pick_g(a.d);
    if (a.U == 0 || a.m == 0 || a.b == 0) return;
    if (bf16) { VMB_DISPATCH_G(G, rstep_launch, __nv_bfloat16, a, s); }
    else      { VMB_DISPATCH_G(G, rstep_launch, float, a, s); }
}
void simt_lstep(const SimtLstepArgs& a, bool bf16, cudaStream_t s) {
    const int G = pick_g(a.d);
    if (a.U == 0 || a.m == 0 || a.b == 0) return;
    if (bf16) { VMB_DISPATCH_G(G, lstep_launch, __nv_bfloat16, a, s); }
    else      { VMB_DISPATCH_G(G, lstep_launch, float, a, s); }
}
void simt_flash(const SimtFlashArgs& a, bool bf16, cudaStream_t s) {
    const int G = pick_g(a.d);
    if (a.U == 0 || a.nq == 0) return;
    if (bf16) { VMB_DISPATCH_G(G, flash_launch, __nv_bfloat16, a, s); }
    else      { VMB_DISPATCH_G(G, flash_launch, float, a, s); }
}
void check_finite_rows(View q, int64_t U, int64_t rows, int64_t d, bool bf16, int32_t* status,
                       cudaStream_t s) {
    const int64_t total = U * rows * d;
    if (total == 0) return;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (bf16) finite_rows_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(q, U, rows, d, status);
    else      finite_rows_kernel<float><<<blocks, 256, 0, s>>>(q, U, rows, d, status);
    count_launch();
    check_launch("check_finite");
}
void check_clamp_domain(const float* cR, int64_t n, int32_t* status, cudaStream_t s) {
    if (n == 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    clamp_domain_kernel<<<blocks, 256, 0, s>>>(cR, n, status);
    count_launch();
    check_launch("check_clamp_domain");
}

}  // namespace vmb
