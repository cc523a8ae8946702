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

// Storage type T (bf16, float, double) and compute type F (float; double for the f64 mode):
// loads widen T -> F, stores narrow F -> T.
template <typename F>
__device__ __forceinline__ F ld1(const float* p) { return (F)__ldg(p); }
template <typename F>
__device__ __forceinline__ F ld1(const double* p) { return (F)__ldg(p); }
template <typename F>
__device__ __forceinline__ F ld1(const __nv_bfloat16* p) { return (F)__bfloat162float(*p); }
__device__ __forceinline__ void st1(float* p, float v) { *p = v; }
__device__ __forceinline__ void st1(double* p, double v) { *p = v; }
__device__ __forceinline__ void st1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// F-precision math: the fp32 mode keeps expf / logf / fmaf (the reference's T = float calls),
// the f64 mode exp / log / fma (T = double)
__device__ __forceinline__ float vexp(float x) { return expf(x); }
__device__ __forceinline__ double vexp(double x) { return exp(x); }
__device__ __forceinline__ float vlog(float x) { return logf(x); }
__device__ __forceinline__ double vlog(double x) { return log(x); }
__device__ __forceinline__ float vfma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double vfma(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return fmax(a, b); }

__device__ __forceinline__ int64_t row_off(const View& v, int64_t u, int64_t a, int64_t c) {
    return (u / v.H) * v.sB + (u % v.H) * v.sH + a * v.sa + c * v.sc;
}

template <int G, typename F>
__device__ __forceinline__ F group_sum(F x) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Load this thread's 32-element slice of row `p` (scaled) into regs.
template <typename T, typename F>
__device__ __forceinline__ void load_slice(const T* p, int d0, int d, F scale, F* r) {
#pragma unroll
    for (int x = 0; x < DPT; ++x) r[x] = (d0 + x < d) ? ld1<F>(p + d0 + x) * scale : (F)0;
}

// Stage KTILE rows (u, a, l0..l0+KTILE) of view `v` into smem as F [KTILE][d].
template <typename T, typename F>
__device__ __forceinline__ void stage_rows(F* sm, const View& v, int64_t u, int64_t a,
                                           int64_t l0, int64_t nrows, int d) {
    const T* base = static_cast<const T*>(v.base);
    for (int e = threadIdx.x; e < KTILE * d; e += blockDim.x) {
        const int r = e / d, x = e % d;
        const int64_t l = l0 + r;
        sm[r * d + x] = (l < nrows) ? ld1<F>(base + row_off(v, u, a, l) + x) : (F)0;
    }
}

template <int G, typename F>
__device__ __forceinline__ F dot_smem(const F* q, const F* krow, int d0, int d) {
    F acc = 0;
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) acc = vfma(q[x], krow[d0 + x], acc);
    return group_sum<G>(acc);
}
template <typename F>
__device__ __forceinline__ F* smem_as() {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    return reinterpret_cast<F*>(smem_raw);
}

// ------------------------------------------------------------------ R half-step
// grid: (ceil(b / rows_per_block), m, U); one query row (u, k, i) per G-lane group.
template <typename T, typename F, int G>
__global__ void __launch_bounds__(BLOCK) simt_rstep_kernel(SimtRstepArgs a) {
    F* sm = smem_as<F>();
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t k = blockIdx.y, u = blockIdx.z;
    const int64_t i = (int64_t)blockIdx.x * RPB + rloc;
    const bool valid = i < a.b;
    const int d = (int)a.d, d0 = g * DPT;
    const F* cR = static_cast<const F*>(a.cR);
    F* cL = static_cast<F*>(a.cL);
    F* Rout = static_cast<F*>(a.R);

    F q[DPT];
    F inv_c = 1;
    if (valid) {
        load_slice(static_cast<const T*>(a.A.base) + row_off(a.A, u, k, i), d0, d, (F)1, q);
        F c = cR ? cR[(u * a.m + k) * a.b + i] : (F)1;
        const F cmin = (F)a.clamp_min;
        if (a.clamp_enabled) {
            c = (c < cmin) ? cmin : c;
        } else if (!(c > (F)0)) {
            if (g == 0) atomicExch(a.status, kStatusClampDomain);
            c = 1;
        }
        inv_c = (F)1 / c;
    } else {
#pragma unroll
        for (int x = 0; x < DPT; ++x) q[x] = 0;
    }
    const F qs = (F)a.qscale;

    if (!Rout) {
        // One pass with running statistics (no R export requested): max m, sum l and
        // A = sum e s in double (monarch.hpp:87-98 accumulate in double), acc = sum e V in F,
        // rescaled whenever the row max grows.  Then aL = acc / l and
        // cL = sum p ln p = A / l - m - ln l.  Same quantities as the three passes below, a
        // third of the dot products.
        F m_run = -INFINITY;
        double l_run = 0.0, a_run = 0.0;
        F acc[DPT];
#pragma unroll
        for (int x = 0; x < DPT; ++x) acc[x] = 0;
        F* smv = sm + KTILE * d;
        for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
            __syncthreads();
            stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
            stage_rows<T>(smv, a.V, u, k, l0, a.b, d);
            __syncthreads();
            const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
            for (int r = 0; r < nl; ++r) {
                const F sv = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
                if (sv > m_run) {
                    const F sc = vexp(m_run - sv);  // 0 on the first key
                    l_run *= sc;
                    a_run *= sc;
#pragma unroll
                    for (int x = 0; x < DPT; ++x) acc[x] *= sc;
                    m_run = sv;
                }
                const F e = vexp(sv - m_run);
                l_run += (double)e;
                a_run += (double)e * (double)sv;
                const F* vr = smv + r * d;
#pragma unroll
                for (int x = 0; x < DPT; ++x)
                    if (d0 + x < d) acc[x] = vfma(e, vr[d0 + x], acc[x]);
            }
        }
        if (!valid) return;
        const F inv_l = (F)(1.0 / l_run);
        T* out = static_cast<T*>(const_cast<void*>(a.Out.base)) + row_off(a.Out, u, k, i);
#pragma unroll
        for (int x = 0; x < DPT; ++x)
            if (d0 + x < d) st1(out + d0 + x, acc[x] * inv_l);
        if (cL && g == 0) cL[(u * a.b + i) * a.m + k] = (F)(a_run / l_run - (double)m_run - log(l_run));
        return;
    }

    // R export: the reference's three passes (the exported R rows need the final max and sum)
    // pass 1: row max of logits * inv_c   (monarch.hpp:81-86)
    F mx = -INFINITY;
    for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
        __syncthreads();
        const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
        for (int r = 0; r < nl; ++r) {
            const F sv = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
            mx = vmax(mx, sv);
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
            const F sv = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
            sum += (double)vexp(sv - mx);
        }
    }
    const F inv_sum = (F)(1.0 / sum);
    // pass 3: p, entropy (double), P * V   (monarch.hpp:92-101)
    double ent = 0.0;
    F acc[DPT];
#pragma unroll
    for (int x = 0; x < DPT; ++x) acc[x] = 0;
    F* smv = sm + KTILE * d;
    for (int64_t l0 = 0; l0 < a.b; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(sm, a.K, u, k, l0, a.b, d);
        stage_rows<T>(smv, a.V, u, k, l0, a.b, d);
        __syncthreads();
        const int nl = (int)((a.b - l0) < KTILE ? (a.b - l0) : KTILE);
        for (int r = 0; r < nl; ++r) {
            const F sv = (dot_smem<G>(q, sm + r * d, d0, d) * qs) * inv_c;
            const F p = vexp(sv - mx) * inv_sum;
            ent += (p > (F)0) ? (double)(p * vlog(p)) : 0.0;
            if (valid && g == 0) Rout[((u * a.m + k) * a.b + i) * a.b + l0 + r] = p;
            const F* vr = smv + r * d;
#pragma unroll
            for (int x = 0; x < DPT; ++x)
                if (d0 + x < d) acc[x] = vfma(p, vr[d0 + x], acc[x]);
        }
    }
    if (!valid) return;
    T* out = static_cast<T*>(const_cast<void*>(a.Out.base)) + row_off(a.Out, u, k, i);
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) st1(out + d0 + x, acc[x]);
    if (cL && g == 0) cL[(u * a.b + i) * a.m + k] = (F)ent;
}

// ------------------------------------------------------------------ L half-step
// grid: (b, U); block handles spatial position i.  Phase 1: row stats per j.
// Phase 2 (ITER): per column k -> cR[k,i], aR[k,i].  Phase 2 (FINAL): per row j -> O.
template <typename T, typename F, int G>
__global__ void __launch_bounds__(BLOCK) simt_lstep_kernel(SimtLstepArgs a) {
    F* sm = smem_as<F>();
    F* s_mx = sm;              // [m]
    F* s_isum = sm + a.m;      // [m]
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t i = blockIdx.x, u = blockIdx.y;
    const int d = (int)a.d, d0 = g * DPT;
    const T* Qbase = static_cast<const T*>(a.Q.base);
    const T* Lbase = static_cast<const T*>(a.aL.base);
    const F* cl = static_cast<const F*>(a.cL) + (u * a.b + i) * a.m;
    F* Lout = static_cast<F*>(a.L);
    const F qs = (F)a.qscale;

    // phase 1  (monarch.hpp:121-138).  Loops are warp-uniform (shuffles need all lanes).
    for (int64_t j0 = 0; j0 < a.m; j0 += RPB) {
        const int64_t j = j0 + rloc;
        const bool valid = j < a.m;
        F q[DPT];
        if (valid) load_slice(Qbase + row_off(a.Q, u, i, j), d0, d, (F)1, q);
        else
#pragma unroll
            for (int x = 0; x < DPT; ++x) q[x] = 0;
        F mx = -INFINITY;
        for (int64_t k = 0; k < a.m; ++k) {
            F kr[DPT];
            load_slice(Lbase + row_off(a.aL, u, i, k), d0, d, (F)1, kr);
            F acc = 0;
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc = vfma(q[x], kr[x], acc);
            const F sv = group_sum<G>(acc) * qs - cl[k];
            mx = vmax(mx, sv);
        }
        double sum = 0.0;
        for (int64_t k = 0; k < a.m; ++k) {
            F kr[DPT];
            load_slice(Lbase + row_off(a.aL, u, i, k), d0, d, (F)1, kr);
            F acc = 0;
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc = vfma(q[x], kr[x], acc);
            const F sv = group_sum<G>(acc) * qs - cl[k];
            sum += (double)vexp(sv - mx);
        }
        if (valid && g == 0) {
            s_mx[j] = mx;
            s_isum[j] = (F)(1.0 / sum);
        }
    }
    __syncthreads();

    if (!a.final_mode) {
        // phase 2 (ITER): column k  (monarch.hpp:139-145)
        F* cRout = static_cast<F*>(a.cR);
        for (int64_t k0 = 0; k0 < a.m; k0 += RPB) {
            const int64_t k = k0 + rloc;
            const bool valid = k < a.m;
            const int64_t kk = valid ? k : 0;
            F kr[DPT], acc[DPT];
            load_slice(Lbase + row_off(a.aL, u, i, kk), d0, d, (F)1, kr);
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc[x] = 0;
            double col = 0.0;
            for (int64_t j = 0; j < a.m; ++j) {
                F q[DPT];
                load_slice(Qbase + row_off(a.Q, u, i, j), d0, d, (F)1, q);
                F dd = 0;
#pragma unroll
                for (int x = 0; x < DPT; ++x) dd = vfma(q[x], kr[x], dd);
                const F sv = group_sum<G>(dd) * qs - cl[kk];
                const F l = vexp(sv - s_mx[j]) * s_isum[j];
                col += (double)l;
                if (valid && Lout && g == 0) Lout[((u * a.b + i) * a.m + j) * a.m + k] = l;
#pragma unroll
                for (int x = 0; x < DPT; ++x) acc[x] = vfma(l, q[x], acc[x]);
            }
            if (!valid) continue;
            T* out = static_cast<T*>(const_cast<void*>(a.aR.base)) + row_off(a.aR, u, k, i);
#pragma unroll
            for (int x = 0; x < DPT; ++x)
                if (d0 + x < d) st1(out + d0 + x, acc[x] * qs);
            if (g == 0) cRout[(u * a.m + k) * a.b + i] = (F)col;
        }
    } else {
        // phase 2 (FINAL): row j of O  (monarch.hpp:187-190)
        const T* Ybase = static_cast<const T*>(a.Y.base);
        for (int64_t j0 = 0; j0 < a.m; j0 += RPB) {
            const int64_t j = j0 + rloc;
            const bool valid = j < a.m;
            const int64_t jj = valid ? j : 0;
            F q[DPT], acc[DPT];
            load_slice(Qbase + row_off(a.Q, u, i, jj), d0, d, (F)1, q);
#pragma unroll
            for (int x = 0; x < DPT; ++x) acc[x] = 0;
            for (int64_t k = 0; k < a.m; ++k) {
                F kr[DPT];
                load_slice(Lbase + row_off(a.aL, u, i, k), d0, d, (F)1, kr);
                F dd = 0;
#pragma unroll
                for (int x = 0; x < DPT; ++x) dd = vfma(q[x], kr[x], dd);
                const F sv = group_sum<G>(dd) * qs - cl[k];
                const F l = vexp(sv - s_mx[jj]) * s_isum[jj];
                if (valid && Lout && g == 0) Lout[((u * a.b + i) * a.m + j) * a.m + k] = l;
                F yr[DPT];
                load_slice(Ybase + row_off(a.Y, u, k, i), d0, d, (F)1, yr);
#pragma unroll
                for (int x = 0; x < DPT; ++x) acc[x] = vfma(l, yr[x], acc[x]);
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
template <typename T, typename F, int G>
__global__ void __launch_bounds__(BLOCK) simt_flash_kernel(SimtFlashArgs a) {
    F* sm = smem_as<F>();
    F* smk = sm;
    F* smv = sm + KTILE * a.d;
    constexpr int RPB = BLOCK / G;
    const int g = threadIdx.x % G, rloc = threadIdx.x / G;
    const int64_t u = blockIdx.y;
    const int64_t r = (int64_t)blockIdx.x * RPB + rloc;
    const bool valid = r < a.nq;
    const int d = (int)a.d, d0 = g * DPT;
    // key range of this split
    const int64_t chunk = (a.nk + a.nsplit - 1) / a.nsplit;
    const int64_t kb = (int64_t)blockIdx.z * chunk, ke = kb + chunk < a.nk ? kb + chunk : a.nk;
    F q[DPT], acc[DPT];
    if (valid) {
        load_slice(static_cast<const T*>(a.Q.base) + row_off(a.Q, u, 0, r), d0, d, (F)a.qscale, q);
    } else {
#pragma unroll
        for (int x = 0; x < DPT; ++x) q[x] = 0;
    }
#pragma unroll
    for (int x = 0; x < DPT; ++x) acc[x] = 0;
    double run_max = -INFINITY, norm = 0.0, ent = 0.0;
    for (int64_t l0 = kb; l0 < ke; l0 += KTILE) {
        __syncthreads();
        stage_rows<T>(smk, a.K, u, 0, l0, ke, d);
        stage_rows<T>(smv, a.V, u, 0, l0, ke, d);
        __syncthreads();
        const int nl = (int)((ke - l0) < KTILE ? (ke - l0) : KTILE);
        F sv[KTILE];
        double tmax = -INFINITY;
#pragma unroll
        for (int rr = 0; rr < KTILE; ++rr) {
            sv[rr] = (rr < nl) ? dot_smem<G>(q, smk + rr * d, d0, d) : (F)-INFINITY;
            tmax = fmax(tmax, (double)sv[rr]);
        }
        const double m_new = fmax(run_max, tmax);
        if (!isinf(run_max)) {
            const double delta = run_max - m_new;
            const double alpha = exp(delta);
            ent = alpha * ent + alpha * delta * norm;
            norm *= alpha;
            if (alpha != 1.0) {
                const F af = (F)alpha;
#pragma unroll
                for (int x = 0; x < DPT; ++x) acc[x] *= af;
            }
        }
#pragma unroll
        for (int rr = 0; rr < KTILE; ++rr) {
            if (rr < nl) {
                const double x = (double)sv[rr];
                const double p = exp(x - m_new);
                norm += p;
                ent += p * (x - m_new);
                const F pf = (F)p;
                const F* vr = smv + rr * d;
#pragma unroll
                for (int xx = 0; xx < DPT; ++xx)
                    if (d0 + xx < d) acc[xx] = vfma(pf, vr[d0 + xx], acc[xx]);
            }
        }
        run_max = m_new;
    }
    if (!valid) return;
    if (a.nsplit > 1) {
        // split-KV partial: unnormalised acc and (max, sum, entropy accumulator)
        const int64_t pr = ((int64_t)blockIdx.z * a.U + u) * a.nq + r;
        F* pa = static_cast<F*>(a.part_acc) + pr * d;
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
    const F inv = (F)(1.0 / norm);
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
template <typename T, typename F, int G>
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
    F acc[DPT];
#pragma unroll
    for (int x = 0; x < DPT; ++x) acc[x] = 0;
    for (int s = 0; s < a.nsplit; ++s) {
        const int64_t pr = ((int64_t)s * a.U + u) * a.nq + r;
        const double ms = a.part_stat[pr * 3 + 0], ls = a.part_stat[pr * 3 + 1], es = a.part_stat[pr * 3 + 2];
        if (isinf(ms)) continue;  // empty split
        const double w = exp(ms - m);
        norm += w * ls;
        ent += w * (es + (ms - m) * ls);
        const F wf = (F)w;
        const F* pa = static_cast<const F*>(a.part_acc) + pr * d;
#pragma unroll
        for (int x = 0; x < DPT; ++x)
            if (d0 + x < d) acc[x] = vfma(wf, pa[d0 + x], acc[x]);
    }
    const F inv = (F)(1.0 / norm);
    T* out = static_cast<T*>(const_cast<void*>(a.O.base)) + row_off(a.O, u, 0, r);
#pragma unroll
    for (int x = 0; x < DPT; ++x)
        if (d0 + x < d) st1(out + d0 + x, acc[x] * inv);
    if (g == 0) {
        if (a.lse) a.lse[u * a.nq + r] = (float)(m + log(norm));
        if (a.ent) a.ent[u * a.nq + r] = (float)(log(norm) - ent / norm);
    }
}

template <typename T, typename F>
__global__ void finite_rows_kernel(View q, int64_t U, int64_t rows, int64_t d, int32_t* status) {
    const int64_t total = U * rows * d;
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = e % d, rr = (e / d) % rows, u = e / (d * rows);
        const F v = ld1<F>(static_cast<const T*>(q.base) + row_off(q, u, 0, rr) + x);
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

template <typename T, typename F, int G>
void rstep_launch(const SimtRstepArgs& a, cudaStream_t s) {
    constexpr int RPB = BLOCK / G;
    dim3 grid((unsigned)((a.b + RPB - 1) / RPB), (unsigned)a.m, (unsigned)a.U);
    const size_t smem = 2 * KTILE * a.d * sizeof(F);
    set_smem(simt_rstep_kernel<T, F, G>, smem);
    ProfScope ps(kKSimt, s);
    simt_rstep_kernel<T, F, G><<<grid, BLOCK, smem, s>>>(a);
    count_launch();
    check_launch("simt_rstep");
}
template <typename T, typename F, int G>
void lstep_launch(const SimtLstepArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)a.b, (unsigned)a.U);
    const size_t smem = 2 * a.m * sizeof(F);
    set_smem(simt_lstep_kernel<T, F, G>, smem);
    ProfScope ps(kKSimt, s);
    simt_lstep_kernel<T, F, G><<<grid, BLOCK, smem, s>>>(a);
    count_launch();
    check_launch("simt_lstep");
}
template <typename T, typename F, int G>
void flash_launch(const SimtFlashArgs& a0, cudaStream_t s) {
    constexpr int RPB = BLOCK / G;
    SimtFlashArgs a = a0;
    const int64_t row_blocks = (a.nq + RPB - 1) / RPB;
    // split the keys when the row blocks of one unit fill less than two waves; the split count
    // depends on the per-unit shape only (bitwise-identical results for any unit count)
    a.nsplit = (int32_t)std::max<int64_t>(1, std::min<int64_t>({(2 * 148 + row_blocks - 1) / row_blocks, 32,
                                                                 a.nk / (8 * KTILE)}));
    if (a.nsplit > 1) {
        scratch_alloc(&a.part_acc, sizeof(F) * a.nsplit * a.U * a.nq * a.d, s);
        scratch_alloc(reinterpret_cast<void**>(&a.part_stat), sizeof(double) * 3 * a.nsplit * a.U * a.nq, s);
    }
    const dim3 grid((unsigned)row_blocks, (unsigned)a.U, (unsigned)a.nsplit);
    const size_t smem = 2 * KTILE * a.d * sizeof(F);
    set_smem(simt_flash_kernel<T, F, G>, smem);
    ProfScope ps(kKSimt, s);
    simt_flash_kernel<T, F, G><<<grid, BLOCK, smem, s>>>(a);
    count_launch();
    check_launch("simt_flash");
    if (a.nsplit > 1) {
        simt_flash_combine_kernel<T, F, G><<<dim3((unsigned)row_blocks, (unsigned)a.U), BLOCK, 0, s>>>(a);
        count_launch();
        check_launch("simt_flash_combine");
        VMB_CHECK_CUDA(cudaFreeAsync(a.part_acc, s));
        VMB_CHECK_CUDA(cudaFreeAsync(a.part_stat, s));
    }
}

#define VMB_DISPATCH_G(G_, FN, T_, F_, ...)                              \
    switch (G_) {                                                        \
        case 1: FN<T_, F_, 1>(__VA_ARGS__); break;                       \
        case 2: FN<T_, F_, 2>(__VA_ARGS__); break;                       \
        case 4: FN<T_, F_, 4>(__VA_ARGS__); break;                       \
        default: FN<T_, F_, 8>(__VA_ARGS__); break;                      \
    }
#define VMB_DISPATCH_DT(DT_, G_, FN, ...)                                              \
    switch (DT_) {                                                                     \
        case VMB_BF16: VMB_DISPATCH_G(G_, FN, __nv_bfloat16, float, __VA_ARGS__); break; \
        case VMB_F64: VMB_DISPATCH_G(G_, FN, double, double, __VA_ARGS__); break;      \
        default: VMB_DISPATCH_G(G_, FN, float, float, __VA_ARGS__); break;             \
    }

}  // namespace

void simt_rstep(const SimtRstepArgs& a, vmb_dtype dt, cudaStream_t s) {
    const int G = pick_g(a.d);
    if (a.U == 0 || a.m == 0 || a.b == 0) return;
    VMB_DISPATCH_DT(dt, G, rstep_launch, a, s);
}
void simt_lstep(const SimtLstepArgs& a, vmb_dtype dt, cudaStream_t s) {
    const int G = pick_g(a.d);
    if (a.U == 0 || a.m == 0 || a.b == 0) return;
    VMB_DISPATCH_DT(dt, G, lstep_launch, a, s);
}
void simt_flash(const SimtFlashArgs& a, vmb_dtype dt, cudaStream_t s) {
    const int G = pick_g(a.d);
    if (a.U == 0 || a.nq == 0) return;
    VMB_DISPATCH_DT(dt, G, flash_launch, a, s);
}
void check_finite_rows(View q, int64_t U, int64_t rows, int64_t d, vmb_dtype dt, int32_t* status,
                       cudaStream_t s) {
    const int64_t total = U * rows * d;
    if (total == 0) return;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (dt == VMB_BF16) finite_rows_kernel<__nv_bfloat16, float><<<blocks, 256, 0, s>>>(q, U, rows, d, status);
    else if (dt == VMB_F64) finite_rows_kernel<double, double><<<blocks, 256, 0, s>>>(q, U, rows, d, status);
    else finite_rows_kernel<float, float><<<blocks, 256, 0, s>>>(q, U, rows, d, status);
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
