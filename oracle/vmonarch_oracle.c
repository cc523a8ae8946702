/*
 * vmonarch_oracle.c — CPU restatement of the reference VMonarch forward path.
 *
 * TEST INFRASTRUCTURE ONLY: linked by tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline leg as the checker.  Never part of the product path.
 * See vmonarch_oracle.h for the contract and the reference citations.
 *
 * Parity status: PINNED — tests/test_oracle_pin.py compares this restatement with
 * the reference compiled from /root/reference/proj (oracle/_ref/libvmref.so) and
 * with the committed golden fixtures (tests/golden/, made by
 * tests/golden/make_golden.py from the reference itself).
 */
#include "vmonarch_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- index / bookkeeping functions (bit-exact integer work) ---------------- */

int vmo_make_perm(int64_t b, int64_t n, int64_t* forward_index) {
    if (!(b >= 1 && n >= 1)) return VMO_ERR_DIM;   /* perm.hpp:20 */
    if (n % b != 0) return VMO_ERR_DIM;              /* perm.hpp:21 */
    const int64_t m = n / b;
    for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < m; ++i) forward_index[j * m + i] = i * b + j; /* perm.hpp:28 */
    return VMO_OK;
}

int vmo_factorize(int64_t t_frames, int64_t h, int64_t w, int64_t om, int64_t ob,
                  int64_t* m_out, int64_t* b_out) {
    if (!(t_frames >= 1 && h >= 1 && w >= 1)) return VMO_ERR_DIM; /* video.cpp:14 */
    const int64_t n = t_frames * h * w;
    if (om != 0 || ob != 0) {                                     /* video.cpp:16-19 */
        if (!(om >= 1 && ob >= 1 && om * ob == n)) return VMO_ERR_DIM;
        *m_out = om;
        *b_out = ob;
        return VMO_OK;
    }
    *m_out = t_frames;
    *b_out = h * w;
    return VMO_OK;
}

int vmo_flops_estimate(int64_t t_frames, int64_t h, int64_t w, int64_t om, int64_t ob,
                       int64_t iters, int recompute, int64_t d, vmo_cost_report* rep) {
    int64_t m = 0, b = 0;
    int st = vmo_factorize(t_frames, h, w, om, ob, &m, &b);
    if (st != VMO_OK) return st;
    const uint64_t n = (uint64_t)m * (uint64_t)b;
    const uint64_t t = (uint64_t)iters, du = (uint64_t)d;
    const uint64_t mb = (uint64_t)m + (uint64_t)b;
    const double nd = (double)m * (double)b;
    rep->sparsity = 1.0 - (double)iters * ((double)m + (double)b) / nd;  /* video.cpp:24-28 */
    rep->sparsity_approx = 1.0 - (double)iters / (double)m;             /* video.cpp:30-34 */
    rep->full_attn_flops = 4 * n * n * du;                              /* video.cpp:45 */
    rep->monarch_flops = 2 * (2 * t * n * du * mb + n * du * mb);       /* video.cpp:49 */
    rep->recompute_flops =
        recompute ? 4 * (uint64_t)(h * w) * n * du : 0;                 /* video.cpp:52-54 */
    rep->reduction_ratio = (double)rep->full_attn_flops /
                           (double)(rep->monarch_flops + rep->recompute_flops);
    return VMO_OK;
}

/* ---- element-type-generic kernels ----------------------------------------- */

#define T float
#define S f32
#define EXPT expf
#define LOGT logf
#include "vmonarch_oracle_impl.inc"
#undef T
#undef S
#undef EXPT
#undef LOGT

#define T double
#define S f64
#define EXPT exp
#define LOGT log
#include "vmonarch_oracle_impl.inc"
#undef T
#undef S
#undef EXPT
#undef LOGT

/* ---- f64-only oracles ------------------------------------------------------ */

static double plogp_d(double p) { return p > 0.0 ? p * log(p) : 0.0; }

int vmo_dense_attention_f64(const double* q, const double* k, const double* v, int64_t nq,
                            int64_t nk, int64_t d, int scale, double* out, double* lse,
                            double* ent, double* probs) {
    if (nk < 1) return VMO_ERR_DIM;                                    /* oracle.cpp:13 */
    const double s = scale ? 1.0 / sqrt((double)d) : 1.0;
    double* p = probs ? probs : (double*)malloc(sizeof(double) * (size_t)(nq * nk));
    double* qs = (double*)malloc(sizeof(double) * (size_t)(nq * d));
    for (int64_t x = 0; x < nq * d; ++x) qs[x] = q[x] * s;
    for (int64_t i = 0; i < nq; ++i)                                   /* oracle.cpp:27 */
        for (int64_t j = 0; j < nk; ++j) {
            double acc = 0.0;
            for (int64_t x = 0; x < d; ++x) acc += qs[i * d + x] * k[j * d + x];
            p[i * nk + j] = acc;
        }
    for (int64_t i = 0; i < nq; ++i) {                                 /* oracle.cpp:28-43 */
        double* row = p + i * nk;
        double mx = row[0];
        for (int64_t j = 1; j < nk; ++j) mx = (mx < row[j]) ? row[j] : mx;
        double sum = 0.0;
        for (int64_t j = 0; j < nk; ++j) {
            row[j] = exp(row[j] - mx);
            sum += row[j];
        }
        if (lse) lse[i] = mx + log(sum);
        double e = 0.0;
        for (int64_t j = 0; j < nk; ++j) {
            row[j] /= sum;
            e -= plogp_d(row[j]);
        }
        if (ent) ent[i] = e;
    }
    if (out)                                                           /* oracle.cpp:44 */
        for (int64_t i = 0; i < nq; ++i) {
            double* o = out + i * d;
            for (int64_t x = 0; x < d; ++x) o[x] = 0.0;
            for (int64_t j = 0; j < nk; ++j) {
                const double w = p[i * nk + j];
                for (int64_t x = 0; x < d; ++x) o[x] += w * v[j * d + x];
            }
        }
    free(qs);
    if (!probs) free(p);
    return VMO_OK;
}

int vmo_materialize_monarch_f64(const double* L, const double* R, int64_t b, int64_t n,
                                double* out) {
    if (!(b >= 1 && n >= 1 && n % b == 0)) return VMO_ERR_DIM;         /* oracle.cpp:73 */
    const int64_t m = n / b;
    for (int64_t j = 0; j < m; ++j)                                    /* oracle.cpp:79-88 */
        for (int64_t i = 0; i < b; ++i) {
            double* row = out + (j * b + i) * n;
            for (int64_t k = 0; k < m; ++k) {
                const double lw = L[(i * m + j) * m + k];
                const double* rrow = R + (k * b + i) * b;
                for (int64_t l = 0; l < b; ++l) row[k * b + l] = lw * rrow[l];
            }
        }
    return VMO_OK;
}

int vmo_monarch_objective_f64(const double* L, const double* R, const double* q,
                              const double* k, int64_t m, int64_t b, int64_t d, int scale,
                              double* obj) {
    if (m < 1 || b < 1 || d < 1) return VMO_ERR_DIM;
    const int64_t n = m * b;
    const double sc = scale ? 1.0 / sqrt((double)d) : 1.0;
    double* qs = (double*)malloc(sizeof(double) * (size_t)(n * d));
    double* qb = (double*)malloc(sizeof(double) * (size_t)(n * d));
    double* alpha = (double*)malloc(sizeof(double) * (size_t)d);
    for (int64_t x = 0; x < n * d; ++x) qs[x] = scale ? q[x] * sc : q[x];
    vmo_to_blocked_permuted_f64(qs, m, b, d, qb);
    double acc = 0.0;
    for (int64_t i = 0; i < b; ++i)                                    /* oracle.cpp:118-137 */
        for (int64_t kk = 0; kk < m; ++kk) {
            for (int64_t x = 0; x < d; ++x) alpha[x] = 0.0;
            double r_sum = 0.0, r_ent = 0.0;
            const double* rrow = R + (kk * b + i) * b;
            for (int64_t l = 0; l < b; ++l) {
                const double r = rrow[l];
                r_sum += r;
                r_ent += plogp_d(r);
                const double* krow = k + (kk * b + l) * d;
                for (int64_t x = 0; x < d; ++x) alpha[x] += r * krow[x];
            }
            double lin = 0.0, l_sum = 0.0, l_ent = 0.0;
            for (int64_t j = 0; j < m; ++j) {
                const double lw = L[(i * m + j) * m + kk];
                l_sum += lw;
                l_ent += plogp_d(lw);
                const double* qrow = qb + (i * m + j) * d;
                double dot = 0.0;
                for (int64_t x = 0; x < d; ++x) dot += qrow[x] * alpha[x];
                lin += lw * dot;
            }
            acc += lin - (l_ent * r_sum + l_sum * r_ent);
        }
    *obj = acc;
    free(qs);
    free(qb);
    free(alpha);
    return VMO_OK;
}
