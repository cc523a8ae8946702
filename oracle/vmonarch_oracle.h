/*
 * vmonarch_oracle.h — CPU restatement of the reference VMonarch forward path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2601_22275_b200/,
 * include/vmb.h, libvmb.so) may include, link or call this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg use it,
 * and only as the checker / CPU baseline.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj) in plain C, in the same operation order, so that the
 * float variant reproduces the reference's float results (pinned against the
 * reference itself, compiled from source into oracle/_ref/, by
 * tests/test_oracle_pin.py and against the committed fixtures in tests/golden/).
 *
 * Element type T in {float, double}: functions are emitted twice with suffixes
 * _f32 and _f64 from vmonarch_oracle_impl.inc.  Row statistics accumulate in
 * double regardless of T, exactly like the reference.
 *
 * Status codes mirror the reference exception classes (check.hpp:10-20):
 *   VMO_OK = 0, VMO_ERR_DIM (std::invalid_argument), VMO_ERR_DOMAIN
 *   (std::domain_error), VMO_ERR_STATE (std::logic_error).
 */
#ifndef VMONARCH_ORACLE_H
#define VMONARCH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VMO_OK = 0, VMO_ERR_DIM = 1, VMO_ERR_DOMAIN = 2, VMO_ERR_STATE = 3 };

/* perm.hpp:19-30  forward_index[j*m+i] = i*b+j, m = n/b. */
int vmo_make_perm(int64_t b, int64_t n, int64_t* forward_index);

/* video.cpp:13-22  (m,b) = (T, h*w) unless override (om, ob) with om*ob == N. */
int vmo_factorize(int64_t t_frames, int64_t h, int64_t w, int64_t om, int64_t ob,
                  int64_t* m_out, int64_t* b_out);

/* video.cpp:36-59  FLOP convention: 2 FLOPs/MAC, matmuls only. */
typedef struct {
    double sparsity, sparsity_approx;
    uint64_t monarch_flops, full_attn_flops, recompute_flops;
    double reduction_ratio;
} vmo_cost_report;
int vmo_flops_estimate(int64_t t_frames, int64_t h, int64_t w, int64_t om, int64_t ob,
                       int64_t iters, int recompute, int64_t d, vmo_cost_report* rep);

#define VMO_DECL(T, S)                                                                      \
    /* mat.hpp:99-113  out[i][j] = x[j*b+i], out (b,m,d). */                                \
    int vmo_to_blocked_permuted_##S(const T* x, int64_t m, int64_t b, int64_t d, T* out);   \
    /* monarch.hpp:53-103.  aR (m,b,d), cR (m,b), Kb (m,b,d) -> aL (b,m,d), cL (b,m),       \
     * R (m,b,b) (R may be NULL; scratch is then allocated internally). */                   \
    int vmo_rstep_##S(int64_t m, int64_t b, int64_t d, const T* aR, const T* cR,            \
                      const T* Kb, double clamp_min, int clamp_enabled, T* aL, T* cL,      \
                      T* R);                                                                \
    /* monarch.hpp:105-147.  Qb (b,m,d), aL (b,m,d), cL (b,m) -> aR (m,b,d), cR (m,b),      \
     * L (b,m,m) (may be NULL). */                                                          \
    int vmo_lstep_##S(int64_t m, int64_t b, int64_t d, const T* Qb, const T* aL,            \
                      const T* cL, T* aR, T* cR, T* L);                                     \
    /* monarch.hpp:155-193 (prescale, layouts, init_state, t iterations, assembly).         \
     * q,k,v (m*b, d) row-major -> out (m*b, d); L (b,m,m), R (m,b,b) optional. */          \
    int vmo_monarch_attention_##S(const T* q, const T* k, const T* v, int64_t m,            \
                                  int64_t b, int64_t d, int64_t iters, double clamp_min,    \
                                  int clamp_enabled, T* out, T* L, T* R);                   \
    /* flash_entropy.hpp:85-139 (with absorb_stats 20-51).  Q pre-scaled by the caller. */  \
    int vmo_flash_entropy_fwd_##S(const T* q, const T* k, const T* v, int64_t nq,           \
                                  int64_t nk, int64_t d, int64_t br, int64_t bc, T* out,    \
                                  T* lse, T* ent);                                          \
    /* flash_entropy.hpp:146-221 tiled backward (entropy_grad adds -dH P (S - lse + H)). */  \
    int vmo_flash_entropy_bwd_##S(const T* q, const T* k, const T* v, const T* o,           \
                                  const T* dout, const T* lse, const T* ent, const T* dent, \
                                  int64_t nq, int64_t nk, int64_t d, int entropy_grad,      \
                                  int64_t br, int64_t bc, T* dq, T* dk, T* dv);             \
    /* video.hpp:84-150 for ONE batch*head unit (units are independent, video.hpp:115).     \
     * override (om, ob) = (0,0) for the default factorization. */                          \
    int vmo_vmonarch_unit_##S(const T* q, const T* k, const T* v, int64_t t_frames,         \
                              int64_t h, int64_t w, int64_t d, int64_t iters,               \
                              double clamp_min, int clamp_enabled, int recompute,           \
                              int64_t om, int64_t ob, int64_t br, int64_t bc, T* out, T* L, \
                              T* R);                                                        \
    /* oracle.hpp:36-72  row-blocked (64 rows) quadratic baseline, scale = 1/sqrt(d). */    \
    int vmo_dense_forward_##S(const T* q, const T* k, const T* v, int64_t nq, int64_t nk,   \
                              int64_t d, int scale, T* out);

VMO_DECL(float, f32)
VMO_DECL(double, f64)
#undef VMO_DECL

/* oracle.cpp:9-47  f64 dense attention; probs (nq,nk) may be NULL. */
int vmo_dense_attention_f64(const double* q, const double* k, const double* v, int64_t nq,
                            int64_t nk, int64_t d, int scale, double* out, double* lse,
                            double* ent, double* probs);
/* oracle.cpp:72-90  M[j*b+i, k*b+l] = L[i][j,k] * R[k][i,l]; out (n,n). */
int vmo_materialize_monarch_f64(const double* L, const double* R, int64_t b, int64_t n,
                                double* out);
/* oracle.cpp:92-139  blockwise <M, QK^T s> + H(M). */
int vmo_monarch_objective_f64(const double* L, const double* R, const double* q,
                              const double* k, int64_t m, int64_t b, int64_t d, int scale,
                              double* obj);

/* Workload generator with the reference's convention (test_support.hpp:17-24,
 * bench_main.cpp:78-90): std::mt19937_64(seed) + std::normal_distribution<double>(0,
 * sigma), one value per element, cast to the element type.  Implemented in C++
 * (oracle/workload.cpp) because the normal sampler is libstdc++'s. */
void vmo_randn_f64(int64_t n, uint64_t seed, double sigma, double* out);
void vmo_randn_f32(int64_t n, uint64_t seed, double sigma, float* out);

#ifdef __cplusplus
}
#endif
#endif
