// ref_shim.cpp — extern "C" entry points onto the UNMODIFIED reference library.
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources (/root/reference/proj/src/*.cpp, headers under
// /root/reference/proj/include) into oracle/_ref/libvmref.so.  No reference source
// is copied into this repository: this file only marshals raw buffers into the
// reference's containers and calls its public templates.
//
// Used (1) to pin the C restatement in oracle/vmonarch_oracle.c, (2) to generate
// tests/golden/ fixtures, (3) as the CPU baseline (`bench.py --impl reference`,
// cpu_baseline.kind = "reference").
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "vmonarch/flash_entropy.hpp"
#include "vmonarch/monarch.hpp"
#include "vmonarch/oracle.hpp"
#include "vmonarch/perm.hpp"
#include "vmonarch/video.hpp"

using namespace vmonarch;

namespace {

// Map the reference's exception classes onto the shared status codes.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::domain_error&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::logic_error&) {
        return 3;
    } catch (...) {
        return 4;
    }
}

template <class T>
Mat<T> mat_from(const T* p, idx rows, idx cols) {
    Mat<T> m(rows, cols);
    std::memcpy(m.data.data(), p, sizeof(T) * static_cast<std::size_t>(rows * cols));
    return m;
}

template <class T>
Tensor3<T> t3_from(const T* p, idx a, idx b, idx c) {
    Tensor3<T> t(a, b, c);
    std::memcpy(t.data.data(), p, sizeof(T) * static_cast<std::size_t>(a * b * c));
    return t;
}

template <class T>
void copy_out(const std::vector<T>& v, T* dst) {
    if (dst) std::memcpy(dst, v.data(), sizeof(T) * v.size());
}

template <class T>
int rstep(int64_t m, int64_t b, int64_t d, const T* aR, const T* cR, const T* Kb,
          double clamp_min, int clamp_enabled, T* aL, T* cL, T* R) {
    return guarded([&] {
        MonarchConfig cfg;
        cfg.m = m;
        cfg.b = b;
        cfg.iters = 1;
        cfg.clamp_min = clamp_min;
        cfg.clamp_enabled = clamp_enabled != 0;
        IterState<T> st;
        st.aR = t3_from(aR, m, b, d);
        st.cR = mat_from(cR, m, b);
        Tensor3<T> kb = t3_from(Kb, m, b, d);
        Tensor3<T> r;
        r_update(st, kb, cfg, r);
        copy_out(st.aL.data, aL);
        copy_out(st.cL.data, cL);
        copy_out(r.data, R);
    });
}

template <class T>
int lstep(int64_t m, int64_t b, int64_t d, const T* Qb, const T* aL, const T* cL, T* aR,
          T* cR, T* L) {
    return guarded([&] {
        MonarchConfig cfg;
        cfg.m = m;
        cfg.b = b;
        cfg.iters = 1;
        IterState<T> st;
        st.aL = t3_from(aL, b, m, d);
        st.cL = mat_from(cL, b, m);
        Tensor3<T> qb = t3_from(Qb, b, m, d);
        Tensor3<T> l;
        l_update(st, qb, cfg, l);
        copy_out(st.aR.data, aR);
        copy_out(st.cR.data, cR);
        copy_out(l.data, L);
    });
}

template <class T>
int monarch(const T* q, const T* k, const T* v, int64_t m, int64_t b, int64_t d,
            int64_t iters, double clamp_min, int clamp_enabled, T* out, T* L, T* R) {
    return guarded([&] {
        MonarchConfig cfg;
        cfg.m = m;
        cfg.b = b;
        cfg.iters = iters;
        cfg.clamp_min = clamp_min;
        cfg.clamp_enabled = clamp_enabled != 0;
        const idx n = m * b;
        auto res = monarch_attention(mat_from(q, n, d), mat_from(k, n, d), mat_from(v, n, d), cfg);
        copy_out(res.output.data, out);
        copy_out(res.factors.L.data, L);
        copy_out(res.factors.R.data, R);
    });
}

template <class T>
int flash(const T* q, const T* k, const T* v, int64_t nq, int64_t nk, int64_t d, int64_t br,
          int64_t bc, T* out, T* lse, T* ent) {
    return guarded([&] {
        TileConfig tc;
        tc.b_r = br;
        tc.b_c = bc;
        auto res = flash_entropy_fwd(mat_from(q, nq, d), mat_from(k, nk, d), mat_from(v, nk, d), tc);
        copy_out(res.output.data, out);
        copy_out(res.lse, lse);
        copy_out(res.entropy, ent);
    });
}

template <class T>
int flash_bwd(const T* q, const T* k, const T* v, const T* o, const T* dout, const T* lse, const T* ent,
              const T* dent, int64_t nq, int64_t nk, int64_t d, int eg, int64_t br, int64_t bc, T* dq, T* dk,
              T* dv) {
    return guarded([&] {
        TileConfig tc;
        tc.b_r = br;
        tc.b_c = bc;
        std::vector<T> l(lse, lse + nq), e, de;
        if (ent) e.assign(ent, ent + nq);
        if (dent) de.assign(dent, dent + nq);
        auto r = flash_entropy_bwd(mat_from(q, nq, d), mat_from(k, nk, d), mat_from(v, nk, d), mat_from(o, nq, d),
                                   mat_from(dout, nq, d), l, e, de, eg != 0, tc);
        copy_out(r.dq.data, dq);
        copy_out(r.dk.data, dk);
        copy_out(r.dv.data, dv);
    });
}

// video.hpp:84-150 over `units` independent (N, d) matrices laid out back to back.
template <class T>
int vmonarch_multi(int64_t units, const T* q, const T* k, const T* v, int64_t t_frames,
                   int64_t h, int64_t w, int64_t d, int64_t iters, double clamp_min,
                   int clamp_enabled, int recompute, int64_t om, int64_t ob, int threads,
                   T* out) {
    return guarded([&] {
        TokenGrid g;
        g.t_frames = t_frames;
        g.h = h;
        g.w = w;
        g.head_dim = d;
        g.heads = units;
        g.batch = 1;
        VMonarchConfig cfg;
        cfg.iters = iters;
        cfg.clamp_min = clamp_min;
        cfg.clamp_enabled = clamp_enabled != 0;
        cfg.recompute_first_frame = recompute != 0;
        if (om != 0 || ob != 0) cfg.override_m_b = std::pair<idx, idx>{om, ob};
        const idx n = g.tokens();
        std::vector<Mat<T>> qs, ks, vs;
        for (idx u = 0; u < units; ++u) {
            qs.push_back(mat_from(q + u * n * d, n, d));
            ks.push_back(mat_from(k + u * n * d, n, d));
            vs.push_back(mat_from(v + u * n * d, n, d));
        }
        auto o = vmonarch_attention<T>(qs, ks, vs, g, cfg, threads);
        for (idx u = 0; u < units; ++u) std::memcpy(out + u * n * d, o[u].data.data(), sizeof(T) * n * d);
    });
}

}  // namespace

extern "C" {

int vmr_make_perm(int64_t b, int64_t n, int64_t* out) {
    return guarded([&] {
        Perm p = make_perm(b, n);
        std::memcpy(out, p.forward_index.data(), sizeof(int64_t) * p.forward_index.size());
    });
}

int vmr_to_blocked_permuted_f32(const float* x, int64_t m, int64_t b, int64_t d, float* out) {
    return guarded([&] { copy_out(to_blocked_permuted(mat_from(x, m * b, d), m, b).data, out); });
}

int vmr_flops_estimate(int64_t t_frames, int64_t h, int64_t w, int64_t om, int64_t ob,
                       int64_t iters, int recompute, int64_t d, double* sparsity,
                       double* sparsity_approx, uint64_t* monarch, uint64_t* full,
                       uint64_t* recomp, double* ratio) {
    return guarded([&] {
        TokenGrid g{t_frames, h, w, d};
        VMonarchConfig cfg;
        cfg.iters = iters;
        cfg.recompute_first_frame = recompute != 0;
        if (om != 0 || ob != 0) cfg.override_m_b = std::pair<idx, idx>{om, ob};
        CostReport r = flops_estimate(g, cfg, d);
        *sparsity = r.sparsity;
        *sparsity_approx = r.sparsity_approx;
        *monarch = r.monarch_flops;
        *full = r.full_attn_flops;
        *recomp = r.recompute_flops;
        *ratio = r.reduction_ratio;
    });
}

#define VMR_TYPED(T, S)                                                                         \
    int vmr_rstep_##S(int64_t m, int64_t b, int64_t d, const T* aR, const T* cR, const T* Kb,  \
                      double cm, int ce, T* aL, T* cL, T* R) {                                  \
        return rstep<T>(m, b, d, aR, cR, Kb, cm, ce, aL, cL, R);                                \
    }                                                                                           \
    int vmr_lstep_##S(int64_t m, int64_t b, int64_t d, const T* Qb, const T* aL, const T* cL,  \
                      T* aR, T* cR, T* L) {                                                     \
        return lstep<T>(m, b, d, Qb, aL, cL, aR, cR, L);                                        \
    }                                                                                           \
    int vmr_monarch_attention_##S(const T* q, const T* k, const T* v, int64_t m, int64_t b,    \
                                  int64_t d, int64_t iters, double cm, int ce, T* out, T* L,   \
                                  T* R) {                                                       \
        return monarch<T>(q, k, v, m, b, d, iters, cm, ce, out, L, R);                          \
    }                                                                                           \
    int vmr_flash_entropy_fwd_##S(const T* q, const T* k, const T* v, int64_t nq, int64_t nk,  \
                                  int64_t d, int64_t br, int64_t bc, T* out, T* lse, T* ent) { \
        return flash<T>(q, k, v, nq, nk, d, br, bc, out, lse, ent);                             \
    }                                                                                           \
    int vmr_flash_entropy_bwd_##S(const T* q, const T* k, const T* v, const T* o, const T* dout, \
                                  const T* lse, const T* ent, const T* dent, int64_t nq,       \
                                  int64_t nk, int64_t d, int eg, int64_t br, int64_t bc, T* dq, \
                                  T* dk, T* dv) {                                               \
        return flash_bwd<T>(q, k, v, o, dout, lse, ent, dent, nq, nk, d, eg, br, bc, dq, dk, dv); \
    }                                                                                           \
    int vmr_vmonarch_attention_##S(int64_t units, const T* q, const T* k, const T* v,          \
                                   int64_t tf, int64_t h, int64_t w, int64_t d, int64_t iters, \
                                   double cm, int ce, int rc, int64_t om, int64_t ob,          \
                                   int threads, T* out) {                                       \
        return vmonarch_multi<T>(units, q, k, v, tf, h, w, d, iters, cm, ce, rc, om, ob,        \
                                 threads, out);                                                 \
    }

VMR_TYPED(float, f32)
VMR_TYPED(double, f64)

int vmr_dense_attention_f64(const double* q, const double* k, const double* v, int64_t nq,
                            int64_t nk, int64_t d, int scale, double* out, double* lse,
                            double* ent) {
    return guarded([&] {
        auto r = dense_attention(mat_from(q, nq, d), mat_from(k, nk, d), mat_from(v, nk, d), scale != 0);
        copy_out(r.output.data, out);
        copy_out(r.logsumexp, lse);
        copy_out(r.entropy, ent);
    });
}

}  // extern "C"
