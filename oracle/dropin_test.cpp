// dropin_test.cpp — the drop-in check of include/vmonarch_b200.hpp against the UNMODIFIED
// reference operator.  TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/
// from the reference's own headers and sources under /root/reference/proj; run on a GPU box
// by tests/test_gpu_dropin.py).
//
// The same vmonarch::Mat<float> / TokenGrid / VMonarchConfig / MonarchFactors<float> objects
// go to both calls:
//     vmonarch::vmonarch_attention<float>(qs, ks, vs, grid, cfg, threads, &factors)  (CPU)
//     vmonarch_b200::vmonarch_attention(qs, ks, vs, grid, cfg, threads, &factors)    (B200)
// and the outputs, the factors and the exception types must agree (fp32 parity <= 1e-4).
#include <cmath>
#include <cstdio>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "vmonarch/flash_entropy.hpp"
#include "vmonarch/monarch.hpp"
#include "vmonarch/oracle.hpp"
#include "vmonarch/video.hpp"
#include "vmonarch_b200.hpp"

using vmonarch::Mat;

template <class T = float>
static std::vector<Mat<T>> randn_units(int units, long rows, long cols, uint64_t seed, double sigma) {
    std::vector<Mat<T>> out;
    for (int u = 0; u < units; ++u) {
        std::mt19937_64 rng(seed + 3 * u);
        std::normal_distribution<double> nd(0.0, 1.0);
        Mat<T> m(rows, cols);
        for (auto& x : m.data) x = static_cast<T>(sigma * nd(rng));
        out.push_back(std::move(m));
    }
    return out;
}

template <class T>
static double relfro(const std::vector<T>& a, const std::vector<T>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
        den += double(b[i]) * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1e-300));
}

static int failures = 0;
static void expect(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

static void parity_case(const char* name, vmonarch::TokenGrid grid, vmonarch::VMonarchConfig cfg, double sigma,
                        bool factors) {
    const long n = grid.tokens();
    auto qs = randn_units((int)grid.units(), n, grid.head_dim, 100, sigma);
    auto ks = randn_units((int)grid.units(), n, grid.head_dim, 101, sigma);
    auto vs = randn_units((int)grid.units(), n, grid.head_dim, 102, sigma);
    std::span<const Mat<float>> sq(qs), sk(ks), sv(vs);
    std::vector<vmonarch::MonarchFactors<float>> fr, fg;
    auto ref = vmonarch::vmonarch_attention<float>(sq, sk, sv, grid, cfg, 4, factors ? &fr : nullptr);
    auto got = vmonarch_b200::vmonarch_attention(sq, sk, sv, grid, cfg, 4, factors ? &fg : nullptr);
    double worst = 0;
    for (size_t u = 0; u < ref.size(); ++u) worst = std::max(worst, relfro(got[u].data, ref[u].data));
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: output rel-Fro %.2e (<= 1e-4)", name, worst);
    expect(got.size() == ref.size() && worst <= 1e-4, buf);
    if (factors) {
        double wl = 0, wr = 0;
        for (size_t u = 0; u < fr.size(); ++u) {
            wl = std::max(wl, relfro(fg[u].L.data, fr[u].L.data));
            wr = std::max(wr, relfro(fg[u].R.data, fr[u].R.data));
        }
        std::snprintf(buf, sizeof buf, "%s: factors L %.2e R %.2e (<= 1e-4)", name, wl, wr);
        expect(fg.size() == fr.size() && wl <= 1e-4 && wr <= 1e-4, buf);
    }
}

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // C1 (BASELINE configs[0]): B=1 H=2 d=64, 4 frames x 8x8, fp32, t=3
    vmonarch::TokenGrid c1{4, 8, 8, 64, 2, 1};
    vmonarch::VMonarchConfig cfg3;
    cfg3.iters = 3;
    parity_case("C1", c1, cfg3, 1.0, true);
    vmonarch::VMonarchConfig norec;
    norec.recompute_first_frame = false;
    parity_case("C1 without first-frame recompute, t=2", c1, norec, 1.0, true);
    vmonarch::VMonarchConfig ov;
    ov.override_m_b = std::make_pair(8L, 32L);
    parity_case("override factorization (m,b)=(8,32)", c1, ov, 1.0, false);
    vmonarch::VMonarchConfig noclamp;
    noclamp.clamp_enabled = false;
    parity_case("clamp disabled, sigma=2", vmonarch::TokenGrid{3, 6, 5, 32, 3, 1}, noclamp, 2.0, false);
    parity_case("batch 2 x heads 2, d=16", vmonarch::TokenGrid{5, 4, 4, 16, 2, 2}, vmonarch::VMonarchConfig{}, 3.0,
                false);

    // T = double (the reference's own tests run in double): the f64 mode, agreement to round-off
    {
        struct DCase {
            const char* name;
            vmonarch::TokenGrid g;
            int iters;
            bool recompute;
            double sigma;
        };
        for (const DCase& dc : {DCase{"f64 C1 t=3", {4, 8, 8, 64, 2, 1}, 3, true, 1.0},
                                DCase{"f64 3x6x5 d=32 sigma=3", {3, 6, 5, 32, 3, 1}, 2, true, 3.0},
                                DCase{"f64 5x4x4 d=16 batch 2, no recompute", {5, 4, 4, 16, 2, 2}, 2, false, 1.0}}) {
            const long n = dc.g.tokens();
            auto qs = randn_units<double>((int)dc.g.units(), n, dc.g.head_dim, 300, dc.sigma);
            auto ks = randn_units<double>((int)dc.g.units(), n, dc.g.head_dim, 301, dc.sigma);
            auto vs = randn_units<double>((int)dc.g.units(), n, dc.g.head_dim, 302, dc.sigma);
            std::span<const Mat<double>> sq(qs), sk(ks), sv(vs);
            vmonarch::VMonarchConfig cf;
            cf.iters = dc.iters;
            cf.recompute_first_frame = dc.recompute;
            std::vector<vmonarch::MonarchFactors<double>> fr, fg;
            auto ref = vmonarch::vmonarch_attention<double>(sq, sk, sv, dc.g, cf, 4, &fr);
            auto got = vmonarch_b200::vmonarch_attention(sq, sk, sv, dc.g, cf, 4, &fg);
            double worst = 0, wl = 0, wr = 0;
            for (size_t u = 0; u < ref.size(); ++u) {
                worst = std::max(worst, relfro(got[u].data, ref[u].data));
                wl = std::max(wl, relfro(fg[u].L.data, fr[u].L.data));
                wr = std::max(wr, relfro(fg[u].R.data, fr[u].R.data));
            }
            char buf[240];
            std::snprintf(buf, sizeof buf, "%s: output rel-Fro %.2e, factors L %.2e R %.2e (<= 1e-11)", dc.name, worst,
                          wl, wr);
            expect(got.size() == ref.size() && worst <= 1e-11 && wl <= 1e-11 && wr <= 1e-11, buf);
        }
    }

    // the pipelined host path: units streamed in chunks (1 and 3 units) equal the one-chunk call
    // bitwise, and equal the reference
    {
        vmonarch::TokenGrid g{4, 8, 16, 128, 7, 1};
        const long n = g.tokens();
        auto qs = randn_units((int)g.units(), n, 128, 400, 1.0);
        auto ks = randn_units((int)g.units(), n, 128, 401, 1.0);
        auto vs = randn_units((int)g.units(), n, 128, 402, 1.0);
        std::span<const Mat<float>> sq(qs), sk(ks), sv(vs);
        vmonarch::VMonarchConfig cf;
        std::vector<vmonarch::MonarchFactors<float>>* none = nullptr;
        for (auto prec : {vmonarch_b200::Precision::fp32, vmonarch_b200::Precision::bf16}) {
            auto whole = vmonarch_b200::vmonarch_attention(sq, sk, sv, g, cf, 1, none, prec, 7);
            bool same = true;
            for (int64_t ch : {1, 3}) {
                auto part = vmonarch_b200::vmonarch_attention(sq, sk, sv, g, cf, 1, none, prec, ch);
                for (size_t u = 0; u < whole.size(); ++u) same = same && part[u].data == whole[u].data;
            }
            auto ref = vmonarch::vmonarch_attention<float>(sq, sk, sv, g, cf, 4);
            double worst = 0;
            for (size_t u = 0; u < ref.size(); ++u) worst = std::max(worst, relfro(whole[u].data, ref[u].data));
            const bool bf = prec == vmonarch_b200::Precision::bf16;
            char buf[200];
            std::snprintf(buf, sizeof buf, "%s host pipeline, chunks of 1/3/7 units: bitwise equal %s, rel-Fro %.2e",
                          bf ? "bf16" : "fp32", same ? "yes" : "NO", worst);
            expect(same && worst <= (bf ? 2e-2 : 1e-4), buf);
        }
        // a non-finite Q in the last chunk is still reported
        qs[6].data[3] = NAN;
        expect(throws<std::domain_error>([&] {
                   vmonarch_b200::vmonarch_attention(sq, sk, sv, g, cf, 1, none, vmonarch_b200::Precision::bf16, 2);
               }),
               "host pipeline: non-finite Q in the last chunk -> std::domain_error");
    }

    // bf16 performance mode of the façade (Precision::bf16): float in / float out on the tcgen05 path
    {
        for (auto g : {vmonarch::TokenGrid{4, 8, 8, 64, 2, 1}, vmonarch::TokenGrid{4, 8, 16, 128, 2, 1},
                       vmonarch::TokenGrid{21, 6, 7, 128, 1, 1}}) {
            const long n = g.tokens();
            auto qs = randn_units((int)g.units(), n, g.head_dim, 200, 1.0);
            auto ks = randn_units((int)g.units(), n, g.head_dim, 201, 1.0);
            auto vs = randn_units((int)g.units(), n, g.head_dim, 202, 1.0);
            std::span<const Mat<float>> sq(qs), sk(ks), sv(vs);
            vmonarch::VMonarchConfig cf;
            auto ref = vmonarch::vmonarch_attention<float>(sq, sk, sv, g, cf, 4);
            std::vector<vmonarch::MonarchFactors<float>>* none = nullptr;
            auto got = vmonarch_b200::vmonarch_attention(sq, sk, sv, g, cf, 4, none, vmonarch_b200::Precision::bf16);
            double worst = 0;
            for (size_t u = 0; u < ref.size(); ++u) worst = std::max(worst, relfro(got[u].data, ref[u].data));
            char buf[200];
            std::snprintf(buf, sizeof buf, "bf16 mode %ldx%ldx%ld d=%ld: output rel-Fro %.2e (<= 2e-2)", (long)g.t_frames,
                          (long)g.h, (long)g.w, (long)g.head_dim, worst);
            expect(worst <= 2e-2, buf);
        }
    }

    // companions: monarch_attention, flash_entropy_fwd / _bwd, dense_forward, flops_estimate
    {
        auto q = randn_units(1, 256, 32, 40, 1.0)[0], k = randn_units(1, 256, 32, 41, 1.0)[0],
             v = randn_units(1, 256, 32, 42, 1.0)[0], g = randn_units(1, 256, 32, 43, 1.0)[0];
        vmonarch::MonarchConfig mc{16, 16, 3, 0.1, true};
        auto r1 = vmonarch::monarch_attention(q, k, v, mc);
        auto r2 = vmonarch_b200::monarch_attention<vmonarch::MonarchResult<float>>(q, k, v, mc);
        char buf[200];
        std::snprintf(buf, sizeof buf, "monarch_attention (m,b)=(16,16) t=3: output %.2e, L %.2e, R %.2e",
                      relfro(r2.output.data, r1.output.data), relfro(r2.factors.L.data, r1.factors.L.data),
                      relfro(r2.factors.R.data, r1.factors.R.data));
        expect(relfro(r2.output.data, r1.output.data) <= 1e-4 && relfro(r2.factors.L.data, r1.factors.L.data) <= 1e-4 &&
                   relfro(r2.factors.R.data, r1.factors.R.data) <= 1e-4, buf);
        vmonarch::Mat<float> qs = q;
        for (auto& x : qs.data) x *= 1.f / std::sqrt(32.f);
        vmonarch::TileConfig tc{16, 32};
        auto f1 = vmonarch::flash_entropy_fwd(qs, k, v, tc);
        auto f2 = vmonarch_b200::flash_entropy_fwd<vmonarch::FlashFwdResult<float>>(qs, k, v, tc);
        const double eo = relfro(f2.output.data, f1.output.data), el = relfro(f2.lse, f1.lse), eh = relfro(f2.entropy, f1.entropy);
        std::snprintf(buf, sizeof buf, "flash_entropy_fwd: output %.2e, lse %.2e, entropy %.2e", eo, el, eh);
        expect(eo <= 1e-4 && el <= 1e-5 && eh <= 1e-4, buf);
        std::vector<float> dh(256);
        for (int i = 0; i < 256; ++i) dh[i] = 0.01f * (i % 7) - 0.03f;
        auto b1 = vmonarch::flash_entropy_bwd(qs, k, v, f1.output, g, f1.lse, f1.entropy, dh, true, tc);
        auto b2 = vmonarch_b200::flash_entropy_bwd<vmonarch::FlashBwdResult<float>>(qs, k, v, f1.output, g, f1.lse,
                                                                                    f1.entropy, dh, true, tc);
        const double gq = relfro(b2.dq.data, b1.dq.data), gk = relfro(b2.dk.data, b1.dk.data), gv = relfro(b2.dv.data, b1.dv.data);
        std::snprintf(buf, sizeof buf, "flash_entropy_bwd (entropy grad): dq %.2e, dk %.2e, dv %.2e", gq, gk, gv);
        expect(gq <= 1e-4 && gk <= 1e-4 && gv <= 1e-4, buf);
        auto d1 = vmonarch::dense_forward(q, k, v, true);
        auto d2 = vmonarch_b200::dense_forward(q, k, v, true);
        std::snprintf(buf, sizeof buf, "dense_forward: %.2e", relfro(d2.data, d1.data));
        expect(relfro(d2.data, d1.data) <= 1e-4, buf);
        vmonarch::TokenGrid wan{81, 28, 52, 64, 1, 1};
        auto c1 = vmonarch::flops_estimate(wan, vmonarch::VMonarchConfig{}, 64);
        auto c2 = vmonarch_b200::flops_estimate<vmonarch::CostReport>(wan, vmonarch::VMonarchConfig{}, 64);
        expect(c1.monarch_flops == c2.monarch_flops && c1.full_attn_flops == c2.full_attn_flops &&
                   c1.recompute_flops == c2.recompute_flops && c1.reduction_ratio == c2.reduction_ratio &&
                   c1.sparsity == c2.sparsity,
               "flops_estimate wan-321f d=64: bit-exact");
        expect(throws<std::domain_error>([&] {
                   vmonarch_b200::flash_entropy_fwd<vmonarch::FlashFwdResult<float>>(qs, vmonarch::Mat<float>(0, 32),
                                                                                     vmonarch::Mat<float>(0, 32), tc);
               }),
               "flash over empty keys -> std::domain_error");
    }

    // error contract (check.hpp:10-20): same exception classes as the reference
    auto qs = randn_units(2, 256, 64, 7, 1.0);
    auto ks = randn_units(2, 256, 64, 8, 1.0);
    auto vs = randn_units(2, 256, 64, 9, 1.0);
    std::span<const Mat<float>> sq(qs), sk(ks), sv(vs);
    std::span<const Mat<float>> sq1(qs.data(), 1);
    expect(throws<std::invalid_argument>([&] { vmonarch::vmonarch_attention<float>(sq1, sk, sv, c1, cfg3); }) &&
               throws<std::invalid_argument>([&] { vmonarch_b200::vmonarch_attention(sq1, sk, sv, c1, cfg3); }),
           "unit-count mismatch -> std::invalid_argument in both");
    vmonarch::VMonarchConfig badov;
    badov.override_m_b = std::make_pair(7L, 37L);
    expect(throws<std::invalid_argument>([&] { vmonarch::vmonarch_attention<float>(sq, sk, sv, c1, badov); }) &&
               throws<std::invalid_argument>([&] { vmonarch_b200::vmonarch_attention(sq, sk, sv, c1, badov); }),
           "override with m*b != N -> std::invalid_argument in both");
    qs[1].data[17] = NAN;
    expect(throws<std::domain_error>([&] { vmonarch::vmonarch_attention<float>(sq, sk, sv, c1, cfg3); }) &&
               throws<std::domain_error>([&] { vmonarch_b200::vmonarch_attention(sq, sk, sv, c1, cfg3); }),
           "non-finite Q -> std::domain_error in both");
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
