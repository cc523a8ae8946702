// vmonarch_b200.hpp — C++ drop-in façade over the libvmb C ABI (include/vmb.h).
//
// Same call shape, argument meaning and exception types as the reference operator
// (/root/reference/proj/include/vmonarch/video.hpp:84-150, check.hpp:10-20) and its
// companions monarch_attention (monarch.hpp:155-193), flash_entropy_fwd / _bwd
// (flash_entropy.hpp:85-221), dense_forward (oracle.hpp:36-72), factorize / flops_estimate
// (video.cpp:13-59); where the reference returns its own aggregate (MonarchResult,
// FlashFwdResult, FlashBwdResult, CostReport) the caller names that type as the first
// template argument, e.g. vmonarch_b200::flash_entropy_fwd<vmonarch::FlashFwdResult<float>>(...):
//
//   // reference                                   // here (B200)
//   vmonarch::vmonarch_attention<float>(            vmonarch_b200::vmonarch_attention(
//       qs, ks, vs, grid, cfg, threads,                 qs, ks, vs, grid, cfg, threads,
//       &factors);                                      &factors);
//
// The façade is generic over the caller's container types, so a reference user passes its
// own vmonarch::Mat<float> / TokenGrid / VMonarchConfig / MonarchFactors<float> objects
// unchanged (duck-typed members: Mat{rows, cols, data}, Tensor3{d0, d1, d2, data},
// TokenGrid{t_frames, h, w, head_dim, heads, batch}, VMonarchConfig{iters, clamp_min,
// clamp_enabled, recompute_first_frame, override_m_b}).  `threads` is accepted for
// signature parity (all units run in one stream-ordered device call).
//
// Host buffers are copied to the device, the forward runs in the fp32 parity mode (CUDA
// cores, the reference precision policy; <= 1e-4 vs the reference) for T = float, and the
// result is copied back.  Device-resident bf16 callers use the C ABI directly
// (vmb_vmonarch_fwd with VMB_BF16: the tcgen05 path).  Errors are thrown as
// std::invalid_argument ("dimension error: ..."), std::domain_error ("domain error: ..."),
// std::logic_error ("state error: ...") or std::runtime_error (CUDA failures).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "vmb.h"

namespace vmonarch_b200 {

// ---------------------------------------------------------------- errors (check.hpp:10-20)
[[noreturn]] inline void raise_status(vmb_status st) {
    const std::string msg = vmb_last_error();
    switch (st) {
        case VMB_ERR_DIM: throw std::invalid_argument(msg);
        case VMB_ERR_DOMAIN: throw std::domain_error(msg);
        case VMB_ERR_STATE: throw std::logic_error(msg);
        default: throw std::runtime_error(msg.empty() ? std::string("libvmb error") : msg);
    }
}
inline void check(vmb_status st) {
    if (st != VMB_OK) raise_status(st);
}
inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda error: ") + what + ": " + cudaGetErrorString(e));
}
inline void check_dim(bool ok, const std::string& msg) {
    if (!ok) throw std::invalid_argument("dimension error: " + msg);
}

// RAII device buffer
class DeviceBuffer {
public:
    explicit DeviceBuffer(size_t bytes) : bytes_(bytes) {
        if (bytes) check_cuda(cudaMalloc(&ptr_, bytes), "cudaMalloc");
    }
    ~DeviceBuffer() {
        if (ptr_) cudaFree(ptr_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_) {
        o.ptr_ = nullptr;
        o.bytes_ = 0;
    }
    void* get() const { return ptr_; }
    size_t size() const { return bytes_; }

private:
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

// ---------------------------------------------------------------- config conversion
template <class GridT>
vmb_grid to_grid(const GridT& g) {
    return vmb_grid{(int64_t)g.t_frames, (int64_t)g.h, (int64_t)g.w, (int64_t)g.head_dim, (int64_t)g.heads,
                    (int64_t)g.batch};
}
template <class CfgT>
vmb_config to_config(const CfgT& c) {
    vmb_config v;
    vmb_config_default(&v);
    v.iters = (int64_t)c.iters;
    v.clamp_min = (double)c.clamp_min;
    v.clamp_enabled = c.clamp_enabled ? 1 : 0;
    v.recompute_first_frame = c.recompute_first_frame ? 1 : 0;
    if (c.override_m_b) {
        v.override_m = (int64_t)c.override_m_b->first;
        v.override_b = (int64_t)c.override_m_b->second;
    }
    return v;
}

// video.cpp:13-22
template <class GridT, class CfgT>
std::pair<int64_t, int64_t> factorize(const GridT& grid, const CfgT& cfg) {
    const vmb_grid g = to_grid(grid);
    const vmb_config c = to_config(cfg);
    int64_t m = 0, b = 0;
    check(vmb_factorize(&g, &c, &m, &b));
    return {m, b};
}

// ---------------------------------------------------------------- host <-> device helpers
template <class MatT>
DeviceBuffer to_device(const MatT& m) {
    DeviceBuffer b((size_t)m.rows * m.cols * sizeof(float));
    if (b.size()) check_cuda(cudaMemcpy(b.get(), m.data.data(), b.size(), cudaMemcpyHostToDevice), "H2D");
    return b;
}
inline DeviceBuffer vec_to_device(const std::vector<float>& v) {
    DeviceBuffer b(v.size() * sizeof(float));
    if (b.size()) check_cuda(cudaMemcpy(b.get(), v.data(), b.size(), cudaMemcpyHostToDevice), "H2D");
    return b;
}
template <class MatT>
MatT mat_from_device(const DeviceBuffer& b, int64_t rows, int64_t cols) {
    MatT m(rows, cols);
    if (rows * cols > 0) check_cuda(cudaMemcpy(m.data.data(), b.get(), (size_t)rows * cols * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
    return m;
}
inline std::vector<float> vec_from_device(const DeviceBuffer& b, size_t n) {
    std::vector<float> v(n);
    if (n) check_cuda(cudaMemcpy(v.data(), b.get(), n * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
    return v;
}

// video.cpp:36-59 (per batch*head unit).  CostT: the caller's CostReport type.
template <class CostT, class GridT, class CfgT>
CostT flops_estimate(const GridT& grid, const CfgT& cfg, int64_t d) {
    const vmb_grid g = to_grid(grid);
    const vmb_config c = to_config(cfg);
    CostT r{};
    uint64_t mf = 0, ff = 0, rf = 0;
    check(vmb_flops_estimate(&g, &c, d, &r.sparsity, &r.sparsity_approx, &mf, &ff, &rf, &r.reduction_ratio));
    r.monarch_flops = mf;
    r.full_attn_flops = ff;
    r.recompute_flops = rf;
    return r;
}

// oracle.hpp:36-72: softmax(Q K^T [/ sqrt d]) V on the device (fp32 parity mode).
template <class MatT>
MatT dense_forward(const MatT& q, const MatT& k, const MatT& v, bool scale) {
    check_dim(q.cols == k.cols && k.cols == v.cols, "Q, K, V must share head dim");
    check_dim(k.rows == v.rows, "K and V must share row count");
    check_dim(k.rows >= 1, "attention over empty keys");
    DeviceBuffer dq = to_device(q), dk = to_device(k), dv = to_device(v), dout((size_t)q.rows * q.cols * sizeof(float));
    const float qs = scale ? (float)(1.0 / std::sqrt((double)q.cols)) : 1.f;
    check(vmb_flash_entropy_fwd(1, q.rows, k.rows, q.cols, VMB_F32, dq.get(), dk.get(), dv.get(), qs, dout.get(), nullptr,
                                nullptr, nullptr));
    check_cuda(cudaDeviceSynchronize(), "dense_forward");
    return mat_from_device<MatT>(dout, q.rows, q.cols);
}

// flash_entropy.hpp:85-139.  ResultT: the caller's FlashFwdResult<float> {output, lse, entropy}.
template <class ResultT, class MatT, class TileT>
ResultT flash_entropy_fwd(const MatT& q, const MatT& k, const MatT& v, const TileT& tiles) {
    check_dim(q.cols == k.cols && k.cols == v.cols, "Q, K, V must share head dim");
    check_dim(k.rows == v.rows, "K and V must share row count");
    if (k.rows < 1) throw std::domain_error("domain error: attention over empty keys");
    check_dim(tiles.b_r >= 1 && tiles.b_c >= 1, "tile sizes must be >= 1");
    DeviceBuffer dq = to_device(q), dk = to_device(k), dv = to_device(v), dout((size_t)q.rows * q.cols * sizeof(float)),
                 dl((size_t)q.rows * sizeof(float)), de((size_t)q.rows * sizeof(float));
    check(vmb_flash_entropy_fwd(1, q.rows, k.rows, q.cols, VMB_F32, dq.get(), dk.get(), dv.get(), 1.f, dout.get(),
                                (float*)dl.get(), (float*)de.get(), nullptr));
    check_cuda(cudaDeviceSynchronize(), "flash_entropy_fwd");
    ResultT r;
    r.output = mat_from_device<MatT>(dout, q.rows, q.cols);
    r.lse = vec_from_device(dl, (size_t)q.rows);
    r.entropy = vec_from_device(de, (size_t)q.rows);
    return r;
}

// flash_entropy.hpp:146-221.  ResultT: the caller's FlashBwdResult<float> {dq, dk, dv}.
template <class ResultT, class MatT, class TileT>
ResultT flash_entropy_bwd(const MatT& q, const MatT& k, const MatT& v, const MatT& o, const MatT& dout,
                          const std::vector<float>& lse, const std::vector<float>& entropy,
                          const std::vector<float>& dentropy, bool entropy_grad, const TileT& tiles) {
    const int64_t nq = q.rows, nk = k.rows, d = q.cols;
    check_dim(k.cols == d && v.cols == d && o.cols == d && dout.cols == d, "all operands must share head dim");
    check_dim(v.rows == nk, "K and V must share row count");
    check_dim(o.rows == nq && dout.rows == nq, "O and dO must have N_q rows");
    check_dim((int64_t)lse.size() == nq, "lse length must equal N_q");
    check_dim(entropy.empty() || (int64_t)entropy.size() == nq, "entropy length must equal N_q");
    check_dim(dentropy.empty() || (int64_t)dentropy.size() == nq, "dH length must equal N_q");
    if (entropy_grad) check_dim(!entropy.empty() && !dentropy.empty(), "entropy_grad requires entropy and dH inputs");
    if (nk < 1) throw std::domain_error("domain error: attention over empty keys");
    check_dim(tiles.b_r >= 1 && tiles.b_c >= 1, "tile sizes must be >= 1");
    DeviceBuffer bq = to_device(q), bk = to_device(k), bv = to_device(v), bo = to_device(o), bg = to_device(dout),
                 bl = vec_to_device(lse), be = vec_to_device(entropy), bd = vec_to_device(dentropy),
                 gq((size_t)nq * d * sizeof(float)), gk((size_t)nk * d * sizeof(float)), gv((size_t)nk * d * sizeof(float));
    check(vmb_flash_entropy_bwd(1, nq, nk, d, VMB_F32, bq.get(), bk.get(), bv.get(), bo.get(), bg.get(), (const float*)bl.get(),
                                entropy.empty() ? nullptr : (const float*)be.get(),
                                dentropy.empty() ? nullptr : (const float*)bd.get(), entropy_grad ? 1 : 0, gq.get(),
                                gk.get(), gv.get(), nullptr));
    check_cuda(cudaDeviceSynchronize(), "flash_entropy_bwd");
    ResultT r;
    r.dq = mat_from_device<MatT>(gq, nq, d);
    r.dk = mat_from_device<MatT>(gk, nk, d);
    r.dv = mat_from_device<MatT>(gv, nk, d);
    return r;
}

// ---------------------------------------------------------------- the operator (video.hpp:84-150)
// Compute precision of the façade.  fp32 (default) is the parity mode: <= 1e-4 of the
// reference, on CUDA cores.  bf16 rounds the float inputs to bf16 on the host and runs the
// tcgen05 path (the performance path, <= 2e-2 of the reference; ~200-350x faster than fp32 at
// the Wan shapes), returning float outputs.  An extra trailing argument, so calls written
// for the reference signature are unchanged.
enum class Precision { fp32, bf16 };

namespace detail {
inline uint16_t f32_to_bf16(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    if ((x & 0x7F800000u) == 0x7F800000u) return (uint16_t)((x >> 16) | ((x & 0xFFFFu) ? 0x40u : 0u));  // inf / NaN
    return (uint16_t)((x + 0x7FFFu + ((x >> 16) & 1u)) >> 16);  // round to nearest even
}
inline float bf16_to_f32(uint16_t h) {
    const uint32_t x = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &x, 4);
    return f;
}
}  // namespace detail

template <class MatT, class GridT, class CfgT, class FactorsVec = std::vector<int>>
std::vector<MatT> vmonarch_attention(std::span<const MatT> qs, std::span<const MatT> ks, std::span<const MatT> vs,
                                     const GridT& grid, const CfgT& cfg, int threads = 1,
                                     FactorsVec* factors_out = nullptr, Precision prec = Precision::fp32) {
    (void)threads;
    using T = typename std::remove_cv_t<std::remove_reference_t<decltype(qs[0].data[0])>>;
    static_assert(std::is_same_v<T, float>, "the drop-in façade takes the reference's T = float matrices");
    const bool bf16 = prec == Precision::bf16;
    const vmb_dtype dt = bf16 ? VMB_BF16 : VMB_F32;
    const size_t es = bf16 ? 2 : 4;
    const int64_t units = (int64_t)grid.heads * (int64_t)grid.batch;
    check_dim((int64_t)qs.size() == units && (int64_t)ks.size() == units && (int64_t)vs.size() == units,
              "expected one Q/K/V matrix per batch*head unit");
    const int64_t n = (int64_t)grid.t_frames * grid.h * grid.w, d = grid.head_dim;
    for (int64_t u = 0; u < units; ++u) {
        check_dim(qs[u].rows == n && ks[u].rows == n && vs[u].rows == n, "each head must have T*h*w rows");
        check_dim(qs[u].cols == d && ks[u].cols == d && vs[u].cols == d, "each head must have head_dim columns");
    }
    const vmb_grid g = to_grid(grid);
    const vmb_config c = to_config(cfg);
    int64_t m = 0, b = 0;
    check(vmb_factorize(&g, &c, &m, &b));

    const size_t unit_elems = (size_t)n * d, unit_bytes = unit_elems * es;
    DeviceBuffer dq(unit_bytes * units), dk(unit_bytes * units), dv(unit_bytes * units), dout(unit_bytes * units);
    std::vector<uint16_t> stage(bf16 ? unit_elems : 0);
    auto upload = [&](const MatT& m, void* dst, const char* what) {
        const void* src = m.data.data();
        if (bf16) {
            for (size_t x = 0; x < unit_elems; ++x) stage[x] = detail::f32_to_bf16(m.data[x]);
            src = stage.data();
        }
        check_cuda(cudaMemcpy(dst, src, unit_bytes, cudaMemcpyHostToDevice), what);
    };
    for (int64_t u = 0; u < units; ++u) {
        upload(qs[u], (char*)dq.get() + u * unit_bytes, "H2D q");
        upload(ks[u], (char*)dk.get() + u * unit_bytes, "H2D k");
        upload(vs[u], (char*)dv.get() + u * unit_bytes, "H2D v");
    }
    const size_t ws_bytes = vmb_workspace_size(&g, &c, dt);
    if (ws_bytes == 0) raise_status(VMB_ERR_DIM);
    DeviceBuffer ws(ws_bytes);
    check(vmb_vmonarch_fwd(&g, &c, dt, dq.get(), dk.get(), dv.get(), dout.get(), nullptr, nullptr, ws.get(), ws_bytes,
                           nullptr));
    check(vmb_workspace_status(ws.get(), nullptr));  // device-raised domain errors (monarch.hpp:44, 78)

    std::vector<MatT> out;
    out.reserve((size_t)units);
    for (int64_t u = 0; u < units; ++u) {
        out.emplace_back(n, d);
        void* dst = bf16 ? (void*)stage.data() : (void*)out.back().data.data();
        check_cuda(cudaMemcpy(dst, (char*)dout.get() + u * unit_bytes, unit_bytes, cudaMemcpyDeviceToHost),
                   "D2H out");
        if (bf16)
            for (size_t x = 0; x < unit_elems; ++x) out.back().data[x] = detail::bf16_to_f32(stage[x]);
    }
    if constexpr (!std::is_same_v<FactorsVec, std::vector<int>>) {
        if (factors_out) {
            // MonarchFactors (monarch.hpp:12-19): L (b, m, m), R (m, b, b) per unit
            DeviceBuffer dL((size_t)units * b * m * m * sizeof(float)), dR((size_t)units * m * b * b * sizeof(float));
            check(vmb_export_factors(&g, &c, dt, dq.get(), dk.get(), nullptr, ws.get(), (float*)dL.get(),
                                     (float*)dR.get(), nullptr));
            check_cuda(cudaDeviceSynchronize(), "factor export");
            factors_out->resize((size_t)units);
            for (int64_t u = 0; u < units; ++u) {
                auto& f = (*factors_out)[(size_t)u];
                f.L = decltype(f.L)(b, m, m);
                f.R = decltype(f.R)(m, b, b);
                check_cuda(cudaMemcpy(f.L.data.data(), (float*)dL.get() + (size_t)u * b * m * m,
                                      (size_t)b * m * m * sizeof(float), cudaMemcpyDeviceToHost),
                           "D2H L");
                check_cuda(cudaMemcpy(f.R.data.data(), (float*)dR.get() + (size_t)u * m * b * b,
                                      (size_t)m * b * b * sizeof(float), cudaMemcpyDeviceToHost),
                           "D2H R");
            }
        }
    }
    return out;
}

// monarch.hpp:155-193 for one (m*b, d) problem: the grid path with T = m, h*w = b and no
// first-frame recompute.  ResultT: the caller's MonarchResult<float> {output, factors{L, R}};
// CfgT: MonarchConfig {m, b, iters, clamp_min, clamp_enabled}.
template <class ResultT, class MatT, class CfgT>
ResultT monarch_attention(const MatT& q, const MatT& k, const MatT& v, const CfgT& cfg) {
    const int64_t n = (int64_t)cfg.m * cfg.b;
    check_dim(q.rows == n && k.rows == n && v.rows == n, "Q, K, V must have m*b rows");
    check_dim(q.cols == k.cols && k.cols == v.cols, "Q, K, V must share head dim");
    check_dim(q.cols >= 1, "head dim must be >= 1");
    struct G { int64_t t_frames, h, w, head_dim, heads, batch; } g{cfg.m, 1, cfg.b, q.cols, 1, 1};
    struct C {
        int64_t iters;
        double clamp_min;
        bool clamp_enabled, recompute_first_frame;
        const std::pair<int64_t, int64_t>* override_m_b;
    } c{cfg.iters, cfg.clamp_min, cfg.clamp_enabled, false, nullptr};
    std::vector<std::remove_reference_t<decltype(std::declval<ResultT&>().factors)>> f;
    std::vector<MatT> qs{q}, ks{k}, vs{v};
    auto out = vmonarch_attention(std::span<const MatT>(qs), std::span<const MatT>(ks), std::span<const MatT>(vs), g, c,
                                  1, &f);
    ResultT r;
    r.output = std::move(out[0]);
    r.factors = std::move(f[0]);
    return r;
}

}  // namespace vmonarch_b200
