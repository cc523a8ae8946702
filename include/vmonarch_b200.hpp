// vmonarch_b200.hpp — C++ drop-in façade over the libvmb C ABI (include/vmb.h).
//
// Same call shape, argument meaning and exception types as the reference operator
// (/root/reference/proj/include/vmonarch/video.hpp:84-150, check.hpp:10-20):
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

#include <cstdint>
#include <cstring>
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

// ---------------------------------------------------------------- the operator (video.hpp:84-150)
template <class MatT, class GridT, class CfgT, class FactorsVec = std::vector<int>>
std::vector<MatT> vmonarch_attention(std::span<const MatT> qs, std::span<const MatT> ks, std::span<const MatT> vs,
                                     const GridT& grid, const CfgT& cfg, int threads = 1,
                                     FactorsVec* factors_out = nullptr) {
    (void)threads;
    using T = typename std::remove_cv_t<std::remove_reference_t<decltype(qs[0].data[0])>>;
    static_assert(std::is_same_v<T, float>, "the drop-in façade runs the fp32 parity mode (T = float)");
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

    const size_t unit_bytes = (size_t)n * d * sizeof(float);
    DeviceBuffer dq(unit_bytes * units), dk(unit_bytes * units), dv(unit_bytes * units), dout(unit_bytes * units);
    for (int64_t u = 0; u < units; ++u) {
        check_cuda(cudaMemcpy((char*)dq.get() + u * unit_bytes, qs[u].data.data(), unit_bytes, cudaMemcpyHostToDevice),
                   "H2D q");
        check_cuda(cudaMemcpy((char*)dk.get() + u * unit_bytes, ks[u].data.data(), unit_bytes, cudaMemcpyHostToDevice),
                   "H2D k");
        check_cuda(cudaMemcpy((char*)dv.get() + u * unit_bytes, vs[u].data.data(), unit_bytes, cudaMemcpyHostToDevice),
                   "H2D v");
    }
    const size_t ws_bytes = vmb_workspace_size(&g, &c, VMB_F32);
    if (ws_bytes == 0) raise_status(VMB_ERR_DIM);
    DeviceBuffer ws(ws_bytes);
    check(vmb_vmonarch_fwd(&g, &c, VMB_F32, dq.get(), dk.get(), dv.get(), dout.get(), nullptr, nullptr, ws.get(),
                           ws_bytes, nullptr));
    check(vmb_workspace_status(ws.get(), nullptr));  // device-raised domain errors (monarch.hpp:44, 78)

    std::vector<MatT> out;
    out.reserve((size_t)units);
    for (int64_t u = 0; u < units; ++u) {
        out.emplace_back(n, d);
        check_cuda(cudaMemcpy(out.back().data.data(), (char*)dout.get() + u * unit_bytes, unit_bytes,
                              cudaMemcpyDeviceToHost),
                   "D2H out");
    }
    if constexpr (!std::is_same_v<FactorsVec, std::vector<int>>) {
        if (factors_out) {
            // MonarchFactors (monarch.hpp:12-19): L (b, m, m), R (m, b, b) per unit
            DeviceBuffer dL((size_t)units * b * m * m * sizeof(float)), dR((size_t)units * m * b * b * sizeof(float));
            check(vmb_export_factors(&g, &c, VMB_F32, dq.get(), dk.get(), nullptr, ws.get(), (float*)dL.get(),
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

}  // namespace vmonarch_b200
