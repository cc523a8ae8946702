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
// Host buffers stream through the device in chunks of batch*head units (pinned staging,
// H2D / forward / D2H overlapped on three CUDA streams).  The forward runs in the fp32 parity
// mode (CUDA cores, the reference precision policy; <= 1e-4 vs the reference) for T = float,
// in the f64 mode for T = double (agreement to round-off, as the reference's double tests
// need), or with the trailing Precision::bf16 on the tcgen05 path.  Device-resident bf16
// callers use the C ABI directly (vmb_vmonarch_fwd with VMB_BF16).  Errors are thrown as
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
    static_assert(std::is_same_v<std::remove_cv_t<std::remove_reference_t<decltype(m.data[0])>>, float>,
                  "flash_entropy_fwd / _bwd / dense_forward take T = float matrices");
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

namespace detail {
// Pinned host staging and device buffers of the pipelined host path, kept per thread and
// grown on demand (page-locking gigabytes per call would cost more than the copies).
struct PinnedBuffer {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t n) {
        if (n <= bytes) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        check_cuda(cudaHostAlloc(&p, n, cudaHostAllocDefault), "cudaHostAlloc");
        bytes = n;
    }
    ~PinnedBuffer() {
        if (p) cudaFreeHost(p);
    }
};
struct HostPipeline {
    PinnedBuffer in[2], out[2];
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t h2d_done[2] = {}, comp_done[2] = {}, d2h_done[2] = {};
    int device = -1;
    void init() {
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        if (device == dev) return;
        release();
        device = dev;
        check_cuda(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking), "stream");
        check_cuda(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking), "stream");
        check_cuda(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < 2; ++i) {
            check_cuda(cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming), "event");
            check_cuda(cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming), "event");
            check_cuda(cudaEventCreateWithFlags(&d2h_done[i], cudaEventDisableTiming), "event");
        }
    }
    void release() {
        if (device < 0) return;
        cudaStreamDestroy(h2d);
        cudaStreamDestroy(comp);
        cudaStreamDestroy(d2h);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(h2d_done[i]);
            cudaEventDestroy(comp_done[i]);
            cudaEventDestroy(d2h_done[i]);
        }
        device = -1;
    }
    ~HostPipeline() { release(); }
};
inline HostPipeline& host_pipeline() {
    static thread_local HostPipeline p;
    p.init();
    return p;
}
}  // namespace detail

// video.hpp:84-150 for host matrices.  T = float runs the fp32 parity mode (Precision::fp32,
// <= 1e-4 of the reference) or, with Precision::bf16, the tcgen05 path; T = double runs the f64
// mode (the reference's T = double, CUDA cores, agreement to round-off).
//
// Host path: batch*head units are independent (video.hpp:115-148; per-unit results are
// bitwise independent of how units are grouped), so they stream through the device in
// chunks of `chunk_units` on three CUDA streams -- host staging into pinned memory, H2D,
// forward and D2H of consecutive chunks overlap (double-buffered pinned and device buffers).
// With factors_out the call runs as one chunk (the factor export reads the forward's state).
template <class MatT, class GridT, class CfgT, class FactorsVec = std::vector<int>>
std::vector<MatT> vmonarch_attention(std::span<const MatT> qs, std::span<const MatT> ks, std::span<const MatT> vs,
                                     const GridT& grid, const CfgT& cfg, int threads = 1,
                                     FactorsVec* factors_out = nullptr, Precision prec = Precision::fp32,
                                     int64_t chunk_units = 0) {
    (void)threads;
    using T = typename std::remove_cv_t<std::remove_reference_t<decltype(qs[0].data[0])>>;
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>,
                  "the drop-in façade takes the reference's T = float or T = double matrices");
    constexpr bool f64 = std::is_same_v<T, double>;
    const bool bf16 = prec == Precision::bf16;
    const vmb_dtype dt = bf16 ? VMB_BF16 : (f64 ? VMB_F64 : VMB_F32);
    const size_t es = bf16 ? 2 : sizeof(T);
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
    std::vector<MatT> out;
    if (units == 0) return out;

    const bool want_factors = [&] {
        if constexpr (!std::is_same_v<FactorsVec, std::vector<int>>) return factors_out != nullptr;
        return false;
    }();
    const size_t unit_elems = (size_t)n * d, unit_bytes = unit_elems * es;
    // default: ~8 chunks (the pipeline depth that hides the copies), at most 512 MB per tensor chunk
    int64_t chunk = chunk_units > 0 ? chunk_units : std::max<int64_t>(1, (units + 7) / 8);
    chunk = std::min<int64_t>(chunk, std::max<int64_t>(1, (int64_t)((size_t(512) << 20) / std::max<size_t>(unit_bytes, 1))));
    if (want_factors) chunk = units;
    chunk = std::min(chunk, units);
    const int64_t n_chunks = (units + chunk - 1) / chunk;

    vmb_grid gc = g;  // a chunk: `cu` contiguous units, unit-major
    gc.heads = chunk;
    gc.batch = 1;
    const size_t ws_bytes = vmb_workspace_size(&gc, &c, dt);
    if (ws_bytes == 0) raise_status(VMB_ERR_DIM);
    const size_t chunk_bytes = (size_t)chunk * unit_bytes;
    DeviceBuffer dev_in[2] = {DeviceBuffer(3 * chunk_bytes), DeviceBuffer(n_chunks > 1 ? 3 * chunk_bytes : 0)};
    DeviceBuffer dev_out[2] = {DeviceBuffer(chunk_bytes), DeviceBuffer(n_chunks > 1 ? chunk_bytes : 0)};
    DeviceBuffer ws[2] = {DeviceBuffer(ws_bytes), DeviceBuffer(n_chunks > 1 ? ws_bytes : 0)};
    // the device status word of each chunk's forward (vmb.h: workspace offset 0), parked in a
    // 256-byte status-only "workspace" so vmb_workspace_status can interpret it
    DeviceBuffer status(2 * 256);
    detail::HostPipeline& hp = detail::host_pipeline();
    for (int s2 = 0; s2 < 2; ++s2) {
        hp.in[s2].reserve(3 * chunk_bytes);
        hp.out[s2].reserve(chunk_bytes);
    }
    out.reserve((size_t)units);
    for (int64_t u = 0; u < units; ++u) out.emplace_back(n, d);

    auto stage_in = [&](const MatT& mtx, uint8_t* dst) {
        if (bf16) {
            uint16_t* h = reinterpret_cast<uint16_t*>(dst);
            for (size_t x = 0; x < unit_elems; ++x) h[x] = detail::f32_to_bf16((float)mtx.data[x]);
        } else {
            std::memcpy(dst, mtx.data.data(), unit_bytes);
        }
    };
    auto unstage_out = [&](const uint8_t* src, MatT& mtx) {
        if (bf16) {
            const uint16_t* h = reinterpret_cast<const uint16_t*>(src);
            for (size_t x = 0; x < unit_elems; ++x) mtx.data[x] = (T)detail::bf16_to_f32(h[x]);
        } else {
            std::memcpy(mtx.data.data(), src, unit_bytes);
        }
    };
    auto drain = [&](int64_t ci) {
        const int sl = (int)(ci % 2);
        const int64_t u0 = ci * chunk, cu = std::min(chunk, units - u0);
        check_cuda(cudaEventSynchronize(hp.d2h_done[sl]), "D2H");
        check(vmb_workspace_status((uint8_t*)status.get() + sl * 256, hp.d2h));  // monarch.hpp:44, 78
        const uint8_t* src = static_cast<const uint8_t*>(hp.out[sl].p);
        for (int64_t u = 0; u < cu; ++u) unstage_out(src + u * unit_bytes, out[(size_t)(u0 + u)]);
    };
    for (int64_t ci = 0; ci < n_chunks; ++ci) {
        const int sl = (int)(ci % 2);
        const int64_t u0 = ci * chunk, cu = std::min(chunk, units - u0);
        // slot sl's pinned input staging is free once chunk ci-2's H2D has landed
        if (ci >= 2) check_cuda(cudaEventSynchronize(hp.h2d_done[sl]), "H2D");
        uint8_t* hin = static_cast<uint8_t*>(hp.in[sl].p);
        for (int64_t u = 0; u < cu; ++u) {
            stage_in(qs[u0 + u], hin + u * unit_bytes);
            stage_in(ks[u0 + u], hin + chunk_bytes + u * unit_bytes);
            stage_in(vs[u0 + u], hin + 2 * chunk_bytes + u * unit_bytes);
        }
        uint8_t* din = static_cast<uint8_t*>(dev_in[sl].get());
        if (ci >= 2) check_cuda(cudaStreamWaitEvent(hp.h2d, hp.comp_done[sl], 0), "wait");  // device inputs reusable
        for (int t = 0; t < 3; ++t)
            check_cuda(cudaMemcpyAsync(din + t * chunk_bytes, hin + t * chunk_bytes, (size_t)cu * unit_bytes,
                                       cudaMemcpyHostToDevice, hp.h2d), "H2D");
        check_cuda(cudaEventRecord(hp.h2d_done[sl], hp.h2d), "event");
        check_cuda(cudaStreamWaitEvent(hp.comp, hp.h2d_done[sl], 0), "wait");
        if (ci >= 2) check_cuda(cudaStreamWaitEvent(hp.comp, hp.d2h_done[sl], 0), "wait");  // device output reusable
        vmb_grid gci = gc;
        gci.heads = cu;
        check(vmb_vmonarch_fwd(&gci, &c, dt, din, din + chunk_bytes, din + 2 * chunk_bytes, dev_out[sl].get(),
                               nullptr, nullptr, ws[sl].get(), ws_bytes, hp.comp));
        check_cuda(cudaMemcpyAsync((uint8_t*)status.get() + sl * 256, ws[sl].get(), sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, hp.comp), "status");
        check_cuda(cudaEventRecord(hp.comp_done[sl], hp.comp), "event");
        // the host drains chunk ci-1 (freeing pinned output slot 1-sl) while chunk ci computes
        if (ci >= 1) drain(ci - 1);
        check_cuda(cudaStreamWaitEvent(hp.d2h, hp.comp_done[sl], 0), "wait");
        check_cuda(cudaMemcpyAsync(hp.out[sl].p, dev_out[sl].get(), (size_t)cu * unit_bytes, cudaMemcpyDeviceToHost,
                                   hp.d2h), "D2H");
        check_cuda(cudaEventRecord(hp.d2h_done[sl], hp.d2h), "event");
    }
    drain(n_chunks - 1);

    if constexpr (!std::is_same_v<FactorsVec, std::vector<int>>) {
        if (factors_out) {
            // MonarchFactors (monarch.hpp:12-19): L (b, m, m), R (m, b, b) per unit, in the
            // state type of the mode (T = double: double)
            using S = std::conditional_t<f64, double, float>;
            DeviceBuffer dL((size_t)units * b * m * m * sizeof(S)), dR((size_t)units * m * b * b * sizeof(S));
            uint8_t* din = static_cast<uint8_t*>(dev_in[0].get());
            check(vmb_export_factors(&g, &c, dt, din, din + chunk_bytes, nullptr, ws[0].get(), (float*)dL.get(),
                                     (float*)dR.get(), hp.comp));
            check_cuda(cudaStreamSynchronize(hp.comp), "factor export");
            factors_out->resize((size_t)units);
            std::vector<S> hL((size_t)b * m * m), hR((size_t)m * b * b);
            for (int64_t u = 0; u < units; ++u) {
                auto& f = (*factors_out)[(size_t)u];
                f.L = decltype(f.L)(b, m, m);
                f.R = decltype(f.R)(m, b, b);
                check_cuda(cudaMemcpy(hL.data(), (S*)dL.get() + (size_t)u * b * m * m, hL.size() * sizeof(S),
                                      cudaMemcpyDeviceToHost), "D2H L");
                check_cuda(cudaMemcpy(hR.data(), (S*)dR.get() + (size_t)u * m * b * b, hR.size() * sizeof(S),
                                      cudaMemcpyDeviceToHost), "D2H R");
                for (size_t x = 0; x < hL.size(); ++x) f.L.data[x] = hL[x];
                for (size_t x = 0; x < hR.size(); ++x) f.R.data[x] = hR[x];
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
