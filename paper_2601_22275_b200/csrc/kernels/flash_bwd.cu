// flash_bwd.cu — backward of the online-entropy attention (flash_entropy.hpp:146-221) on CUDA
// cores: the paper's fine-tuning path (Alg. 2), SURVEY §8(f) row 2.
//
// Reference semantics, per unit (Q pre-scaled by the caller, lse / H from the matching forward):
//   P  = exp(Q K^T - lse)            D_i = sum_x O[i,x] dO[i,x]   (double accumulation)
//   dV = P^T dO                      dP  = dO V^T
//   dS = P (dP - D)   [- dH P (S - lse + H)  with entropy_grad]
//   dQ = dS K                        dK  = dS^T Q
// Three kernels: D (one warp per query row), dQ (one warp per query row, looping over keys)
// and dK/dV (one warp per key row, looping over queries).  A lane owns d/32 head-dim elements;
// dot products are warp-shuffle reductions.  fp32 arithmetic for fp32 and bf16 storage.
#include <cuda_bf16.h>

#include "../internal.hpp"

namespace vmb {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kMaxDPL = 8;  // head-dim elements per lane (d <= 256)

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
    return static_cast<float>(*p);
}
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st(T* p, float v) {
    *p = static_cast<T>(v);
}
template <>
__device__ __forceinline__ void st<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

struct BwdArgs {
    const void *q, *k, *v, *o, *dout;
    const float *lse, *ent, *dent;
    float* dvec;  // (U, nq) scratch
    void *dq, *dk, *dv;
    int64_t U, nq, nk, d;
    int32_t entropy_grad;
};

template <typename T>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) bwd_dvec_kernel(BwdArgs a) {
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= a.U * a.nq) return;
    const T* o = static_cast<const T*>(a.o) + row * a.d;
    const T* g = static_cast<const T*>(a.dout) + row * a.d;
    double acc = 0.0;
    for (int64_t x = lane; x < a.d; x += 32) acc += (double)ld(o + x) * (double)ld(g + x);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) a.dvec[row] = (float)acc;
}

// dS for one (query i, key l) pair given this lane's slices
__device__ __forceinline__ float dscore(float s, float dp, float lse, float di, float dh, float lh, bool eg) {
    const float p = expf(s - lse);
    float ds = p * (dp - di);
    if (eg) ds -= dh * p * (s + lh);
    return ds;
}

template <typename T>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) bwd_dq_kernel(BwdArgs a) {
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= a.U * a.nq) return;
    const int64_t u = row / a.nq;
    const int dpl = (int)((a.d + 31) / 32);
    float q[kMaxDPL], g[kMaxDPL], acc[kMaxDPL];
    const T* qr = static_cast<const T*>(a.q) + row * a.d;
    const T* gr = static_cast<const T*>(a.dout) + row * a.d;
#pragma unroll
    for (int e = 0; e < kMaxDPL; ++e) {
        const int64_t x = lane + 32 * e;
        q[e] = (e < dpl && x < a.d) ? ld(qr + x) : 0.f;
        g[e] = (e < dpl && x < a.d) ? ld(gr + x) : 0.f;
        acc[e] = 0.f;
    }
    const float lse = a.lse[row], di = a.dvec[row];
    const bool eg = a.entropy_grad != 0;
    const float dh = eg ? a.dent[row] : 0.f, lh = eg ? a.ent[row] - a.lse[row] : 0.f;
    const T* kb = static_cast<const T*>(a.k) + u * a.nk * a.d;
    const T* vb = static_cast<const T*>(a.v) + u * a.nk * a.d;
    for (int64_t l = 0; l < a.nk; ++l) {
        float s = 0.f, dp = 0.f, kk[kMaxDPL];
#pragma unroll
        for (int e = 0; e < kMaxDPL; ++e) {
            const int64_t x = lane + 32 * e;
            const bool in = e < dpl && x < a.d;
            kk[e] = in ? ld(kb + l * a.d + x) : 0.f;
            s += q[e] * kk[e];
            dp += g[e] * (in ? ld(vb + l * a.d + x) : 0.f);
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float ds = dscore(s, dp, lse, di, dh, lh, eg);
#pragma unroll
        for (int e = 0; e < kMaxDPL; ++e) acc[e] += ds * kk[e];
    }
    T* out = static_cast<T*>(a.dq) + row * a.d;
#pragma unroll
    for (int e = 0; e < kMaxDPL; ++e) {
        const int64_t x = lane + 32 * e;
        if (e < dpl && x < a.d) st(out + x, acc[e]);
    }
}

template <typename T>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) bwd_dkv_kernel(BwdArgs a) {
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);  // key row
    const int lane = threadIdx.x & 31;
    if (row >= a.U * a.nk) return;
    const int64_t u = row / a.nk;
    const int dpl = (int)((a.d + 31) / 32);
    float k[kMaxDPL], v[kMaxDPL], dk[kMaxDPL], dv[kMaxDPL];
    const T* kr = static_cast<const T*>(a.k) + row * a.d;
    const T* vr = static_cast<const T*>(a.v) + row * a.d;
#pragma unroll
    for (int e = 0; e < kMaxDPL; ++e) {
        const int64_t x = lane + 32 * e;
        k[e] = (e < dpl && x < a.d) ? ld(kr + x) : 0.f;
        v[e] = (e < dpl && x < a.d) ? ld(vr + x) : 0.f;
        dk[e] = dv[e] = 0.f;
    }
    const bool eg = a.entropy_grad != 0;
    const T* qb = static_cast<const T*>(a.q) + u * a.nq * a.d;
    const T* gb = static_cast<const T*>(a.dout) + u * a.nq * a.d;
    for (int64_t i = 0; i < a.nq; ++i) {
        const int64_t qi = u * a.nq + i;
        float s = 0.f, dp = 0.f, qq[kMaxDPL], gg[kMaxDPL];
#pragma unroll
        for (int e = 0; e < kMaxDPL; ++e) {
            const int64_t x = lane + 32 * e;
            const bool in = e < dpl && x < a.d;
            qq[e] = in ? ld(qb + i * a.d + x) : 0.f;
            gg[e] = in ? ld(gb + i * a.d + x) : 0.f;
            s += qq[e] * k[e];
            dp += gg[e] * v[e];
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float lse = a.lse[qi];
        const float p = expf(s - lse);
        const float ds = dscore(s, dp, lse, a.dvec[qi], eg ? a.dent[qi] : 0.f, eg ? a.ent[qi] - lse : 0.f, eg);
#pragma unroll
        for (int e = 0; e < kMaxDPL; ++e) {
            dv[e] += p * gg[e];
            dk[e] += ds * qq[e];
        }
    }
    T* okr = static_cast<T*>(a.dk) + row * a.d;
    T* ovr = static_cast<T*>(a.dv) + row * a.d;
#pragma unroll
    for (int e = 0; e < kMaxDPL; ++e) {
        const int64_t x = lane + 32 * e;
        if (e < dpl && x < a.d) {
            st(okr + x, dk[e]);
            st(ovr + x, dv[e]);
        }
    }
}

template <typename T>
void launch_all(const BwdArgs& a, cudaStream_t s) {
    const int threads = 32 * kWarpsPerBlock;
    const int64_t qrows = a.U * a.nq, krows = a.U * a.nk;
    ProfScope ps(kKSimt, s);
    if (qrows > 0) {
        bwd_dvec_kernel<T><<<(unsigned)((qrows + kWarpsPerBlock - 1) / kWarpsPerBlock), threads, 0, s>>>(a);
        bwd_dq_kernel<T><<<(unsigned)((qrows + kWarpsPerBlock - 1) / kWarpsPerBlock), threads, 0, s>>>(a);
        count_launch(2);
    }
    if (krows > 0) {
        bwd_dkv_kernel<T><<<(unsigned)((krows + kWarpsPerBlock - 1) / kWarpsPerBlock), threads, 0, s>>>(a);
        count_launch();
    }
    check_launch("flash_entropy_bwd");
}

}  // namespace

void flash_bwd_launch(int64_t U, int64_t nq, int64_t nk, int64_t d, bool bf16, const void* q, const void* k,
                      const void* v, const void* o, const void* dout, const float* lse, const float* ent,
                      const float* dent, int entropy_grad, float* dvec, void* dq, void* dk, void* dv,
                      cudaStream_t s) {
    VMB_REQUIRE_DIM(d >= 1 && d <= 32 * kMaxDPL, "flash backward supports head dim <= 256");
    BwdArgs a{q, k, v, o, dout, lse, ent, dent, dvec, dq, dk, dv, U, nq, nk, d, entropy_grad};
    if (bf16) launch_all<__nv_bfloat16>(a, s);
    else launch_all<float>(a, s);
}

}  // namespace vmb
