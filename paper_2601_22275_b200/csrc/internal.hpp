// internal.hpp — host-side declarations shared by the libvmb translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/vmb.h"

namespace vmb {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
    vmb_status status;
    std::string msg;
};
#define VMB_CHECK_CUDA(expr)                                                                    \
    do {                                                                                        \
        cudaError_t e__ = (expr);                                                               \
        if (e__ != cudaSuccess)                                                                 \
            throw ::vmb::Error{VMB_ERR_CUDA, std::string("cuda error: ") + #expr + ": " +       \
                                                 cudaGetErrorString(e__)};                      \
    } while (0)
#define VMB_REQUIRE_DIM(cond, msg)                                                              \
    do {                                                                                        \
        if (!(cond)) throw ::vmb::Error{VMB_ERR_DIM, std::string("dimension error: ") + (msg)}; \
    } while (0)
#define VMB_REQUIRE_DOMAIN(cond, msg)                                                           \
    do {                                                                                        \
        if (!(cond)) throw ::vmb::Error{VMB_ERR_DOMAIN, std::string("domain error: ") + (msg)}; \
    } while (0)

// Per-call scratch from the device's default stream-ordered pool.  The pool's release
// threshold is raised once per device, so freed scratch stays mapped for the next call instead
// of being returned at every synchronisation (which made each call pay for the mapping again).
void scratch_alloc(void** p, size_t bytes, cudaStream_t s);

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Optional per-kernel CUDA-event timing (vmb_profile_enable): a scope records an event
// pair on the launching stream around one kernel launch; vmb_profile_read sums them.
enum KernelId : int {
    kKRstep = 0,      // R half-step (fa2)
    kKRstepY = 1,     // last R half-step with y = R V fused (fa4)
    kKAttn = 2,       // recompute / flash / dense attention (fa3)
    kKLstep = 3,      // lstep_tc ITER
    kKLfinal = 4,     // lstep_tc FINAL (apply)
    kKSimt = 5,       // CUDA-core kernels
    kKCombine = 6,    // split-KV combine
    kKNum = 7
};
struct ProfScope {
    ProfScope(int id, cudaStream_t s);
    ~ProfScope();
    int id;
    cudaStream_t s;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};
// Throws on a launch error of the kernel just enqueued.
void check_launch(const char* what);

// ---------------------------------------------------------------- views
// Row (u, a, c) of a [batch, head, a, c, d] view lives at element offset
//   (u / H) * sB + (u % H) * sH + a * sa + c * sc,  d contiguous.
struct View {
    const void* base = nullptr;
    int64_t sB = 0, sH = 0, sa = 0, sc = 0;
    int32_t H = 1;
};

// Device status word (first 16 bytes of every workspace).
enum : int32_t { kStatusOk = 0, kStatusNonFiniteQ = 1, kStatusClampDomain = 2 };

// ---------------------------------------------------------------- TMA maps
// bf16 5-D tiled map over `base` with dims (innermost first) and byte strides of
// dims 1..4; 128B swizzle, zero OOB fill.
CUtensorMap make_tmap_bf16_5d(const void* base, const uint64_t dims[5],
                              const uint64_t strides_bytes[4], const uint32_t box[5]);
bool tmap_supported();

// ---------------------------------------------------------------- SIMT kernels (any dtype)
// CUDA-core kernels (simt.cu).  State pointers (cR, cL, R, L, part_acc) hold the compute type:
// float for VMB_F32 / VMB_BF16, double for VMB_F64.
struct SimtRstepArgs {
    View A;            // query rows (u, k, i): aR or Q
    double qscale;     // multiplies the logits (rounded to the compute type in the kernel)
    const void* cR;    // (U, m, b) or nullptr (== 1)
    double clamp_min;
    int clamp_enabled;
    View K;            // key rows (u, k, l)
    View V;            // value rows (u, k, l)
    View Out;          // output rows (u, k, i)  (aL or y)
    void* cL;          // (U, b, m) or nullptr
    void* R;           // (U, m, b, b) or nullptr
    int64_t U, m, b, d;
    int32_t* status;
};
struct SimtLstepArgs {
    View Q;            // Qb rows (u, i, j)
    double qscale;
    View aL;           // rows (u, i, k)
    const void* cL;    // (U, b, m)
    View aR;           // ITER: output rows (u, k, i)
    void* cR;          // ITER: (U, m, b)
    View Y;            // FINAL: rows (u, k, i)
    View O;            // FINAL: output rows (u, j, i)
    int32_t skip_j0;   // FINAL: rows j == 0 are produced elsewhere (recompute)
    void* L;           // (U, b, m, m) or nullptr
    int32_t final_mode;
    int64_t U, m, b, d;
};
struct SimtFlashArgs {
    View Q;            // rows (u, 0, r), r < nq
    double qscale;
    View K, V;         // rows (u, 0, l), l < nk
    View O;            // rows (u, 0, r)
    float* lse;        // (U, nq) or nullptr (VMB_F32 / VMB_BF16 only)
    float* ent;        // (U, nq) or nullptr (VMB_F32 / VMB_BF16 only)
    int64_t U, nq, nk, d;
    // split-KV (set by simt_flash): key range split `blockIdx.z` of `nsplit`; partial rows
    // (unnormalised acc, fp32) and statistics (max, sum, entropy accumulator; double)
    int32_t nsplit = 1;
    void* part_acc = nullptr;      // (nsplit, U, nq, d), compute type
    double* part_stat = nullptr;   // (nsplit, U, nq, 3)
};
void simt_rstep(const SimtRstepArgs& a, vmb_dtype dt, cudaStream_t s);
void simt_lstep(const SimtLstepArgs& a, vmb_dtype dt, cudaStream_t s);
void simt_flash(const SimtFlashArgs& a, vmb_dtype dt, cudaStream_t s);
void check_finite_rows(View q, int64_t U, int64_t rows, int64_t d, vmb_dtype dt, int32_t* status,
                       cudaStream_t s);
void check_clamp_domain(const float* cR, int64_t n, int32_t* status, cudaStream_t s);
// hilo.cu: x = hi + lo, hi = bf16(x), lo = bf16(x - hi) for the fp32 rows (u, 0, t) of `v`
// (t < rows), into contiguous (U, rows, d) bf16 tensors; d % 4 == 0, rows 16-byte aligned
void split_hilo(const View& v, int64_t U, int64_t rows, int64_t d, void* hi, void* lo, cudaStream_t s);
// out[e] = hi[e] + lo[e] (fp32 state back from its hi/lo pair; the factor export)
void merge_hilo(const void* hi, const void* lo, float* out, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------- tcgen05 kernels (bf16, d = 128)
// fa2_tc.cu: 2 CTAs/SM flash attention with one value operand (R half-step: value = key,
// BN = 128; attention: separate V, BN = 64, optional split-KV + combine).
struct Tc2Args {
    CUtensorMap tmQ, tmK, tmV;   // 5-D maps (d, row, seg, head, batch); Q box rows 128, K/V box rows tc2_kv_tile(nv)
    int32_t nseg;                // segments per unit
    int32_t q_len, kv_len;       // rows per segment
    int32_t qH, kH, oHn;         // heads per batch of the q map, the k/v maps, the output
    const float* cR;             // per-row temperature source (U, nseg, q_len) or nullptr
    float qscale;                // logits multiplier (log2e applied inside)
    float clamp_min;
    int32_t clamp_enabled;
    int32_t nv;                  // 1: value = key tile (R-step); 2: separate V
    // output row (u, s, r) at out + (u/oHn)*oB + (u%oHn)*oH + s*oS + r*oR (bf16)
    void* out;
    int64_t oB, oH, oS, oR;
    float* cl_out;               // sum p ln p per row: (u, r, s) at (u*q_len + r)*nseg + s   (nv == 1 only)
    float* lse_out;              // natural-log lse: (u, s, r) at (u*nseg + s)*q_len + r
    float* ent_out;              // fa3 only: row entropy -sum P ln P, laid out as lse_out (nullptr: off)
    float* part_ent;             // fa3 split-KV: per-split entropies (n_useg, nsplit, q_len)
    int32_t* status;
    int32_t check_finite;
    // split-KV (attention): fp32 partials (n_useg, nsplit, q_len, 128) + lse (n_useg, nsplit, q_len)
    float* part_o;
    float* part_lse;
    int32_t max_split;           // 1 disables split-KV
    int32_t nsplit;              // set by the launcher
    int64_t n_useg;              // set by the launcher
    int32_t out_align32;         // set by the launcher: every output row 32-B aligned (256-bit stores)
    // optional low half of the bf16 output (R half-step: aL = hi + lo, hi = bf16(aL),
    // lo = bf16(aL - hi)), same layout as `out`; nullptr = not written
    void* out_lo;
    // bf16 plan, aL's low half (§5 of DESIGN.md): aln_out receives |aL row| (layout as cl_out);
    // qn_out (first R half-step) the max over frames of |Q row|^2 per (unit, position), (U, q_len)
    // (atomicMax; zeroed by the caller)
    float* aln_out;
    float* qn_out;
    // fp32 parity mode on tensor cores (hilo = 1): every operand is a pair of bf16 tensors
    // x = hi + lo; tmQ/tmK/tmV map the hi halves, these the lo halves (same boxes).  Products
    // run as three bf16 MMA groups (hi hi + hi lo + lo hi) into fp32.  out_f32: `out` rows are
    // fp32 (strides in floats), else bf16.
    CUtensorMap tmQlo, tmKlo, tmVlo;
    int32_t hilo;
    int32_t out_f32;
};
int tc2_kv_tile(int nv);
// 32-byte alignment of every bf16 output row of an attention launch (256-bit epilogue stores)
inline bool rows_align32(const void* base, int64_t oB, int64_t oH, int64_t oS, int64_t oR) {
    return reinterpret_cast<uintptr_t>(base) % 32 == 0 && oB % 16 == 0 && oH % 16 == 0 && oS % 16 == 0 &&
           oR % 16 == 0;
}
int tc2_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int nv, int max_split);
// Largest split count tc2_fa_launch may pick (sizes the partial buffers).
constexpr int kTc2MaxSplit = 16;
void tc2_fa_launch(Tc2Args a, int64_t U, cudaStream_t s);
// LSE combine of split-KV partials (a.nsplit, a.n_useg set by the launcher).
void tc2_combine_launch(const Tc2Args& a, cudaStream_t s);
// fa3_tc.cu: two 128-row query tiles per CTA, ping-pong softmax warpgroups, 128-key tiles
// (K/V maps with box rows 128).  Same argument block as fa2.
int tc3_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int max_split);
// returns the launched arguments (nsplit / n_useg set); do_combine = false leaves the split-KV
// combine to the caller (tc2_combine_launch), e.g. on another stream
Tc2Args tc3_fa_launch(Tc2Args a, int64_t U, cudaStream_t s, bool do_combine = true);
// fa4_tc.cu: persistent (one CTA per SM) flash attention over a flattened stream of
// (query tile, segment, kv-split) items; 128-key tiles (K/V maps with box rows 128).
//   nv = 1, v_is_k = 1: R half-step (out0 = aL, cl_out)
//   nv = 2            : R half-step + y (out0 = aL, out1 = y, cl_out), O = P [K | V]
//   nv = 1, v_is_k = 0: attention (out0), optional split-KV (part_o / part_lse / max_split)
struct Tc4Args {
    CUtensorMap tmQ, tmK, tmV;   // 5-D maps (d, row, seg, head, batch)
    int32_t nseg;
    int32_t q_len, kv_len;
    int32_t qH, kH, oHn;
    const float* cR;
    float qscale;
    float clamp_min;
    int32_t clamp_enabled;
    int32_t nv;
    int32_t v_is_k;
    void* out0;
    void* out1;
    int64_t oB[2], oH[2], oS[2], oR[2];
    float* cl_out;
    float* lse_out;
    int32_t* status;
    int32_t check_finite;
    float* part_o;
    float* part_lse;
    int32_t max_split;
    int32_t nsplit;              // set by the launcher
    // query rows for the epilogue's entropy dot (cl_out): row (u, s, r) at
    // q_rows + (u/qrHn)*qrB + (u%qrHn)*qrH + s*qrS + r*qrR (bf16)
    const void* q_rows;
    int64_t qrB, qrH, qrS, qrR;
    int32_t qrHn;
    int32_t out_align32;         // every output row 32-byte aligned: 256-bit epilogue stores
    void* out0_lo;               // optional low half of operand 0 (aL), laid out as out0
    // the low half is written for a row only where the L-step can need it: qn == nullptr
    // (always) or qn[u] * |aL row|^2 > lo_thresh2 (qn: max |Q row|^2 of the unit, from the first
    // R half-step, per (unit, position): (U, q_len)); aln_out / qn_out as in Tc2Args
    const float* qn;
    float lo_thresh2;
    float* aln_out;
    float* qn_out;
};  // (Tc4Args)
int tc4_plan_splits(int64_t q_len, int64_t kv_len, int64_t n_useg, int max_split);
void tc4_fa_launch(Tc4Args a, int64_t U, cudaStream_t s);
// All L-step tiles are boxes of `rows = lstep_rows(m)` rows (m rounded up to 16); rows
// >= m are OOB (zero-filled on load, clipped on store).
inline int32_t lstep_rows(int64_t m) { return (int32_t)((m + 15) & ~int64_t(15)); }
// bf16 tcgen05 L-step (lstep_tc.cu): spatial positions per CTA (stacked in the 128 tile rows)
// and the rows per position of its TMA boxes (the maps of Qb, aL, y, aR and O use these)
inline int32_t lstep_positions(int64_t m) { return m <= 32 ? 4 : (m <= 64 ? 2 : 1); }
inline int32_t lstep_box_rows(int64_t m) {
    const int32_t P = lstep_positions(m);
    return P > 1 ? 128 / P : lstep_rows(m);
}
struct TcLstepArgs {
    CUtensorMap tmQ;    // Q rows, 5-D (d, i, j, head, batch): Qb[i][j], box (64, 1, rows)
    CUtensorMap tmAL;   // aL rows, 5-D (d, k, i, 1, unit), box (64, rows, 1)
    CUtensorMap tmY;    // FINAL: y rows, 5-D (d, i, k, 1, unit), box (64, 1, rows)
    CUtensorMap tmOut;  // ITER: aR rows (d, i, k, 1, unit); FINAL: O rows (d, i, j, head, batch); box (64, 1, rows)
    const float* cL;    // (U, b, m)
    float qscale;
    int32_t m, b;
    int32_t H;          // heads per batch of the Q map
    int32_t oHn;        // heads per batch of the output map (FINAL)
    int32_t final_mode;
    float* cR;          // ITER: (U, m, b)
    float out_scale;    // multiplies the epilogue (ITER: aR scale)
    // aL = hi + lo (the R half-step writes the low half where it can matter): the low half,
    // same boxes as tmAL (use_lo = 0: never read).  The logit error of the hi half alone for
    // row k is at most qscale |Qb_j| |aL_k - hi_k| <= qscale Qmax |aL_k| 2^-9, so row k uses
    // its low half iff qscale^2 Qmax^2 |aL_k|^2 > kLoBound^2, i.e. qn[u, i] aln[k]^2 > lo_thresh2
    // (aln: (U, b, m) row norms of aL from the R half-step; qn: (U, b) max over the block's
    // query rows Qb[i][j] of |Q row|^2).
    CUtensorMap tmALlo;
    int32_t use_lo;
    const float* aln;
    const float* qn;
    float lo_thresh2;
};
// Logit-error bound below which a row of aL needs no low half: 2 * 2^-9 ~ 3.9e-3.
constexpr float kLoBound = 2.0f;
void tc_lstep_launch(const TcLstepArgs& a, int64_t U, cudaStream_t s);
// The fp32 parity mode's L half-step / apply on tensor cores (lstep_tc.cu, lstep_hl_kernel):
// every operand is a bf16 hi/lo pair (x = hi + lo), each product three bf16 MMA groups into
// fp32; L is stored as hi/lo; outputs are written from registers: ITER aR as hi/lo bf16
// (U, m, b, d) rows plus cR, FINAL O as fp32 rows of the caller's tensor.  d = 128, m <= 128.
struct TcLstepHlArgs {
    CUtensorMap tmQ, tmQlo;     // Qb rows of the hi/lo copies of Q, (d, i, j, 1, unit), box (64, 1, rows)
    CUtensorMap tmAL, tmALlo;   // aL hi/lo (d, k, i, 1, unit), box (64, rows, 1)
    CUtensorMap tmY, tmYlo;     // FINAL: y hi/lo (d, i, k, 1, unit), box (64, 1, rows)
    const float* cL;            // (U, b, m)
    float qscale;
    int32_t m, b;
    int32_t final_mode;
    float* cR;                  // ITER: (U, m, b)
    void* ar_hi;                // ITER: aR * qscale as bf16 hi/lo, (U, m, b, d)
    void* ar_lo;
    float* out;                 // FINAL: O row (u, token j*b + i) at (u/oHn)*oB + (u%oHn)*oH + token*oT
    int64_t oB, oH, oT;
    int32_t oHn;
};
void tc_lstep_hl_launch(const TcLstepHlArgs& a, int64_t U, cudaStream_t s);
// lstep_big.cu: L half-step / apply for m > 128 (row statistics pass + ITER or FINAL pass)
struct TcLstepBigArgs {
    CUtensorMap tmQ128, tmQ64;    // Qb rows (d, i, j, head, batch), boxes (64, 1, 128) / (64, 1, 64)
    CUtensorMap tmAL128, tmAL64;  // aL rows (d, k, i, 1, unit), boxes (64, 128, 1) / (64, 64, 1)
    CUtensorMap tmY64;            // FINAL: y rows (d, i, k, 1, unit), box (64, 1, 64)
    const float* cL;              // (U, b, m)
    float* lse2;                  // (U, b, m) scratch: base-2 row log-sum-exp of S
    float* cR;                    // ITER: (U, m, b)
    __nv_bfloat16* aR;            // ITER: (U, m, b, d)
    __nv_bfloat16* out;           // FINAL: O, row j*b + i of unit (ob, oh) at ob*oB + oh*oH + row*oT
    int64_t oB, oH, oT;
    float qscale, out_scale;
    int32_t m, b, H, oHn;
};
void tc_lstep_big_launch(const TcLstepBigArgs& a, int64_t U, bool final_mode, cudaStream_t s);
// flash_bwd.cu: backward of the online-entropy attention (flash_entropy.hpp:146-221)
void flash_bwd_launch(int64_t U, int64_t nq, int64_t nk, int64_t d, bool bf16, const void* q, const void* k,
                      const void* v, const void* o, const void* dout, const float* lse, const float* ent,
                      const float* dent, int entropy_grad, float* dvec, void* dq, void* dk, void* dv,
                      cudaStream_t s);

// flash_bwd_tc.cu: tcgen05 backward (bf16, d = 128, nq >= 1); rowstat scratch holds
// flash_bwd_tc_rowstat_rows(nq) float4 per unit
int64_t flash_bwd_tc_rowstat_rows(int64_t nq);
void flash_bwd_tc_launch(int64_t U, int64_t nq, int64_t nk, const void* q, const void* k, const void* v,
                         const void* o, const void* dout, const float* lse, const float* ent, const float* dent,
                         int entropy_grad, void* rowstat, void* dq, void* dk, void* dv, cudaStream_t s);

// seq_gather.cu: head-dim padding for d < 128 on the tcgen05 path.  to_padded: user rows
// (unit u = b*H + h at b*sb + h*sh + n*st elements, d columns) -> contiguous (U, N, 128) with
// zero columns [d, 128); otherwise the reverse (first d columns back to the user layout).
void pad_rows(const void* src, void* dst, int64_t U, int64_t N, int64_t d, int64_t H, int64_t sb, int64_t sh,
              int64_t st, bool to_padded, cudaStream_t s);

// seq_gather.cu: sequence-sharded K/V layout
constexpr int kMaxSeqRanks = 64;
void seq_assemble(const void* gathered, void* full, int64_t units, int64_t T, int64_t hw, int64_t slab_max,
                  int64_t row_bytes, int world, const int64_t* off, const int64_t* cnt, cudaStream_t s);
// device-side all-gather over peer memory: slab r of K/V (units, T, cnt[r], d) at k_src[r] /
// v_src[r] (any device with peer access) -> frame-major (units, T*hw, d) at k_dst / v_dst
void peer_gather(const void* const* k_src, const void* const* v_src, void* k_dst, void* v_dst, int64_t units,
                 int64_t T, int64_t hw, int64_t row_bytes, int world, const int64_t* off, const int64_t* cnt,
                 cudaStream_t s, int which = 3);  // which: 1 = K, 2 = V, 3 = both

void selftest_umma(int mode, const void* A, const void* B, float* C, cudaStream_t s);

}  // namespace vmb
