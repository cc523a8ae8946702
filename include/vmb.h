/*
 * vmb.h — C ABI of the B200-native VMonarch attention forward (libvmb.so).
 *
 * Drop-in boundary for the reference operator API (/root/reference/proj):
 *   vmonarch::vmonarch_attention<T>(qs, ks, vs, TokenGrid, VMonarchConfig, threads,
 *                                    factors_out)                  video.hpp:84-150
 *   vmonarch::r_update / l_update (IterState half-steps)           monarch.hpp:53-147
 *   vmonarch::flash_entropy_fwd (online-entropy attention)         flash_entropy.hpp:85-139
 *   vmonarch::dense_forward (quadratic baseline)                   oracle.hpp:36-72
 *   vmonarch::factorize / flops_estimate / make_perm               video.cpp:13-59, perm.hpp:19-30
 * The C++ façade include/vmonarch_b200.hpp re-exposes these with the reference's
 * signatures and exception types on top of this ABI.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Tensor pointers are DEVICE pointers; every
 *    compute entry point is stream-ordered on `stream` (a cudaStream_t passed as
 *    void*, NULL = legacy default stream) and returns after enqueueing work.
 *  - Q/K/V/O of the operator: one (N, d) matrix per batch*head unit, d contiguous.
 *    `vmb_strides` gives element strides of batch, head and token (so both the
 *    reference's unit-major layout and BSHD activations are accepted).  NULL means
 *    contiguous unit-major: unit u = b*H + h at offset u*N*d, token stride d.
 *  - dtype VMB_F32: fp32 storage and fp32/f64 arithmetic mirroring the reference
 *    precision policy for T = float (parity mode, <= 1e-4).  VMB_F64: the same on f64
 *    storage and arithmetic, the reference's T = double (video.hpp:84 is a template over
 *    T; its tests run in double); vmb_vmonarch_fwd and vmb_export_factors only.
 *    VMB_BF16: bf16 storage, tcgen05 bf16 tensor-core math with fp32 accumulation and fp32
 *    row statistics (<= 2e-2).
 *  - Errors mirror check.hpp:10-20: VMB_ERR_DIM (std::invalid_argument "dimension
 *    error"), VMB_ERR_DOMAIN (std::domain_error), VMB_ERR_STATE (std::logic_error).
 *    Host-detectable errors are returned synchronously; data-dependent domain
 *    errors (non-finite Q, monarch.hpp:44; c_R <= 0 without clamp, monarch.hpp:78)
 *    are raised on the device into the workspace status word and returned by
 *    vmb_workspace_status().  vmb_last_error() gives the thread-local message.
 *  - Reentrant per stream; one workspace per concurrent call.  No CPU fallback:
 *    every compute path is a CUDA kernel; a missing GPU returns VMB_ERR_CUDA.
 */
#ifndef VMB_H
#define VMB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    VMB_OK = 0,
    VMB_ERR_DIM = 1,     /* std::invalid_argument, "dimension error: ..." */
    VMB_ERR_DOMAIN = 2,  /* std::domain_error,     "domain error: ..."    */
    VMB_ERR_STATE = 3,   /* std::logic_error,      "state error: ..."     */
    VMB_ERR_CUDA = 4,    /* CUDA runtime / launch failure                 */
    VMB_ERR_NCCL = 5     /* collective failure (sequence-sharded mode)    */
} vmb_status;

typedef enum { VMB_F32 = 0, VMB_BF16 = 1, VMB_F64 = 2 } vmb_dtype;

/* TokenGrid (video.hpp:16-27): frame-major tokens, token = t*(h*w) + r*w + c. */
typedef struct {
    int64_t t_frames, h, w, head_dim, heads, batch;
} vmb_grid;

/* VMonarchConfig (video.hpp:29-36) + TileConfig (flash_entropy.hpp:13-16).
 * override_m = override_b = 0 selects the default factorization (T, h*w). */
typedef struct {
    int64_t iters;               /* default 2 */
    double clamp_min;            /* default 0.1 */
    int32_t clamp_enabled;       /* default 1 */
    int32_t recompute_first_frame; /* default 1 */
    int64_t override_m, override_b;
    int64_t tile_br, tile_bc;    /* accepted for API parity; outputs are tile independent */
} vmb_config;

/* Element strides of a (batch, head, token, d) view; d is contiguous. */
typedef struct {
    int64_t batch, head, token;
} vmb_strides;

/* ---- host-side bookkeeping (bit-exact integer work, no device needed) ---- */
void vmb_config_default(vmb_config* cfg);
/* video.cpp:13-22 */
vmb_status vmb_factorize(const vmb_grid* grid, const vmb_config* cfg, int64_t* m, int64_t* b);
/* perm.hpp:19-30: forward_index[j*(n/b) + i] = i*b + j. */
vmb_status vmb_make_perm(int64_t b, int64_t n, int64_t* forward_index);
/* video.cpp:36-59 (per batch*head unit). */
vmb_status vmb_flops_estimate(const vmb_grid* grid, const vmb_config* cfg, int64_t d,
                              double* sparsity, double* sparsity_approx,
                              uint64_t* monarch_flops, uint64_t* full_attn_flops,
                              uint64_t* recompute_flops, double* reduction_ratio);
const char* vmb_last_error(void);
const char* vmb_version(void);

/* ---- the operator (video.hpp:84-150) ---- */
size_t vmb_workspace_size(const vmb_grid* grid, const vmb_config* cfg, vmb_dtype dtype);
/* q, k, v: inputs with `in_strides` (NULL = contiguous unit-major); o: output with
 * `out_strides`.  `workspace` (device, >= vmb_workspace_size bytes, 256-B aligned)
 * also carries the device status word read by vmb_workspace_status(). */
vmb_status vmb_vmonarch_fwd(const vmb_grid* grid, const vmb_config* cfg, vmb_dtype dtype,
                            const void* q, const void* k, const void* v, void* o,
                            const vmb_strides* in_strides, const vmb_strides* out_strides,
                            void* workspace, size_t workspace_bytes, void* stream);
/* Synchronises `stream` and returns the device-raised status of the last call that
 * used `workspace` (VMB_OK or VMB_ERR_DOMAIN), then clears it. */
vmb_status vmb_workspace_status(void* workspace, void* stream);

/* Factor export (MonarchFactors, monarch.hpp:12-19) for the most recent
 * vmb_vmonarch_fwd that used `workspace`: L (units, b, m, m) and R (units, m, b, b)
 * in fp32 -- f64 for dtype VMB_F64, the buffers passed cast to float* -- (device pointers;
 * either may be NULL), recomputed from the workspace state with
 * the same q/k the forward used.  Call R before or together with L (the L export reuses
 * the aR/cR scratch).  Small N only: R is m*b*b per unit. */
vmb_status vmb_export_factors(const vmb_grid* grid, const vmb_config* cfg, vmb_dtype dtype,
                              const void* q, const void* k, const vmb_strides* in_strides,
                              void* workspace, float* L, float* R, void* stream);

/* ---- sequence-sharded mode (multi-GPU) ----
 * Rank r owns spatial positions [pos_begin, pos_begin + pos_count) of every frame.  Its
 * queries/outputs are the local slab, contiguous unit-major (units, T * pos_count, d) with
 * local token = t * pos_count + (position - pos_begin); keys/values are the full tensors
 * (units, N, d), assembled from the ranks' slabs by one all-gather (NCCL) and
 * vmb_seq_assemble.  R-step queries, L-step blocks and the first-frame recompute rows are
 * all slab-local, so this is the only exchange (video.hpp:115-126 per unit).  Default
 * factorization only; bf16, d = 128, T <= 128. */
size_t vmb_workspace_size_seq(const vmb_grid* grid, const vmb_config* cfg, vmb_dtype dtype, int64_t pos_count);
vmb_status vmb_vmonarch_fwd_seq(const vmb_grid* grid, const vmb_config* cfg, vmb_dtype dtype,
                                int64_t pos_begin, int64_t pos_count, const void* q_local,
                                const void* k_full, const void* v_full, void* o_local,
                                void* workspace, size_t workspace_bytes, void* stream);
/* As vmb_vmonarch_fwd_seq, with V still in flight: `v_ready` (a cudaEvent_t passed as void*,
 * may be NULL) completes when v_full is assembled; the stream waits on it just before the first
 * launch that reads V (the last R half-step), so the V all-gather overlaps the first R and L
 * half-steps. */
vmb_status vmb_vmonarch_fwd_seq_v(const vmb_grid* grid, const vmb_config* cfg, vmb_dtype dtype,
                                  int64_t pos_begin, int64_t pos_count, const void* q_local,
                                  const void* k_full, const void* v_full, void* o_local,
                                  void* workspace, size_t workspace_bytes, void* stream, void* v_ready);
/* gathered: `world` blocks of (units, T, slab_max, d) (slab r padded to slab_max rows) ->
 * full (units, T*h*w, d); rank r's rows land at positions [pos_begin[r], +pos_count[r]). */
vmb_status vmb_seq_assemble(const vmb_grid* grid, vmb_dtype dtype, int32_t world, const int64_t* pos_begin,
                            const int64_t* pos_count, int64_t slab_max, const void* gathered, void* full,
                            void* stream);

/* ---- single-process multi-GPU ----
 * One call drives n_dev devices: devices[r] is a CUDA ordinal, streams[r] a stream on it
 * (streams == NULL: the legacy default streams), and q/k/v/o[r], workspace[r] live on it.
 * Parts are contiguous and differ in size by at most one (vmb_shard_range).
 *  VMB_SHARD_HEADS: device r owns the unit block vmb_shard_range(batch*heads, n_dev, r);
 *    q/k/v/o[r] are (units_r, N, d) contiguous.  Units are independent (video.hpp:115-148),
 *    so there is no inter-device traffic; results are bitwise equal to the 1-device call.
 *  VMB_SHARD_SEQ: device r owns spatial positions vmb_shard_range(h*w, n_dev, r) of every
 *    frame, for every unit: q/k/v/o[r] are (units, T*count_r, d), token t*count_r + i, as in
 *    vmb_vmonarch_fwd_seq.  The K/V slabs are all-gathered inside the call by one kernel
 *    per device reading its peers' HBM over NVLink (P2P; peer access is enabled here and
 *    required, VMB_ERR_NCCL otherwise) into workspace[r]; then the slab forward runs.  V is
 *    gathered on a side stream and overlaps the first R/L half-steps (first read by the last
 *    R half-step).
 *    Default factorization; bf16, d = 128, T <= 128.
 * Stream-ordered on every streams[r]; the call joins all streams (cross-device events)
 * before the gather and after it, so inputs may be rewritten once streams[r] moves on.
 * The process-per-GPU equivalent is vmb_vmonarch_fwd_seq + the caller's all-gather
 * (NCCL) + vmb_seq_assemble. */
typedef enum { VMB_SHARD_HEADS = 0, VMB_SHARD_SEQ = 1 } vmb_shard_mode;
void vmb_shard_range(int64_t n, int32_t parts, int32_t r, int64_t* begin, int64_t* count);
size_t vmb_workspace_size_multi(int32_t n_dev, int32_t rank, vmb_shard_mode mode, const vmb_grid* grid,
                                const vmb_config* cfg, vmb_dtype dtype);
vmb_status vmb_vmonarch_fwd_multi(int32_t n_dev, const int32_t* devices, vmb_shard_mode mode, const vmb_grid* grid,
                                  const vmb_config* cfg, vmb_dtype dtype, const void* const* q, const void* const* k,
                                  const void* const* v, void* const* o, void* const* workspace,
                                  const size_t* workspace_bytes, void* const* streams);

/* ---- half steps (monarch.hpp:53-147), unit-major contiguous state tensors ----
 * aR (units,m,b,d) dtype; cR (units,m,b) f32; Kb (units,m,b,d) dtype;
 * aL (units,b,m,d) dtype; cL (units,b,m) f32; Qb (units,b,m,d) dtype (the permuted,
 * pre-scaled Q as in monarch.hpp:173).  R (units,m,b,b) / L (units,b,m,m) f32 may be
 * NULL.  Domain errors (c_R <= 0 without clamp) are checked synchronously. */
vmb_status vmb_rstep(int64_t units, int64_t m, int64_t b, int64_t d, vmb_dtype dtype,
                     const void* aR, const float* cR, const void* Kb, double clamp_min,
                     int32_t clamp_enabled, void* aL, float* cL, float* R, void* stream);
vmb_status vmb_lstep(int64_t units, int64_t m, int64_t b, int64_t d, vmb_dtype dtype,
                     const void* Qb, const void* aL, const float* cL, void* aR, float* cR,
                     float* L, void* stream);

/* ---- online-entropy attention (flash_entropy.hpp:85-139) ----
 * q (units,nq,d), k/v (units,nk,d), contiguous; Q must already carry its scale
 * (q_scale multiplies the logits, 1.0 = reference semantics).  lse/ent (units,nq)
 * f32, may be NULL. */
vmb_status vmb_flash_entropy_fwd(int64_t units, int64_t nq, int64_t nk, int64_t d,
                                 vmb_dtype dtype, const void* q, const void* k, const void* v,
                                 float q_scale, void* o, float* lse, float* ent, void* stream);

/* ---- its backward (flash_entropy.hpp:146-221; the paper's fine-tuning path, Alg. 2) ----
 * q (pre-scaled), k, v, o, dout (units, n, d) dtype; lse / ent / dent (units, nq) f32 from the
 * matching forward (ent, dent may be NULL unless entropy_grad).  dq (units, nq, d), dk / dv
 * (units, nk, d) in dtype are overwritten.  entropy_grad adds -dH P (S - lse + H) to dS. */
vmb_status vmb_flash_entropy_bwd(int64_t units, int64_t nq, int64_t nk, int64_t d, vmb_dtype dtype,
                                 const void* q, const void* k, const void* v, const void* o,
                                 const void* dout, const float* lse, const float* ent,
                                 const float* dent, int32_t entropy_grad, void* dq, void* dk,
                                 void* dv, void* stream);

/* ---- dense attention baseline (oracle.hpp:36-72 semantics, scale 1/sqrt(d)) ---- */
vmb_status vmb_dense_fwd(int64_t units, int64_t n, int64_t d, vmb_dtype dtype, const void* q,
                         const void* k, const void* v, void* o, void* stream);

/* ---- caller-side harness (host only) ----
 * The reference bench's workload generator (bench_main.cpp:78-90): count values from
 * std::mt19937_64(seed) through normal_distribution<double>(0,1) (dist 0) or
 * uniform_real_distribution<double>(-1,1) (dist 1), cast to float (host buffer). */
vmb_status vmb_workload_fill(uint64_t seed, int64_t count, int32_t dist, float* out);

/* ---- diagnostics ---- */
/* Number of kernels the library launched since load (all entry points). */
uint64_t vmb_kernel_launch_count(void);
/* Per-kernel CUDA-event timing (off by default).  Kernel ids: 0 R half-step, 1 last R
 * half-step (+ y), 2 attention (recompute / dense), 3 L half-step, 4 L half-step + apply,
 * 5 CUDA-core kernels, 6 split-KV combine.  vmb_profile_read fills up to 7 entries and
 * returns the count. */
void vmb_profile_enable(int32_t on);
int32_t vmb_profile_read(double* ms, uint64_t* counts, int32_t reset);
/* Self-test of the tcgen05/TMA building blocks: mode 0 C = A B^T, 1 C = A B,
 * 2 C = A B with A staged in TMEM.  A, B (128x128 bf16 row-major), C (128x128 f32). */
vmb_status vmb_selftest_umma(int32_t mode, const void* A, const void* B, float* C, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VMB_H */
