// seq_gather.cu — layout kernel of the sequence-sharded mode.
//
// Rank r owns spatial positions [off_r, off_r + cnt_r) of every frame.  After the NCCL
// all-gather of K (or V) slabs the buffer holds, per rank, a (units, T, slab_max, d) block
// (slabs padded to the largest); this kernel scatters those rows into the frame-major
// (units, T, h*w, d) layout the attention kernels read (token = t*h*w + position).
// Pure data movement: 16-byte vectors, one warp per row of d elements, HBM-bound.
#include "../internal.hpp"

namespace vmb {
namespace {

struct AsmParams {
    const uint8_t* src;
    uint8_t* dst;
    int64_t units, T, hw, slab_max, row_bytes;
    int32_t world;
    int64_t off[kMaxSeqRanks];
    int64_t cnt[kMaxSeqRanks];
};

__global__ void __launch_bounds__(256) seq_assemble_kernel(const __grid_constant__ AsmParams p) {
    // one 16-B chunk per thread; grid covers (rank, unit, frame, slab position, chunk)
    const int64_t chunks = p.row_bytes / 16;
    const int64_t per_rank = p.units * p.T * p.slab_max * chunks;
    const int64_t total = per_rank * p.world;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(idx / per_rank);
        int64_t rest = idx % per_rank;
        const int64_t c = rest % chunks;
        rest /= chunks;
        const int64_t i = rest % p.slab_max;
        rest /= p.slab_max;
        const int64_t t = rest % p.T;
        const int64_t u = rest / p.T;
        if (i >= p.cnt[r]) continue;  // padding of a short slab
        const int64_t srow = idx / chunks;  // rows of the gathered buffer: (rank, unit, frame, position)
        const uint4 v = reinterpret_cast<const uint4*>(p.src + srow * p.row_bytes)[c];
        const int64_t drow = (u * p.T + t) * p.hw + p.off[r] + i;
        reinterpret_cast<uint4*>(p.dst + drow * p.row_bytes)[c] = v;
    }
}

}  // namespace

void seq_assemble(const void* gathered, void* full, int64_t units, int64_t T, int64_t hw, int64_t slab_max,
                  int64_t row_bytes, int world, const int64_t* off, const int64_t* cnt, cudaStream_t s) {
    VMB_REQUIRE_DIM(world >= 1 && world <= kMaxSeqRanks, "sequence-sharded world size out of range");
    VMB_REQUIRE_DIM(row_bytes % 16 == 0, "row size must be a multiple of 16 bytes");
    AsmParams p;
    p.src = static_cast<const uint8_t*>(gathered);
    p.dst = static_cast<uint8_t*>(full);
    p.units = units;
    p.T = T;
    p.hw = hw;
    p.slab_max = slab_max;
    p.row_bytes = row_bytes;
    p.world = world;
    for (int r = 0; r < kMaxSeqRanks; ++r) {
        p.off[r] = r < world ? off[r] : 0;
        p.cnt[r] = r < world ? cnt[r] : 0;
        if (r < world) VMB_REQUIRE_DIM(cnt[r] <= slab_max && off[r] + cnt[r] <= hw, "slab outside the frame");
    }
    const int64_t total = (int64_t)world * units * T * slab_max * (row_bytes / 16);
    if (total == 0) return;
    int dev = 0, sms = 148;
    VMB_CHECK_CUDA(cudaGetDevice(&dev));
    VMB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 16);
    ProfScope ps(kKSimt, s);
    seq_assemble_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
    count_launch();
    check_launch("seq_assemble");
}

}  // namespace vmb

// ---------------------------------------------------------------- peer-memory all-gather
// Single-process multi-GPU sequence-sharded mode (vmb_vmonarch_fwd_multi): device r reads
// every peer's K and V slab (units, T, cnt_p, d) straight out of the peer's HBM over NVLink
// (P2P loads through the unified address space) and writes the frame-major (units, N, d)
// tensors into its own workspace.  One kernel per device replaces the NCCL all-gather plus
// the assemble pass of the process-per-GPU mode: no padded staging buffer, no second copy.
namespace vmb {
namespace {

struct PeerGatherParams {
    const uint8_t* k_src[kMaxSeqRanks];
    const uint8_t* v_src[kMaxSeqRanks];
    uint8_t* k_dst;
    uint8_t* v_dst;
    int64_t off[kMaxSeqRanks];
    int64_t cnt[kMaxSeqRanks];
    int64_t rows_before[kMaxSeqRanks + 1];  // prefix sum of units * T * cnt_p
    int64_t units, T, hw, row_bytes;
    int32_t world;
    int32_t which;  // 1: K, 2: V, 3: both
};

__global__ void __launch_bounds__(256) peer_gather_kernel(const __grid_constant__ PeerGatherParams p) {
    const int64_t chunks = p.row_bytes / 16;
    const int64_t rows = p.rows_before[p.world];
    const int64_t total = (p.which == 3 ? 2 : 1) * rows * chunks;  // K then V
    // consecutive threads take consecutive 16-B chunks of one row, so every warp moves whole
    // 256-B rows and the peer reads coalesce into full NVLink packets
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx % chunks;
        int64_t row = idx / chunks;
        const bool is_v = p.which == 2 || (p.which == 3 && row >= rows);
        if (row >= rows) row -= rows;
        int r = 0;
        while (row >= p.rows_before[r + 1]) ++r;
        const int64_t local = row - p.rows_before[r];  // (unit, frame, position) within slab r
        const int64_t i = local % p.cnt[r];
        const int64_t ut = local / p.cnt[r];
        const uint8_t* src = (is_v ? p.v_src[r] : p.k_src[r]) + local * p.row_bytes;
        uint8_t* dst = (is_v ? p.v_dst : p.k_dst) + (ut * p.hw + p.off[r] + i) * p.row_bytes;
        reinterpret_cast<uint4*>(dst)[c] = __ldcs(reinterpret_cast<const uint4*>(src) + c);
    }
}

}  // namespace

void peer_gather(const void* const* k_src, const void* const* v_src, void* k_dst, void* v_dst, int64_t units,
                 int64_t T, int64_t hw, int64_t row_bytes, int world, const int64_t* off, const int64_t* cnt,
                 cudaStream_t s, int which) {
    VMB_REQUIRE_DIM(world >= 1 && world <= kMaxSeqRanks, "sequence-sharded world size out of range");
    VMB_REQUIRE_DIM(row_bytes % 16 == 0, "row size must be a multiple of 16 bytes");
    PeerGatherParams p;
    p.k_dst = static_cast<uint8_t*>(k_dst);
    p.v_dst = static_cast<uint8_t*>(v_dst);
    p.units = units;
    p.T = T;
    p.hw = hw;
    p.row_bytes = row_bytes;
    p.world = world;
    p.which = which;
    p.rows_before[0] = 0;
    for (int r = 0; r < kMaxSeqRanks; ++r) {
        const bool in = r < world;
        p.k_src[r] = in ? static_cast<const uint8_t*>(k_src[r]) : nullptr;
        p.v_src[r] = in ? static_cast<const uint8_t*>(v_src[r]) : nullptr;
        p.off[r] = in ? off[r] : 0;
        p.cnt[r] = in ? cnt[r] : 1;
        if (in) {
            VMB_REQUIRE_DIM(cnt[r] >= 1 && off[r] >= 0 && off[r] + cnt[r] <= hw, "slab outside the frame");
            p.rows_before[r + 1] = p.rows_before[r] + units * T * cnt[r];
        } else {
            p.rows_before[r + 1] = p.rows_before[r];
        }
    }
    const int64_t total = (which == 3 ? 2 : 1) * p.rows_before[world] * (row_bytes / 16);
    if (total == 0) return;
    int dev = 0, sms = 148;
    VMB_CHECK_CUDA(cudaGetDevice(&dev));
    VMB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    ProfScope ps(kKSimt, s);
    peer_gather_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
    count_launch();
    check_launch("peer_gather");
}

}  // namespace vmb

// ---------------------------------------------------------------- head-dim padding (d < 128)
namespace vmb {
namespace {

__global__ void __launch_bounds__(256) pad_rows_kernel(const uint8_t* src, uint8_t* dst, int64_t U, int64_t N,
                                                       int64_t chunks_real, int64_t H, int64_t sb, int64_t sh,
                                                       int64_t st, int to_padded) {
    // one 16-byte chunk per thread; a padded row is 16 chunks (128 bf16)
    const int64_t total = U * N * 16;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx & 15, row = idx >> 4;
        const int64_t u = row / N, n = row % N;
        const int64_t user = ((u / H) * sb + (u % H) * sh + n * st) * 2;  // bytes
        if (to_padded) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (c < chunks_real) v = reinterpret_cast<const uint4*>(src + user)[c];
            reinterpret_cast<uint4*>(dst + row * 256)[c] = v;
        } else if (c < chunks_real) {
            reinterpret_cast<uint4*>(dst + user)[c] = reinterpret_cast<const uint4*>(src + row * 256)[c];
        }
    }
}

// element-wise variant for user tensors whose rows are not 16-byte aligned
__global__ void __launch_bounds__(256) pad_rows_any_kernel(const uint16_t* src, uint16_t* dst, int64_t U, int64_t N,
                                                           int64_t d, int64_t H, int64_t sb, int64_t sh, int64_t st,
                                                           int to_padded) {
    const int64_t total = U * N * 128;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = idx & 127, row = idx >> 7;
        const int64_t u = row / N, n = row % N;
        const int64_t user = (u / H) * sb + (u % H) * sh + n * st;
        if (to_padded) dst[idx] = x < d ? src[user + x] : (uint16_t)0;
        else if (x < d) dst[user + x] = src[idx];
    }
}

}  // namespace

void pad_rows(const void* src, void* dst, int64_t U, int64_t N, int64_t d, int64_t H, int64_t sb, int64_t sh,
              int64_t st, bool to_padded, cudaStream_t s) {
    if (U * N == 0) return;
    const void* user = to_padded ? src : dst;
    const bool vec = (reinterpret_cast<uintptr_t>(user) & 15) == 0 && d % 8 == 0 && sb % 8 == 0 && sh % 8 == 0 &&
                     st % 8 == 0;
    const int64_t total = U * N * (vec ? 16 : 128);
    int dev = 0, sms = 148;
    VMB_CHECK_CUDA(cudaGetDevice(&dev));
    VMB_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 16);
    ProfScope ps(kKSimt, s);
    if (vec)
        pad_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst),
                                                         U, N, d / 8, H, sb, sh, st, to_padded ? 1 : 0);
    else
        pad_rows_any_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint16_t*>(src),
                                                             static_cast<uint16_t*>(dst), U, N, d, H, sb, sh, st,
                                                             to_padded ? 1 : 0);
    count_launch();
    check_launch("pad_rows");
}

}  // namespace vmb
