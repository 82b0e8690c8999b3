// Device-side parameter blocks for the non-tensor-core kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ed {

constexpr int kMaxRank = 8;
constexpr int kMaxDeps = 64;

// One inner EinSum over one chunk pair (kernel_eval, kernel.cc:15-68).
// Output labels z (chunk row-major), aggregation labels a (in the order of
// the distinct labels, so the fold runs in kernel_eval's odometer order).
struct GenericParams {
  int nz, na;
  int64_t zext[kMaxRank], aext[kMaxRank];
  int64_t xs_z[kMaxRank], ys_z[kMaxRank];   // input strides per output dim (0 = absent)
  int64_t xs_a[kMaxRank], ys_a[kMaxRank];   // input strides per aggregation dim
  int join, map, agg;                       // ed_join_op / ed_map_op / ed_agg_op, -1 absent
  double c;                                 // scale constant
  const void* x;
  const void* y;
  void* out;                                // storage dtype
  void* out16;                              // optional bf16 shadow
  int64_t n_out;
  int* err;                                 // device flag: 1 = division by zero
};

// One producer-side chunk folded into a refinement (runtime.cc:198-269).
struct DepRect {
  const void* src;
  int64_t r0[kMaxRank];     // region start, global coordinates
  int64_t ext[kMaxRank];    // region extent (= src chunk bound)
};

struct RefineParams {
  int rank;
  int n_deps;
  int agg;                  // -1 none
  int64_t c0[kMaxRank];     // consumer chunk start, global
  int64_t cext[kMaxRank];   // consumer chunk bound
  int64_t n_out;
  const DepRect* deps;      // device array, fold order
  void* out;
  void* out16;
  int lo;                   // 1: out16 is the fp32 lo shadow x - tf32(x) (fp32x3), 0: bf16
};

// Fast refinement: the overlap rectangle of one producer region with the
// consumer chunk, folding the region's aggregation siblings in dep order.
constexpr int kRectSrc = 8;
struct RectGroup {
  int n_src;
  const void* src[kRectSrc];
  int64_t src_off, dst_off;           // element offset of the rectangle's origin
  int64_t ext[kMaxRank];              // rectangle extents
  int64_t sstr[kMaxRank], dstr[kMaxRank];  // row-major strides of source region / consumer chunk
  int64_t rows;                       // prod(ext[0..rank-2])
};

struct RectParams {
  int rank;
  int agg;
  int vec;                            // 1: inner runs and offsets are 16-byte aligned
  int rows_per_block;
  const RectGroup* groups;            // device array
  void* out;
  void* out16;
  int lo;                             // 1: out16 is the fp32 lo shadow (fp32x3), 0: bf16
};

// Whole tensor <-> chunk buffers (chunk / assemble, relation.cc:31-78).
struct ChunkMapParams {
  int rank;
  int64_t bound[kMaxRank];
  int64_t cb[kMaxRank];     // chunk bound
  int64_t part[kMaxRank];   // partition d
  int64_t n;                // elements of the whole tensor
  void* const* chunks;      // device array, one pointer per key (lexicographic)
  void* const* shadows;     // optional bf16 shadows per key (nullable array)
};

enum class DT : int { F64 = 0, F32 = 1, BF16 = 2 };

// Rectangle copies between a whole tensor and its chunks (chunk / assemble,
// relation.cc:31-78), with dtype conversion and an optional bf16 shadow.
struct BlockCopy {
  const void* src;
  void* dst;
  void* dst16;                       // optional bf16 shadow of dst
  int64_t src_off, dst_off;
  int64_t ext[kMaxRank];
  int64_t sstr[kMaxRank], dstr[kMaxRank];
  int64_t rows;                      // prod(ext[0..rank-2])
};

struct BlockCopyParams {
  int rank;
  int in_dt, out_dt;                 // DT
  const BlockCopy* groups;           // device array
};

cudaError_t launch_generic(const GenericParams& p, bool f64, cudaStream_t s);
cudaError_t launch_refine(const RefineParams& p, bool f64, cudaStream_t s);
cudaError_t launch_rect(const RectParams& p, int n_groups, int64_t max_rows, bool f64, cudaStream_t s);
cudaError_t launch_scatter(const ChunkMapParams& p, const void* whole, DT in, DT store, cudaStream_t s);
cudaError_t launch_gather(const ChunkMapParams& p, void* whole, DT store, DT out, cudaStream_t s);
cudaError_t launch_blockcopy(const BlockCopyParams& p, int n_groups, int64_t max_rows, cudaStream_t s);
// 3xTF32 split: lo = x - tf32(x) (the low mantissa bits kind::tf32 drops)
cudaError_t launch_split_lo(const float* x, float* lo, int64_t n, cudaStream_t s);
cudaError_t launch_convert(const void* src, DT in, void* dst, DT out, int64_t n, cudaStream_t s);
cudaError_t launch_add_one(void* p, DT dt, cudaStream_t s);  // exec_options_t::corrupt hook

// generate_inputs (runtime.cc:552-571) on the device: one block per tensor
// runs std::mt19937_64(seed) 156 words at a time (the recurrence reaches 156
// words back at most) and applies libstdc++'s uniform_int_distribution<int>
// (-4, 4) (Lemire's nearly-divisionless downscale) or uniform_real_distribution
// <double>(-1, 1) (generate_canonical), bit for bit. A rejected integer draw
// (probability 7 / 2^64) would shift the stream: it is flagged in *err.
struct GenTensor {
  void* out;          // whole tensor, row-major, store dtype
  int64_t n;
  uint64_t seed;      // seed * 7919 + vid
};
cudaError_t launch_generate(const GenTensor* jobs, int n_jobs, bool integer_valued, DT store, int* err,
                            cudaStream_t s);

// Peer-memory transport (CUDA IPC / NVLink): run epochs and ready flags.
cudaError_t launch_peer_tick(int* epoch, cudaStream_t s);                     // epoch += 1
cudaError_t launch_peer_signal(int* flag, const int* epoch, cudaStream_t s);  // flag = epoch (release, system scope)
// spin until every flags[i] >= epoch + delta (acquire, system scope); after
// 20 s give up and set *err = 1 + tag * 64 + i (the stream then continues)
cudaError_t launch_peer_wait(int* const* flags, int n, const int* epoch, int delta, cudaStream_t s, int* err = nullptr,
                             int tag = -1);

}  // namespace ed
