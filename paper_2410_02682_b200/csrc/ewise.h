// Grouped memory-bound join kernels (see ewise.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ed {

// Per-join operand pointers of a grouped launch (blockIdx.y = join).
struct JoinPtrs {
  const void* x;
  const void* y;
  void* out;     // storage dtype (nullable)
  void* out16;   // bf16 shadow (nullable)
};

struct EwiseParams {
  const JoinPtrs* joins;  // device array
  int64_t n;              // elements per join output
  int binary;             // 1: join op with y
  int y_mode;             // 1: y has Z's layout, 2: y broadcast over Z's trailing `inner` elements
  int64_t inner;
  int join, map;
  double c;
  int* err;               // division-by-zero flag
};

struct RowReduceParams {
  const JoinPtrs* joins;
  int64_t rows, len;      // Z elements, aggregated elements per Z element (trailing in X)
  int map, agg;
  double c;
};

// Fused row softmax (max, sub, exp, sum, div of one row block in registers):
// Y = exp(X - max_row) / sum_row exp(X - max_row), rows of `len` elements.
// One column segment of a softmax input row read in place from a producer
// region (the refinement that would paste it is elided).
struct RowSeg {
  const float* ptr;
  int64_t row0;     // row of the consumer chunk's first row inside this region
  int64_t stride;   // region row stride (elements)
};

struct SoftmaxParams {
  const JoinPtrs* joins;  // x = the chain's input chunk, y = row maxima or null, out/out16 = Y's chunk
  int64_t rows;
  int len;
  const RowSeg* segs;     // nullable: n_seg segments per join, each seg_w columns
  int n_seg, seg_w;
  int lo;                 // 1: out16 is the fp32 lo shadow y - tf32(y) (fp32x3 consumers), 0: bf16
};

cudaError_t launch_softmax(const SoftmaxParams& p, int n_joins, cudaStream_t s);
cudaError_t launch_ewise(const EwiseParams& p, int n_joins, bool f64, bool exact, cudaStream_t s);
cudaError_t launch_rowreduce(const RowReduceParams& p, int n_joins, bool f64, bool exact, cudaStream_t s);

}  // namespace ed
