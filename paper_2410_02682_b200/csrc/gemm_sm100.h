// tcgen05 block-contraction kernel interface (see gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace ed {

constexpr int kMaxSib = 8;  // aggregation siblings folded in one accumulator

struct GemmParams {
  CUtensorMap a[kMaxSib];   // MMA-A operand of each sibling (M x K), 3-D {inner, outer, batch}
  CUtensorMap b[kMaxSib];   // MMA-B operand of each sibling (N x K)
  int n_sib;
  int M, N, K, batch;
  int a_mn, b_mn;           // 1: operand is MN-major (M or N contiguous)
  int vec_ok;               // 1: output rows 16-byte aligned (vector stores)
  float* c32;               // fp32 output (nullable)
  void* c16;                // bf16 shadow output (nullable)
  long long c_sm, c_sb;     // output element strides for M and batch; N stride is 1
};

int gemm_bk(bool bf16);
int gemm_bn(bool bf16);
cudaError_t gemm_prepare();  // sets the dynamic-smem attribute (call before capture)
cudaError_t launch_gemm(const GemmParams& p, bool bf16, cudaStream_t stream);

}  // namespace ed
