// Microbenchmark: mbarrier ping-pong latency between two warps of one CTA for
// try_wait (default suspend), try_wait with a suspend-time hint, and a
// test_wait spin. Build: nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2410_02682_b200/csrc mbar_latency.cu -o mbar_latency
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ed;

__device__ __forceinline__ void wait_hint(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
      "@!P bra W_%=;\n\t}" ::"r"(addr), "r"(parity), "r"(ns) : "memory");
}
__device__ __forceinline__ void wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "S_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra S_%=;\n\t}" ::"r"(addr), "r"(parity) : "memory");
}

template <int MODE>
__global__ void k(long long* out, int iters) {
  __shared__ uint64_t a, b;
  if (threadIdx.x == 0) { mbar_init(&a, 1); mbar_init(&b, 1); fence_mbar_init(); }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto wait = [&](uint64_t* bar, uint32_t ph) {
    if (MODE == 0) mbar_wait(bar, ph);
    else if (MODE == 1) wait_hint(bar, ph, 20);
    else wait_spin(bar, ph);
  };
  if (lane == 0 && warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_arrive(&a);
      wait(&b, i & 1);
    }
    out[MODE] = (clock64() - t0) / iters;
  } else if (lane == 0 && warp == 1) {
    for (int i = 0; i < iters; ++i) {
      wait(&a, i & 1);
      mbar_arrive(&b);
    }
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  k<0><<<1, 64>>>(d, 10000);
  k<1><<<1, 64>>>(d, 10000);
  k<2><<<1, 64>>>(d, 10000);
  long long h[3];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  std::printf("round trip cycles: try_wait %lld, try_wait(20ns hint) %lld, test_wait spin %lld [%s]\n", h[0], h[1],
              h[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
