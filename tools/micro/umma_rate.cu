// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) for the
// shared-memory (SS) and A-from-TMEM (TS) forms at N = 64 / 128 / 256, one
// CTA, operands left uninitialised (rate only). Built by hand:
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2410_02682_b200/csrc umma_rate.cu -o umma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ed;

template <int N, bool TS, int LOADERS, int BMN = 0>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc(1u, 128, N, 0u, uint32_t(BMN));
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t bd = BMN ? umma_desc_sw128(sb + (i & 7) * 2048, 16384, 1024)  // V: MN-major atoms
                              : umma_desc_sw128(sb + (i & 3) * 32, 16, 1024);
      if (TS) mma_f16_ts(tmem + 256, tmem + (i & 7) * 8, bd, idesc, 1u);
      else mma_f16(tmem + 256, umma_desc_sw128(sa + (i & 3) * 32, 16, 1024), bd, idesc, 1u);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
    *(volatile int*)&slot = 0xFFFFFFFF;  // stop the loaders
  } else if (LOADERS < 0 && warp >= 4) {
    // busy warps doing softmax-like math on every SMSP (incl. the MMA thread's)
    float x = threadIdx.x * 0.001f, acc = 0.f;
    for (int it = 0; it < 200000 && *(volatile uint32_t*)&slot != 0xFFFFFFFF; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x + u));
        acc = fmaf(y, 0.5f, acc);
      }
    }
    if (acc == 12345.f) out[2] = 1;
  } else if (LOADERS >= 100 && warp >= 4 && warp < 4 + (LOADERS - 100)) {
    // concurrent TMEM stores (and loads) like the softmax's P and the O rescale
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16);
    uint32_t r[32];
    for (int e = 0; e < 32; ++e) r[e] = e;
    for (int it = 0; it < 100000 && *(volatile uint32_t*)&slot != 0xFFFFFFFF; ++it) {
      tmem_st_32x32b_x32(base + 64 + (it % 6) * 32, r);
      tmem_st_wait();
      tmem_ld_32x32b_x32(base + 64 + ((it + 3) % 6) * 32, r);
      tmem_ld_wait();
    }
    if (r[3] == 12345) out[2] = 1;
  } else if (warp >= 4 && warp < 4 + LOADERS) {
    // concurrent TMEM traffic: other warps stream tcgen05.ld over columns [64, 256)
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16);
    uint32_t r[32], acc = 0;
    for (int it = 0; it < 100000 && *(volatile uint32_t*)&slot != 0xFFFFFFFF; ++it) {
      tmem_ld_32x32b_x32(base + 64 + (it % 6) * 32, r);
      tmem_ld_wait();
      acc += r[it & 31];
    }
    if (acc == 12345) out[2] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS, int LOADERS = 0, int BMN = 0>
void run(long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(k<N, TS, LOADERS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 32768);
  const int threads = LOADERS < 0 ? 128 + 32 * (-LOADERS) : LOADERS >= 100 ? 128 + 32 * (LOADERS - 100) : 256;
  k<N, TS, LOADERS, BMN><<<1, threads, 65536 + 32768>>>(d, iters);
  k<N, TS, LOADERS, BMN><<<1, threads, 65536 + 32768>>>(d, iters);
  long long h[2];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  std::printf("%s%s N=%3d loaders=%d: %.1f cycles per MMA (issue loop %.1f)  [%s]\n", TS ? "TS" : "SS", BMN ? " B-MN-major" : "", N, LOADERS, double(h[1]) / iters,
              double(h[0]) / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<64, true>(d); run<128, true>(d); run<256, true>(d);
  run<128, false, 4>(d); run<128, true, 4>(d);
  run<128, true, 0, 1>(d); run<128, true, 104, 1>(d); run<128, true, 108, 1>(d); run<128, false, 108, 0>(d);
  return 0;
}
