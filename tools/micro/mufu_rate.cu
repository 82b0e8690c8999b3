// MUFU.EX2 / FFMA2 issue rates on one SM: W warps, each issuing N
// independent ex2.approx.ftz (8 chains) — cycles per warp-instruction.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (MODE == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0f3A000000;" : "+f"(a[i]));
      else if (MODE == 2) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0f3A000000;" : "+f"(a[i]));
      } else if (MODE == 3) {  // F2FP pack: bf16x2 from two f32
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        a[i] = __uint_as_float(r);
      } else if (MODE == 4) {  // F2FP + ex2 interleaved
        unsigned r;
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 3) & 7]));
        a[i] = __uint_as_float(r) * 1e-30f;
      } else {  // PRMT high halves
        unsigned r;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a[i])), "r"(__float_as_uint(a[(i + 1) & 7])));
        a[i] = __uint_as_float(r);
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  const int iters = 4096;
  for (int mode = 0; mode < 6; ++mode)
    for (int w : {1, 4, 16}) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : k<5>;
      f<<<1, 32 * w>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double instr = double(iters) * 8 * w * (mode == 2 || mode == 4 ? 2 : 1);  // warp-instructions on the SM
      std::printf("mode %d (%s) warps %2d: %.2f cycles per warp-instr per SMSP, %.1f lanes/clk/SM\n", mode,
                  mode == 0 ? "ex2" : mode == 1 ? "fma" : mode == 2 ? "ex2+fma" : mode == 3 ? "f2fp" : mode == 4 ? "ex2+f2fp" : "prmt", w, double(c) / (instr / (w < 4 ? w : 4)),
                  instr * 32 / double(c));
    }
  return 0;
}
