// Memory-bound join kernels (HBM roofline), grouped: one launch covers every
// join of one einsum on this rank (blockIdx.y = join).
//
//   ewise     : no aggregation; Z = X's layout, Y absent / same layout /
//               broadcast over Z's trailing labels (sub(C[i,k], M[i]))
//   rowreduce : unary map + aggregation over X's trailing labels
//               (max[k] map identity(C[i,k]), sum[s2] map identity(E[h,s,s2]))
//
// Both reproduce kernel_eval (kernel.cc:32-65) exactly in the exact modes:
// ops in double with round-to-nearest intrinsics, rounded to the storage
// type; the row fold runs in the odometer's order (index 0..L-1), each row
// owned by one thread that walks a coalesced smem-transposed tile.
#include <cuda_bf16.h>

#include "ewise.h"

namespace ed {

namespace {

template <typename T> __device__ __forceinline__ T rnd(double v);
template <> __device__ __forceinline__ float rnd<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double rnd<double>(double v) { return v; }

// ops.cc:5-38 in double (exact modes)
__device__ __forceinline__ double join_x(int op, double x, double y, int* err) {
  switch (op) {
    case 0: return __dmul_rn(x, y);
    case 1: return __dadd_rn(x, y);
    case 2: return __dsub_rn(x, y);
    case 3:
      if (y == 0.0) {
        atomicExch(err, 1);
        return 0.0;
      }
      return __ddiv_rn(x, y);
    case 4: {
      double d = __dsub_rn(x, y);
      return __dmul_rn(d, d);
    }
    default: return fabs(__dsub_rn(x, y));
  }
}
__device__ __forceinline__ double map_x(int op, double c, double x) {
  switch (op) {
    case 0: return x > 0.0 ? x : 0.0;
    case 1: return exp(x);
    case 2: return -x;
    case 3: return __dmul_rn(c, x);
    default: return x;
  }
}
// the same in float (tensor-core modes, tolerance-bound)
__device__ __forceinline__ float join_f(int op, float x, float y, int* err) {
  switch (op) {
    case 0: return __fmul_rn(x, y);
    case 1: return __fadd_rn(x, y);
    case 2: return __fsub_rn(x, y);
    case 3:
      if (y == 0.0f) {
        atomicExch(err, 1);
        return 0.0f;
      }
      return __fdiv_rn(x, y);
    case 4: {
      float d = __fsub_rn(x, y);
      return __fmul_rn(d, d);
    }
    default: return fabsf(__fsub_rn(x, y));
  }
}
__device__ __forceinline__ float map_f(int op, float c, float x) {
  switch (op) {
    case 0: return x > 0.0f ? x : 0.0f;
    case 1: return expf(x);
    case 2: return -x;
    case 3: return __fmul_rn(c, x);
    default: return x;
  }
}

template <typename T, bool kExact>
__device__ __forceinline__ T apply(const EwiseParams& p, T x, T y) {
  if (kExact || sizeof(T) == 8) {
    double v = p.binary ? join_x(p.join, double(x), double(y), p.err) : map_x(p.map, p.c, double(x));
    return rnd<T>(v);
  } else {
    return T(p.binary ? join_f(p.join, float(x), float(y), p.err) : map_f(p.map, float(p.c), float(x)));
  }
}

template <typename T, bool kExact>
__global__ void __launch_bounds__(256) ewise_kernel(const EwiseParams p) {
  const JoinPtrs jp = p.joins[blockIdx.y];
  const T* __restrict__ x = static_cast<const T*>(jp.x);
  const T* __restrict__ y = static_cast<const T*>(jp.y);
  T* __restrict__ out = static_cast<T*>(jp.out);
  __nv_bfloat16* o16 = static_cast<__nv_bfloat16*>(jp.out16);
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  const int64_t nvec = p.n / V;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < nvec; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = v * V;
    T xv[V], yv[V], r[V];
    *reinterpret_cast<uint4*>(xv) = __ldcs(reinterpret_cast<const uint4*>(x + o));
    if (p.binary) {
      if (p.y_mode == 1) {
        *reinterpret_cast<uint4*>(yv) = __ldcs(reinterpret_cast<const uint4*>(y + o));
      } else {  // broadcast: y index = o / inner (inner % V == 0 keeps it uniform)
        const T yy = y[o / p.inner];
#pragma unroll
        for (int i = 0; i < V; ++i) yv[i] = yy;
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) r[i] = apply<T, kExact>(p, xv[i], p.binary ? yv[i] : T(0));
    if (out) __stcs(reinterpret_cast<uint4*>(out + o), *reinterpret_cast<uint4*>(r));
    if (o16) {
#pragma unroll
      for (int i = 0; i < V; ++i) o16[o + i] = __double2bfloat16(double(r[i]));
    }
  }
  // scalar tail
  for (int64_t o = nvec * V + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < p.n;
       o += int64_t(gridDim.x) * blockDim.x) {
    const T yy = p.binary ? (p.y_mode == 1 ? y[o] : y[o / p.inner]) : T(0);
    const T r = apply<T, kExact>(p, x[o], yy);
    if (out) out[o] = r;
    if (o16) o16[o] = __double2bfloat16(double(r));
  }
}

// 32 rows per block; tiles of 32 rows x TC columns are loaded coalesced into
// smem by all 8 warps, then each of warp 0's lanes folds its row in order.
template <typename T, bool kExact>
__global__ void __launch_bounds__(256) rowreduce_kernel(const RowReduceParams p) {
  constexpr int R = 32;
  constexpr int TC = sizeof(T) == 4 ? 128 : 64;
  __shared__ T tile[2][R][TC + 1];
  const JoinPtrs jp = p.joins[blockIdx.y];
  const T* __restrict__ x = static_cast<const T*>(jp.x);
  T* out = static_cast<T*>(jp.out);
  __nv_bfloat16* o16 = static_cast<__nv_bfloat16*>(jp.out16);
  const int64_t row0 = int64_t(blockIdx.x) * R;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t L = p.len;
  const int ntiles = int((L + TC - 1) / TC);
  double acc = 0.0;
  auto load = [&](int t, int b) {
    // warp w loads rows w, w+8, w+16, w+24 of the tile
    const int64_t c0 = int64_t(t) * TC;
    for (int rr = warp; rr < R; rr += 8) {
      const int64_t row = row0 + rr;
      for (int c = lane; c < TC; c += 32) {
        T v = T(0);
        if (row < p.rows && c0 + c < L) v = x[row * L + c0 + c];
        tile[b][rr][c] = v;
      }
    }
  };
  load(0, 0);
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles && warp > 0) {
      // warps 1..7 prefetch the next tile while warp 0 folds this one
      const int64_t c0 = int64_t(t + 1) * TC;
      for (int rr = warp - 1; rr < R; rr += 7) {
        const int64_t row = row0 + rr;
        for (int c = lane; c < TC; c += 32) {
          T v = T(0);
          if (row < p.rows && c0 + c < L) v = x[row * L + c0 + c];
          tile[(t + 1) & 1][rr][c] = v;
        }
      }
    }
    if (warp == 0) {
      const int n = int(L - int64_t(t) * TC < TC ? L - int64_t(t) * TC : TC);
      for (int c = 0; c < n; ++c) {
        const T xv = tile[t & 1][lane][c];
        double v;
        if (kExact || sizeof(T) == 8) v = double(rnd<T>(map_x(p.map, p.c, double(xv))));
        else v = double(map_f(p.map, float(p.c), float(xv)));
        if (t == 0 && c == 0) acc = v;
        else if (p.agg == 0) acc = kExact || sizeof(T) == 8 ? double(rnd<T>(__dadd_rn(acc, v))) : double(float(acc) + float(v));
        else acc = acc < v ? v : acc;
      }
    }
    __syncthreads();
  }
  if (warp == 0 && row0 + lane < p.rows) {
    if (out) out[row0 + lane] = rnd<T>(acc);
    if (o16) o16[row0 + lane] = __double2bfloat16(acc);
  }
}

int blocks_for(int64_t work, int per_block, int joins) {
  int64_t b = (work + per_block - 1) / per_block;
  const int64_t cap = (148 * 8 + joins - 1) / joins;  // ~8 CTAs per SM across the launch
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

cudaError_t launch_ewise(const EwiseParams& p, int n_joins, bool f64, bool exact, cudaStream_t s) {
  dim3 grid(blocks_for(p.n / (f64 ? 2 : 4), 256, n_joins), n_joins);
  if (f64) ewise_kernel<double, true><<<grid, 256, 0, s>>>(p);
  else if (exact) ewise_kernel<float, true><<<grid, 256, 0, s>>>(p);
  else ewise_kernel<float, false><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_rowreduce(const RowReduceParams& p, int n_joins, bool f64, bool exact, cudaStream_t s) {
  dim3 grid(unsigned((p.rows + 31) / 32), n_joins);
  if (f64) rowreduce_kernel<double, true><<<grid, 256, 0, s>>>(p);
  else if (exact) rowreduce_kernel<float, true><<<grid, 256, 0, s>>>(p);
  else rowreduce_kernel<float, false><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ed
