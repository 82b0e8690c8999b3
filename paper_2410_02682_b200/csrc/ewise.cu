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

#include "libm_exp.cuh"
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
    case 1: return libm_exp(x);  // the host's std::exp bit for bit (ops.cc:24)
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
    if (!kExact && sizeof(T) == 4 && p.binary && p.join == 3 && p.y_mode == 2) {
      // broadcast divide (softmax normalisation): one reciprocal per vector
      if (yv[0] == T(0)) atomicExch(p.err, 1);
      const float inv = __frcp_rn(float(yv[0]));
#pragma unroll
      for (int i = 0; i < V; ++i) r[i] = T(__fmul_rn(float(xv[i]), inv));
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) r[i] = apply<T, kExact>(p, xv[i], p.binary ? yv[i] : T(0));
    }
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

// Order-free folds (max in every mode, sum in the tensor-core modes): one
// warp per row, 16-byte loads, shuffle tree.
template <typename T, bool kExact>
__global__ void __launch_bounds__(256) rowreduce_warp_kernel(const RowReduceParams p) {
  const JoinPtrs jp = p.joins[blockIdx.y];
  const T* __restrict__ x = static_cast<const T*>(jp.x);
  T* out = static_cast<T*>(jp.out);
  __nv_bfloat16* o16 = static_cast<__nv_bfloat16*>(jp.out16);
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x % 32;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  const bool vec = p.len % V == 0;
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; row < p.rows; row += warps) {
    const T* xr = x + row * p.len;
    double acc = 0.0;
    bool any = false;
    auto fold = [&](T xv) {
      double v;
      if (kExact || sizeof(T) == 8) v = double(rnd<T>(map_x(p.map, p.c, double(xv))));
      else v = double(map_f(p.map, float(p.c), float(xv)));
      if (!any) acc = v;
      else acc = p.agg == 0 ? double(float(acc) + float(v)) : (acc < v ? v : acc);
      any = true;
    };
    if (vec) {
      for (int64_t i = int64_t(lane) * V; i < p.len; i += 32 * V) {
        T xv[V];
        *reinterpret_cast<uint4*>(xv) = __ldcs(reinterpret_cast<const uint4*>(xr + i));
#pragma unroll
        for (int e = 0; e < V; ++e) fold(xv[e]);
      }
    } else {
      for (int64_t i = lane; i < p.len; i += 32) fold(xr[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double other = __shfl_xor_sync(0xffffffffu, acc, o);
      bool other_any = __shfl_xor_sync(0xffffffffu, any, o);
      if (other_any) {
        if (!any) acc = other;
        else acc = p.agg == 0 ? double(float(acc) + float(other)) : (acc < other ? other : acc);
        any = true;
      }
    }
    if (lane == 0) {
      if (out) out[row] = rnd<T>(acc);
      if (o16) o16[row] = __double2bfloat16(acc);
    }
  }
}

// Exact-order sums (the fp32/fp64 modes): each thread owns a row and folds it
// in odometer order (index 0..L-1) from coalesced smem-transposed tiles of
// 128 rows x 32 columns.
template <typename T>
__global__ void __launch_bounds__(128) rowreduce_seq_kernel(const RowReduceParams p) {
  constexpr int R = 128, TC = 32;
  __shared__ T tile[R][TC + 1];
  const JoinPtrs jp = p.joins[blockIdx.y];
  const T* __restrict__ x = static_cast<const T*>(jp.x);
  T* out = static_cast<T*>(jp.out);
  __nv_bfloat16* o16 = static_cast<__nv_bfloat16*>(jp.out16);
  const int64_t row0 = int64_t(blockIdx.x) * R;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t L = p.len;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < L; c0 += TC) {
    for (int rr = warp; rr < R; rr += 4) {
      const int64_t row = row0 + rr;
      T v = T(0);
      if (row < p.rows && c0 + lane < L) v = x[row * L + c0 + lane];
      tile[rr][lane] = v;
    }
    __syncthreads();
    const int n = int(L - c0 < TC ? L - c0 : TC);
    for (int c = 0; c < n; ++c) {
      const double v = double(rnd<T>(map_x(p.map, p.c, double(tile[threadIdx.x][c]))));
      acc = (c0 == 0 && c == 0) ? v : (p.agg == 0 ? double(rnd<T>(__dadd_rn(acc, v))) : (acc < v ? v : acc));
    }
    __syncthreads();
  }
  const int64_t row = row0 + threadIdx.x;
  if (row < p.rows) {
    if (out) out[row] = rnd<T>(acc);
    if (o16) o16[row] = __double2bfloat16(acc);
  }
}

// One block of NT threads per row; the row lives in registers (EPT per
// thread), so X is read once and Y written once (the five unfused vertices
// move the row eight times). Long rows use 256 threads so a thread holds at
// most 32 values and more rows are in flight per SM.
template <int EPT, int NT>
__global__ void __launch_bounds__(NT) softmax_kernel(const SoftmaxParams p) {
  constexpr int NV = EPT / 4;
  constexpr int NW = NT / 32;
  __shared__ float red[NW];
  const JoinPtrs jp = p.joins[blockIdx.y];
  const int t = threadIdx.x, lane = t % 32, warp = t / 32;
  auto block_reduce = [&](float v, bool is_max) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, w) : v + w;
    }
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = red[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) r = is_max ? fmaxf(r, red[i]) : r + red[i];
    __syncthreads();
    return r;
  };
  for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
    const float* xr = static_cast<const float*>(jp.x) + row * p.len;
    const RowSeg* sg = p.segs ? p.segs + size_t(blockIdx.y) * p.n_seg : nullptr;
    float v[EPT];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = (j * NT + t) * 4;
      const float* src = xr + i;
      if (sg && i < p.len) {  // gather the row from its column segments in place (past the row: no segment)
        const RowSeg s = sg[i / p.seg_w];
        src = s.ptr + (row + s.row0) * s.stride + (i % p.seg_w);
      }
      float4 q = i < p.len ? __ldcs(reinterpret_cast<const float4*>(src)) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      v[4 * j] = q.x;
      v[4 * j + 1] = q.y;
      v[4 * j + 2] = q.z;
      v[4 * j + 3] = q.w;
#pragma unroll
      for (int e = 0; e < 4; ++e) mx = fmaxf(mx, v[4 * j + e]);
    }
    if (jp.y) mx = static_cast<const float*>(jp.y)[row];  // the planned row max, computed upstream
    else mx = block_reduce(mx, true);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = (j * NT + t) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[4 * j + e] = i < p.len ? __expf(v[4 * j + e] - mx) : 0.f;
        sum += v[4 * j + e];
      }
    }
    sum = block_reduce(sum, false);
    const float inv = __frcp_rn(sum);
    float* yo = jp.out ? static_cast<float*>(jp.out) + row * p.len : nullptr;
    __nv_bfloat16* y16 = jp.out16 && !p.lo ? static_cast<__nv_bfloat16*>(jp.out16) + row * p.len : nullptr;
    float* ylo = jp.out16 && p.lo ? static_cast<float*>(jp.out16) + row * p.len : nullptr;
    auto lo_of = [](float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); };
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = (j * NT + t) * 4;
      if (i >= p.len) continue;
      const float a = v[4 * j] * inv, b = v[4 * j + 1] * inv, c = v[4 * j + 2] * inv, d = v[4 * j + 3] * inv;
      if (yo) __stcs(reinterpret_cast<float4*>(yo + i), make_float4(a, b, c, d));
      if (ylo) __stcs(reinterpret_cast<float4*>(ylo + i), make_float4(lo_of(a), lo_of(b), lo_of(c), lo_of(d)));
      if (y16) {
        __nv_bfloat162 h0 = __floats2bfloat162_rn(a, b), h1 = __floats2bfloat162_rn(c, d);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(y16 + i) = w;
      }
    }
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

cudaError_t launch_softmax(const SoftmaxParams& p, int n_joins, cudaStream_t s) {
  const unsigned rows = unsigned(p.rows < 65535 * 8 ? p.rows : 65535 * 8);
  dim3 grid(rows, n_joins);
  if (p.len <= 128 * 8) softmax_kernel<8, 128><<<grid, 128, 0, s>>>(p);
  else if (p.len <= 128 * 16) softmax_kernel<16, 128><<<grid, 128, 0, s>>>(p);
  else if (p.len <= 128 * 32) softmax_kernel<32, 128><<<grid, 128, 0, s>>>(p);
  else if (p.len <= 256 * 32) softmax_kernel<32, 256><<<grid, 256, 0, s>>>(p);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_rowreduce(const RowReduceParams& p, int n_joins, bool f64, bool exact, cudaStream_t s) {
  if ((exact || f64) && p.agg == 0) {
    dim3 grid(unsigned((p.rows + 127) / 128), n_joins);
    if (f64) rowreduce_seq_kernel<double><<<grid, 128, 0, s>>>(p);
    else rowreduce_seq_kernel<float><<<grid, 128, 0, s>>>(p);
  } else {
    dim3 grid(blocks_for(p.rows, 8, n_joins), n_joins);
    if (f64) rowreduce_warp_kernel<double, true><<<grid, 256, 0, s>>>(p);
    else if (exact) rowreduce_warp_kernel<float, true><<<grid, 256, 0, s>>>(p);
    else rowreduce_warp_kernel<float, false><<<grid, 256, 0, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace ed
