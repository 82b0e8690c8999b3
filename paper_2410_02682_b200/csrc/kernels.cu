// Exact-semantics CUDA-core kernels: the generic inner EinSum, the
// refinement fold, chunk scatter/gather and dtype conversion.
//
// Arithmetic follows ops.cc:5-38 in double with round-to-nearest intrinsics
// (no FMA contraction), then rounds to the storage type. For f32 storage
// this is exactly the reference's f32 mode (every operand and result
// rounded through float, kernel.cc:43-44; runtime.cc:257-259): double has
// more than 2*24+2 bits, so rounding an exact-in-double result of + - * /
// to float equals the correctly rounded float op. For f64 storage it is
// the reference's default mode bit for bit.
#include <cuda_bf16.h>

#include "libm_exp.cuh"
#include "kernels.h"

namespace ed {

namespace {

// x - tf32(x): the fp32 "lo" shadow an fp32x3 contraction reads beside x
__device__ __forceinline__ float lo_f(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <typename T> __device__ __forceinline__ T from_d(double v);
template <> __device__ __forceinline__ float from_d<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double from_d<double>(double v) { return v; }

__device__ __forceinline__ double join_d(int op, double x, double y, int* err) {
  switch (op) {
    case 0: return __dmul_rn(x, y);
    case 1: return __dadd_rn(x, y);
    case 2: return __dsub_rn(x, y);
    case 3:
      if (y == 0.0) {
        atomicExch(err, 1);  // eval_error_t("division by zero"), ops.cc:10-14
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

__device__ __forceinline__ double map_d(int op, double c, double x) {
  switch (op) {
    case 0: return x > 0.0 ? x : 0.0;
    case 1: return libm_exp(x);  // the host's std::exp bit for bit (ops.cc:24)
    case 2: return -x;
    case 3: return __dmul_rn(c, x);
    default: return x;
  }
}

__device__ __forceinline__ double agg_d(int op, double acc, double v) {
  // sum / std::max(acc, v) (ops.cc:31-36)
  return op == 0 ? __dadd_rn(acc, v) : (acc < v ? v : acc);
}

template <typename T>
__global__ void generic_kernel(const GenericParams p) {
  const T* x = static_cast<const T*>(p.x);
  const T* y = static_cast<const T*>(p.y);
  T* out = static_cast<T*>(p.out);
  __nv_bfloat16* o16 = static_cast<__nv_bfloat16*>(p.out16);
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < p.n_out;
       o += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = o, xo = 0, yo = 0;
    for (int d = p.nz - 1; d >= 0; --d) {
      int64_t c = rem % p.zext[d];
      rem /= p.zext[d];
      xo += c * p.xs_z[d];
      yo += c * p.ys_z[d];
    }
    int64_t a[kMaxRank];
    int64_t total = 1;
    for (int d = 0; d < p.na; ++d) {
      a[d] = 0;
      total *= p.aext[d];
    }
    double acc = 0.0;
    for (int64_t t = 0; t < total; ++t) {
      double v;
      if (y) v = join_d(p.join, double(x[xo]), double(y[yo]), p.err);
      else v = map_d(p.map, p.c, double(x[xo]));
      v = double(from_d<T>(v));
      acc = t == 0 ? v : double(from_d<T>(agg_d(p.agg, acc, v)));
      for (int d = p.na - 1; d >= 0; --d) {
        xo += p.xs_a[d];
        yo += p.ys_a[d];
        if (++a[d] < p.aext[d]) break;
        xo -= p.xs_a[d] * p.aext[d];
        yo -= p.ys_a[d] * p.aext[d];
        a[d] = 0;
      }
    }
    if (out) out[o] = from_d<T>(acc);
    if (o16) o16[o] = __double2bfloat16(acc);
  }
}

template <typename T>
__global__ void refine_kernel(const RefineParams p) {
  __shared__ DepRect deps[kMaxDeps];
  for (int i = threadIdx.x; i < p.n_deps; i += blockDim.x) deps[i] = p.deps[i];
  __syncthreads();
  T* out = static_cast<T*>(p.out);
  __nv_bfloat16* o16 = p.lo ? nullptr : static_cast<__nv_bfloat16*>(p.out16);
  float* olo = p.lo ? static_cast<float*>(p.out16) : nullptr;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < p.n_out;
       o += int64_t(gridDim.x) * blockDim.x) {
    int64_t g[kMaxRank];
    int64_t rem = o;
    for (int d = p.rank - 1; d >= 0; --d) {
      g[d] = p.c0[d] + rem % p.cext[d];
      rem /= p.cext[d];
    }
    double acc = 0.0;
    bool touched = false;
    for (int k = 0; k < p.n_deps; ++k) {
      const DepRect& r = deps[k];
      int64_t off = 0;
      bool in = true;
      for (int d = 0; d < p.rank; ++d) {
        int64_t l = g[d] - r.r0[d];
        in = in && l >= 0 && l < r.ext[d];
        off = off * r.ext[d] + l;
      }
      if (!in) continue;
      double v = double(static_cast<const T*>(r.src)[off]);
      acc = touched ? double(from_d<T>(agg_d(p.agg, acc, v))) : v;
      touched = true;
    }
    if (out) out[o] = from_d<T>(acc);
    if (o16) o16[o] = __double2bfloat16(acc);
    if (olo) olo[o] = lo_f(__double2float_rn(acc));
  }
}

template <typename T>
__global__ void __launch_bounds__(256) rect_kernel(const RectParams p) {
  const RectGroup& g = p.groups[blockIdx.y];
  T* out = static_cast<T*>(p.out);
  __nv_bfloat16* o16 = p.lo ? nullptr : static_cast<__nv_bfloat16*>(p.out16);
  float* olo = p.lo ? static_cast<float*>(p.out16) : nullptr;
  const int r = p.rank;
  constexpr int V = 16 / sizeof(T);
  const int W = p.vec ? V : 1;                      // elements per slot
  const int64_t per_row = g.ext[r - 1] / W;         // slots per row
  const int64_t r_begin = int64_t(blockIdx.x) * p.rows_per_block;
  if (r_begin >= g.rows) return;
  const int64_t r_end = r_begin + p.rows_per_block < g.rows ? r_begin + p.rows_per_block : g.rows;
  const int64_t slots = (r_end - r_begin) * per_row;
  for (int64_t sl = threadIdx.x; sl < slots; sl += blockDim.x) {
    const int64_t row = r_begin + sl / per_row;
    const int64_t i = (sl % per_row) * W;
    int64_t rem = row, so = g.src_off + i, dofs = g.dst_off + i;
    for (int d = r - 2; d >= 0; --d) {
      const int64_t c = rem % g.ext[d];
      rem /= g.ext[d];
      so += c * g.sstr[d];
      dofs += c * g.dstr[d];
    }
    if (p.vec) {
      T acc[V], v[V];
      *reinterpret_cast<uint4*>(acc) = *reinterpret_cast<const uint4*>(static_cast<const T*>(g.src[0]) + so);
      for (int k = 1; k < g.n_src; ++k) {
        *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(static_cast<const T*>(g.src[k]) + so);
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = from_d<T>(agg_d(p.agg, double(acc[e]), double(v[e])));
      }
      if (out) *reinterpret_cast<uint4*>(out + dofs) = *reinterpret_cast<uint4*>(acc);
      if (o16) {
#pragma unroll
        for (int e = 0; e < V; ++e) o16[dofs + e] = __double2bfloat16(double(acc[e]));
      }
      if (olo) {
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(olo + dofs) =
              make_float4(lo_f(float(acc[0])), lo_f(float(acc[1])), lo_f(float(acc[2])), lo_f(float(acc[3])));
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) olo[dofs + e] = lo_f(float(acc[e]));
        }
      }
    } else {
      double acc = double(static_cast<const T*>(g.src[0])[so]);
      for (int k = 1; k < g.n_src; ++k)
        acc = double(from_d<T>(agg_d(p.agg, acc, double(static_cast<const T*>(g.src[k])[so]))));
      if (out) out[dofs] = from_d<T>(acc);
      if (o16) o16[dofs] = __double2bfloat16(acc);
      if (olo) olo[dofs] = lo_f(__double2float_rn(acc));
    }
  }
}

template <typename T> __device__ __forceinline__ double ld(const void* p, int64_t i) {
  return double(static_cast<const T*>(p)[i]);
}
__device__ __forceinline__ double ld_dt(const void* p, int dt, int64_t i) {
  if (dt == 0) return ld<double>(p, i);
  if (dt == 1) return ld<float>(p, i);
  return double(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
}
__device__ __forceinline__ void st_dt(void* p, int dt, int64_t i, double v) {
  if (dt == 0) static_cast<double*>(p)[i] = v;
  else if (dt == 1) static_cast<float*>(p)[i] = __double2float_rn(v);
  else static_cast<__nv_bfloat16*>(p)[i] = __double2bfloat16(v);
}

__global__ void scatter_kernel(const ChunkMapParams p, const void* whole, int in_dt, int st_dt_) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < p.n;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = i, key = 0, loc = 0, kmul = 1, lmul = 1;
    for (int d = p.rank - 1; d >= 0; --d) {
      int64_t c = rem % p.bound[d];
      rem /= p.bound[d];
      key += (c / p.cb[d]) * kmul;
      loc += (c % p.cb[d]) * lmul;
      kmul *= p.part[d];
      lmul *= p.cb[d];
    }
    if (!p.chunks[key]) continue;  // chunk lives on another rank
    double v = ld_dt(whole, in_dt, i);
    st_dt(p.chunks[key], st_dt_, loc, v);
    if (p.shadows && p.shadows[key]) st_dt(p.shadows[key], 2, loc, v);
  }
}

__global__ void gather_kernel(const ChunkMapParams p, void* whole, int st_dt_, int out_dt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < p.n;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = i, key = 0, loc = 0, kmul = 1, lmul = 1;
    for (int d = p.rank - 1; d >= 0; --d) {
      int64_t c = rem % p.bound[d];
      rem /= p.bound[d];
      key += (c / p.cb[d]) * kmul;
      loc += (c % p.cb[d]) * lmul;
      kmul *= p.part[d];
      lmul *= p.cb[d];
    }
    st_dt(whole, out_dt, i, ld_dt(p.chunks[key], st_dt_, loc));
  }
}

// A rectangle flattened into (row, slot) pairs spread over every thread of the
// group's blocks: 16-byte slots when the runs allow it. (One row per block
// left 7 of every 8 threads idle on 128-float runs: hoc's 1 GiB input chunking
// took ~18 ms.)
__global__ void __launch_bounds__(256) blockcopy_kernel(const BlockCopyParams p) {
  const BlockCopy& g = p.groups[blockIdx.y];
  const int r = p.rank;
  const int64_t inner = g.ext[r - 1];
  bool vec = p.in_dt == 1 && p.out_dt == 1 && !g.dst16 && inner % 4 == 0 && g.src_off % 4 == 0 && g.dst_off % 4 == 0;
  for (int d = 0; d < r - 1; ++d) vec = vec && g.sstr[d] % 4 == 0 && g.dstr[d] % 4 == 0;
  const int64_t per_row = vec ? inner / 4 : inner;
  const int64_t slots = g.rows * per_row;
  for (int64_t sl = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; sl < slots; sl += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = sl / per_row;
    const int64_t i = (sl - rem * per_row) * (vec ? 4 : 1);
    int64_t so = g.src_off + i, dofs = g.dst_off + i;
    for (int d = r - 2; d >= 0; --d) {
      const int64_t c = rem % g.ext[d];
      rem /= g.ext[d];
      so += c * g.sstr[d];
      dofs += c * g.dstr[d];
    }
    if (vec) {
      *reinterpret_cast<float4*>(static_cast<float*>(g.dst) + dofs) =
          __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(g.src) + so));
      continue;
    }
    const double v = ld_dt(g.src, p.in_dt, so);
    if (g.dst) st_dt(g.dst, p.out_dt, dofs, v);
    if (g.dst16) st_dt(g.dst16, 2, dofs, v);
  }
}

__global__ void convert_kernel(const void* src, int in_dt, void* dst, int out_dt, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    st_dt(dst, out_dt, i, ld_dt(src, in_dt, i));
}

__global__ void split_lo_kernel(const float4* __restrict__ x, float4* __restrict__ lo, int64_t n4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    float4 v = x[i], r;
    r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    lo[i] = r;
  }
}

__global__ void split_lo_tail(const float* x, float* lo, int64_t from, int64_t n) {
  for (int64_t i = from + threadIdx.x; i < n; i += blockDim.x)
    lo[i] = x[i] - __uint_as_float(__float_as_uint(x[i]) & 0xFFFFE000u);
}

__global__ void add_one_kernel(void* p, int dt) { st_dt(p, dt, 0, ld_dt(p, dt, 0) + 1.0); }

int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  // enough CTAs for 8 waves of 148 SMs; grid-stride loops cover the rest
  return int(g < 148 * 8 * 4 ? (g < 1 ? 1 : g) : 148 * 8 * 4);
}

}  // namespace

cudaError_t launch_generic(const GenericParams& p, bool f64, cudaStream_t s) {
  const int block = 256;
  if (f64) generic_kernel<double><<<grid_for(p.n_out, block), block, 0, s>>>(p);
  else generic_kernel<float><<<grid_for(p.n_out, block), block, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_refine(const RefineParams& p, bool f64, cudaStream_t s) {
  const int block = 256;
  if (f64) refine_kernel<double><<<grid_for(p.n_out, block), block, 0, s>>>(p);
  else refine_kernel<float><<<grid_for(p.n_out, block), block, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_rect(const RectParams& p, int n_groups, int64_t max_rows, bool f64, cudaStream_t s) {
  dim3 grid(unsigned((max_rows + p.rows_per_block - 1) / p.rows_per_block), unsigned(n_groups));
  if (f64) rect_kernel<double><<<grid, 256, 0, s>>>(p);
  else rect_kernel<float><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const ChunkMapParams& p, const void* whole, DT in, DT store, cudaStream_t s) {
  scatter_kernel<<<grid_for(p.n, 256), 256, 0, s>>>(p, whole, int(in), int(store));
  return cudaGetLastError();
}

cudaError_t launch_gather(const ChunkMapParams& p, void* whole, DT store, DT out, cudaStream_t s) {
  gather_kernel<<<grid_for(p.n, 256), 256, 0, s>>>(p, whole, int(store), int(out));
  return cudaGetLastError();
}

cudaError_t launch_blockcopy(const BlockCopyParams& p, int n_groups, int64_t max_rows, cudaStream_t s) {
  // ~8 resident 256-thread blocks per SM across the launch; max_rows bounds a group's
  // rows (its slots are at most max_rows * 256 float-runs of up to 1024 elements)
  const int64_t per = (148 * 8 + n_groups - 1) / n_groups;
  const int64_t want = (max_rows * 64 + 255) / 256;  // >= 64 slots per row on typical runs
  dim3 grid(unsigned(want < per ? (want < 1 ? 1 : want) : per), unsigned(n_groups));
  blockcopy_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_convert(const void* src, DT in, void* dst, DT out, int64_t n, cudaStream_t s) {
  convert_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, int(in), dst, int(out), n);
  return cudaGetLastError();
}

cudaError_t launch_split_lo(const float* x, float* lo, int64_t n, cudaStream_t s) {
  const int64_t n4 = n / 4;
  if (n4) split_lo_kernel<<<grid_for(n4, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x),
                                                            reinterpret_cast<float4*>(lo), n4);
  if (n % 4) split_lo_tail<<<1, 32, 0, s>>>(x, lo, n4 * 4, n);
  return cudaGetLastError();
}

namespace {
constexpr int kMtN = 312, kMtM = 156;

// std::mt19937_64 (MT19937-64): x[k+312] = x[k+156] ^ ((x[k] & UM | x[k+1] & LM) >> 1) ^ (x[k+1] & 1 ? A : 0);
// output k = temper(x[312 + k]). The 312-word window lives in shared memory;
// each step, threads 0-155 make the next 156 words while threads 156-311
// temper, transform and store the 156 words made in the step before (they
// sit in the half of the window the current step does not overwrite).
__device__ __forceinline__ void gen_emit(const GenTensor& J, int64_t k, uint64_t y, int integer_valued, int store,
                                         int* err) {
  if (k >= J.n) return;
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  double v;
  if (integer_valued) {
    // _S_nd<unsigned __int128>(g, 9): product = g() * 9, reject if low < (-9) % 9 = 7
    if (y * 9ULL < 7ULL) atomicExch(err, 1);
    v = double(int64_t(__umul64hi(y, 9ULL)) - 4);
  } else {
    // generate_canonical<double, 53>: double(g()) / 2^64, clamped below 1; then u * (b - a) + a
    double u = __dmul_rn(__ull2double_rn(y), 0x1p-64);
    if (u >= 1.0) u = 0x1.fffffffffffffp-1;
    v = __dadd_rn(__dmul_rn(u, 2.0), -1.0);
  }
  if (store == int(DT::F64)) static_cast<double*>(J.out)[k] = v;
  else static_cast<float*>(J.out)[k] = __double2float_rn(v);
}

__global__ void __launch_bounds__(2 * kMtM) generate_kernel(const GenTensor* jobs, int integer_valued, int store,
                                                            int* err) {
  __shared__ uint64_t w[kMtN];
  const GenTensor J = jobs[blockIdx.x];
  const bool maker = threadIdx.x < kMtM;
  const int i = maker ? threadIdx.x : threadIdx.x - kMtM;
  if (threadIdx.x == 0) {  // init_genrand64: seeding is sequential
    uint64_t x = J.seed;
    w[0] = x;
    for (int k = 1; k < kMtN; ++k) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + uint64_t(k);
      w[k] = x;
    }
  }
  __syncthreads();
  int b = 0;  // w[b .. b+155] holds x[t .. t+155], w[b^156 ..] holds x[t+156 .. t+311]
  for (int64_t base = 0; base < J.n + kMtM; base += kMtM) {
    uint64_t nx = 0;
    if (maker) {
      const uint64_t a = w[b + i];
      const uint64_t a1 = i + 1 < kMtM ? w[b + i + 1] : w[(b ^ kMtM)];
      const uint64_t m = w[(b ^ kMtM) + i];
      const uint64_t x = (a & 0xFFFFFFFF80000000ULL) | (a1 & 0x7FFFFFFFULL);
      nx = m ^ (x >> 1) ^ ((a1 & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    } else if (base > 0) {
      // outputs base - 156 + i = x[t + 156 + i], made by the previous step
      gen_emit(J, base - kMtM + i, w[(b ^ kMtM) + i], integer_valued, store, err);
    }
    __syncthreads();
    if (maker) w[b + i] = nx;  // x[t+i] is dead once every thread has read it
    __syncthreads();
    b ^= kMtM;
  }
}

__global__ void peer_tick_kernel(int* epoch) { *epoch += 1; }
__global__ void peer_signal_kernel(int* flag, const int* epoch) {
  const int e = *epoch;
  __threadfence_system();
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(flag), "r"(e) : "memory");
}
struct PeerFlags {
  int* f[16];
};
__global__ void peer_wait_kernel(PeerFlags fl, int n, const int* epoch, int delta, int* err, int tag) {
  const int want = *epoch + delta;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < n; ++i) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(fl.f[i]) : "memory");
      if (v >= want) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {  // 20 s: report instead of hanging the stream
        if (err) atomicExch(err, 1 + tag * 64 + i);
        return;
      }
      __nanosleep(64);
    }
  }
}
}  // namespace

cudaError_t launch_generate(const GenTensor* jobs, int n_jobs, bool integer_valued, DT store, int* err,
                            cudaStream_t s) {
  generate_kernel<<<n_jobs, 2 * kMtM, 0, s>>>(jobs, int(integer_valued), int(store), err);
  return cudaGetLastError();
}

cudaError_t launch_peer_tick(int* epoch, cudaStream_t s) {
  peer_tick_kernel<<<1, 1, 0, s>>>(epoch);
  return cudaGetLastError();
}
cudaError_t launch_peer_signal(int* flag, const int* epoch, cudaStream_t s) {
  peer_signal_kernel<<<1, 1, 0, s>>>(flag, epoch);
  return cudaGetLastError();
}
cudaError_t launch_peer_wait(int* const* flags, int n, const int* epoch, int delta, cudaStream_t s, int* err,
                             int tag) {
  PeerFlags fl{};
  for (int done = 0; done < n; done += 16) {  // 16 flags per launch
    const int k = n - done < 16 ? n - done : 16;
    for (int i = 0; i < k; ++i) fl.f[i] = flags[done + i];
    peer_wait_kernel<<<1, 1, 0, s>>>(fl, k, epoch, delta, err, tag);
  }
  return cudaGetLastError();
}

cudaError_t launch_add_one(void* p, DT dt, cudaStream_t s) {
  add_one_kernel<<<1, 1, 0, s>>>(p, int(dt));
  return cudaGetLastError();
}

}  // namespace ed
