// Fused attention block: T1 = QK^T (+ fused scale), the five-vertex row
// softmax, and O = T3 V — three einsums of the plan executed as one tcgen05
// kernel per (region, head, 128-row tile), so the [h, s, s2] logits and
// probabilities never reach HBM.
//
// Per job: for each key block j, S_j = Q K_j^T (128 x 128 keys, TMEM); each
// column half h of the block keeps its own running reference max m_h and
// accumulates O_h += exp2(c*log2e*S_j - m_h) V_j in its own TMEM
// accumulator. A row's O_h is rescaled (TMEM read-modify-write) only when its
// max grows by more than 2^8, so P stays in bf16 range without a second
// pass. The halves merge in the epilogue: O = (O_0 2^(m_0-M) + O_1 2^(m_1-M)) / L.
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator and
// single-thread MMA issuer, warps 2-9 softmax and epilogue: two warps per
// TMEM lane quarter, each owning half of every key block's columns (row
// statistics merged once per job through smem); the epilogue goes TMEM ->
// swizzled smem (the warp's own rows of the P buffers) -> TMA store.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "attn_sm100.h"
#include "ptx.cuh"

namespace ed {

namespace {

constexpr int BQ = 128;   // query rows per job (TMEM lanes)
constexpr int BKV = 128;  // keys per block
constexpr int kThreads = 320;
constexpr int kSoftmaxWarps = 8;

template <int D>
struct ACfg {
  static constexpr int Q_BYTES = BQ * D * 2;   // D/64 K-major chunks of 16 KiB
  static constexpr int K_BYTES = BKV * D * 2;
  static constexpr int V_BYTES = BKV * D * 2;  // D/64 MN atoms of 128 key-rows x 128 B
  static constexpr int P_BYTES = BQ * BKV * 2; // 2 K-chunks of 16 KiB
  static constexpr int STAGE = K_BYTES + V_BYTES;
  static constexpr int SMEM = Q_BYTES + 2 * STAGE + 2 * P_BYTES + 1024 + 256;
  static constexpr int S_COL = 0;               // TMEM columns: S0 [0,128), S1 [128,256),
  static constexpr int O_COL = 2 * BKV;         // O_0 [256, 256+D), O_1 [256+D, 256+2D)
};

struct Job {
  int region, h, s0;
};

__device__ __forceinline__ Job job_of(const AttnLaunch& p, int j) {
  const int tiles = p.S / BQ;
  Job r;
  r.region = j / (p.H * tiles);
  int rem = j - r.region * p.H * tiles;
  r.h = rem / tiles;
  r.s0 = (rem % tiles) * BQ;
  return r;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(const __grid_constant__ AttnLaunch p) {
  using C_ = ACfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C_::Q_BYTES;                 // 2 stages of K then V
  uint8_t* sP = sKV + 2 * C_::STAGE;               // 2 P buffers
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * C_::P_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* kv_full = bar + 2;    // [2]
  uint64_t* kv_empty = bar + 4;   // [2]
  uint64_t* s_full = bar + 6;     // [2]
  uint64_t* s_empty = bar + 8;    // [2]
  uint64_t* p_full = bar + 10;    // [buffer][half]
  uint64_t* p_empty = bar + 14;   // [buffer][half]
  uint64_t* o_full = bar + 18;
  uint64_t* o_empty = bar + 19;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 20);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = p.T / BKV;
  const int jobs = p.n_regions * p.H * (p.S / BQ);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kSoftmaxWarps);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&p_full[i], kSoftmaxWarps / 2);
      mbar_init(&p_empty[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, kSoftmaxWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int it = 0, local = 0;
      for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x, ++local) {
        const Job J = job_of(p, jb);
        const AttnRegion R = p.regions[J.region];
        const CUtensorMap* mq = p.maps + R.q;
        auto src_map = [&](const AttnSrc& a, int key, int dcol) {
          return p.maps + a.base + (key / a.keys) * a.nd + dcol / a.dw;
        };
        mbar_wait(q_empty, (local & 1) ^ 1);
        mbar_expect_tx(q_full, C_::Q_BYTES);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tma_load_3d(sQ + c * 16384, mq, q_full, c * 64, J.s0, J.h);
        for (int j = 0; j < nb; ++j, ++it) {
          const int st = it & 1;
          mbar_wait(&kv_empty[st], ((it >> 1) & 1) ^ 1);
          uint8_t* sk = sKV + st * C_::STAGE;
          uint8_t* sv = sk + C_::K_BYTES;
          mbar_expect_tx(&kv_full[st], C_::STAGE);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sk + c * 16384, src_map(R.k, j * BKV, c * 64), &kv_full[st], (c * 64) % R.k.dw,
                        (j * BKV) % R.k.keys, J.h + R.k.hoff);
#pragma unroll
          for (int a = 0; a < D / 64; ++a)
            tma_load_3d(sv + a * (BKV * 128), src_map(R.v, j * BKV, a * 64), &kv_full[st], (a * 64) % R.v.dw,
                        (j * BKV) % R.v.keys, J.h + R.v.hoff);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc_s = umma_idesc(1u, BQ, BKV, 0u, 0u);  // Q, K both K-major (d)
      const uint32_t idesc_o = umma_idesc(1u, BQ, D, 0u, 1u);    // P K-major (keys), V MN-major (d)
      int it = 0, sc = 0, pc = 0, local = 0;
      auto issue_s = [&](int st) {
        const int sb = sc & 1;
        mbar_wait(&s_empty[sb], ((sc >> 1) & 1) ^ 1);
        mbar_wait(&kv_full[st], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ), ka = smem_u32(sKV + st * C_::STAGE);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k / 4) * 16384 + (k % 4) * 32;
          mma_f16(tmem + C_::S_COL + sb * BKV, umma_desc_sw128(qa + off, 16, 1024),
                  umma_desc_sw128(ka + off, 16, 1024), idesc_s, k != 0);
        }
        mma_commit(&s_full[sb]);
        ++sc;
      };
      for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x, ++local) {
        mbar_wait(q_full, local & 1);
        mbar_wait(o_empty, (local & 1) ^ 1);  // the last job's epilogue drained O_0, O_1
        tc_fence_after();
        const int it0 = it;
        issue_s(it0 & 1);
        for (int j = 0; j < nb; ++j) {
          const int st = (it0 + j) & 1;
          if (j + 1 < nb) {
            it = it0 + j + 1;
            issue_s(st ^ 1);
          }
          const int pb = pc & 1;
          const uint32_t pa = smem_u32(sP + pb * C_::P_BYTES);
          const uint32_t va = smem_u32(sKV + st * C_::STAGE + C_::K_BYTES);
          for (int h = 0; h < 2; ++h) {  // O_h += P_h V_h over the 64 keys of half h
            mbar_wait(&p_full[pb * 2 + h], (pc >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = umma_desc_sw128(pa + h * 16384 + k * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(va + (h * 4 + k) * 2048, BKV * 128, 1024);
              mma_f16(tmem + C_::O_COL + h * D, ad, bd, idesc_o, (j | k) != 0);
            }
            mma_commit(&p_empty[pb * 2 + h]);
          }
          mma_commit(&kv_empty[st]);
          ++pc;
        }
        it = it0 + nb;
        mma_commit(o_full);
        mma_commit(q_empty);
      }
    }
  } else {
    // ---------------- softmax + epilogue ----------------
    // warp w: TMEM lane quarter w % 4 (its rows), column half (w - 2) / 4
    const int wq = warp & 3, half = (warp - 2) / 4;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    const float sc2 = p.scale * 1.4426950408889634f;  // c * log2(e)
    auto ex2 = [](float x) {
      float y;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
      return y;
    };
    const uint32_t o_col = uint32_t(C_::O_COL + half * D);
    int sc = 0, pc = 0, local = 0;
    for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x, ++local) {
      const Job J = job_of(p, jb);
      const AttnRegion R = p.regions[J.region];
      float m = -INFINITY, l = 0.f;  // this half's reference max (log2 domain) and sum
      // my rows of the P buffers were staging for the last epilogue's stores
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      for (int j = 0; j < nb; ++j, ++sc, ++pc) {
        const int sb = sc & 1, pb = pc & 1;
        mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc_fence_after();
        uint32_t v[64];
        const uint32_t col = uint32_t(C_::S_COL + sb * BKV + half * 64);
        tmem_ld_32x32b_x32(tmem + lane_base + col, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld_32x32b_x32(tmem + lane_base + col + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < 64; ++e) mx = fmaxf(mx, __uint_as_float(v[e]) * sc2);
        if (j == 0) {
          m = mx;
        } else {
          const bool grow = mx > m + 8.0f;
          if (__any_sync(0xffffffffu, grow)) {
            // rescale this half's O rows once every earlier P V MMA is done
            const int pq = pc - 1;
            mbar_wait(&p_empty[(pq & 1) * 2 + half], (pq >> 1) & 1);
            tc_fence_after();
            const float f = grow ? ex2(m - mx) : 1.0f;
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(tmem + lane_base + o_col + uint32_t(c * 32), o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
              tmem_st_32x32b_x32(tmem + lane_base + o_col + uint32_t(c * 32), o);
            }
            tmem_st_wait();
            l *= f;
            if (grow) m = mx;
          }
        }
        uint32_t w[32];
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const float a = ex2(fmaf(__uint_as_float(v[2 * q]), sc2, -m));
          const float b = ex2(fmaf(__uint_as_float(v[2 * q + 1]), sc2, -m));
          acc += a + b;
          __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
          w[q] = *reinterpret_cast<uint32_t*>(&h2);
        }
        l += acc;
        mbar_wait(&p_empty[pb * 2 + half], ((pc >> 1) & 1) ^ 1);
        uint8_t* prow = sP + pb * C_::P_BYTES + half * 16384 + r * 128;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<uint4*>(prow + ((g ^ (r & 7)) << 4)) =
              make_uint4(w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb * 2 + half]);
      }
      // merge the halves' statistics through this warp's own rows of P buffer 0
      mbar_wait(o_full, local & 1);
      tc_fence_after();
      float f_own, f_other;
      {
        float* mine = reinterpret_cast<float*>(sP + half * 16384 + wq * 4096);
        const float* other = reinterpret_cast<const float*>(sP + (half ^ 1) * 16384 + wq * 4096);
        mine[lane] = m;
        mine[32 + lane] = l;
        asm volatile("bar.sync 1, %0;" ::"n"(kSoftmaxWarps * 32) : "memory");
        const float m2 = other[lane], l2 = other[32 + lane];
        asm volatile("bar.sync 1, %0;" ::"n"(kSoftmaxWarps * 32) : "memory");
        const float M = fmaxf(m, m2);
        const float L = l * ex2(m - M) + l2 * ex2(m2 - M);
        f_own = ex2(m - M) / L;
        f_other = ex2(m2 - M) / L;
      }
      const float f0 = half == 0 ? f_own : f_other, f1 = half == 0 ? f_other : f_own;
      // epilogue: this warp's half of O's columns, O_0 f0 + O_1 f1 -> staging in
      // its own rows of its own P K-chunk (free: every P V MMA has completed)
      uint8_t* tiles[2] = {sP + half * 16384 + wq * 4096, sP + C_::P_BYTES + half * 16384 + wq * 4096};
      int t_used = 0;
      for (int pass = 0; pass < 2; ++pass) {
        const int cm = pass == 0 ? R.o32 : R.o16;
        if (cm < 0) continue;
        const int cols = pass == 0 ? 32 : 64;
        const int per_half = (D / cols + 1) / 2;
#pragma unroll 1
        for (int ci = 0; ci < per_half; ++ci) {
          const int c = half * per_half + ci;
          if (c * cols >= D) break;
          uint32_t v[64];
          for (int part = 0; part < (pass == 0 ? 1 : 2); ++part) {
            uint32_t a0[32], a1[32];
            const uint32_t cc = uint32_t(c * cols + part * 32);
            tmem_ld_32x32b_x32(tmem + lane_base + uint32_t(C_::O_COL) + cc, a0);
            tmem_ld_32x32b_x32(tmem + lane_base + uint32_t(C_::O_COL + D) + cc, a1);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
              v[part * 32 + e] = __float_as_uint(__uint_as_float(a0[e]) * f0 + __uint_as_float(a1[e]) * f1);
          }
          if (t_used == 2) {  // recycle staging tiles
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            t_used = 0;
          }
          uint8_t* rowp = tiles[t_used++] + lane * 128;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            uint4 q4;
            if (pass == 0) {
              q4 = make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
            } else {
              __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(v[8 * g]), __uint_as_float(v[8 * g + 1]));
              __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(v[8 * g + 2]), __uint_as_float(v[8 * g + 3]));
              __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[8 * g + 4]), __uint_as_float(v[8 * g + 5]));
              __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(v[8 * g + 6]), __uint_as_float(v[8 * g + 7]));
              q4 = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                              *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
            }
            *reinterpret_cast<uint4*>(rowp + ((g ^ (lane & 7)) << 4)) = q4;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(p.maps + cm, tiles[t_used - 1], c * cols, J.s0 + wq * 32, J.h);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D>
cudaError_t launch_d(const AttnLaunch& p, int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<D>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int jobs = p.n_regions * p.H * (p.S / BQ);
  attn_kernel<D><<<jobs < num_sms ? jobs : num_sms, kThreads, ACfg<D>::SMEM, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t attn_prepare() {
  cudaError_t e = cudaFuncSetAttribute(attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<64>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<128>::SMEM);
}

bool attn_supported(int S, int T, int D) { return (D == 64 || D == 128) && S % BQ == 0 && T % BKV == 0 && T > 0; }

cudaError_t launch_attn(const AttnLaunch& p, int num_sms, cudaStream_t s) {
  if (p.D == 128) return launch_d<128>(p, num_sms, s);
  if (p.D == 64) return launch_d<64>(p, num_sms, s);
  return cudaErrorInvalidValue;
}

}  // namespace ed
