// Fused attention block: T1 = QK^T (+ fused scale), the five-vertex row
// softmax, and O = T3 V — three einsums of the plan executed as one tcgen05
// kernel, so the [h, s, s2] logits and probabilities never reach HBM.
//
// A job is a pair of 128-row query tiles of one head (or a single tile in
// the last wave, to fill the grid): K_j and V_j are loaded once per pair
// into a ring of shared-memory stages (K0, V0, K1, V1, ...).
//
// One thread issues every MMA in a fixed order,
//
//   S_0(0) S_1(0) | PV_0(0) S_0(1) PV_1(0) S_1(1) | PV_0(1) S_0(2) ...
//
// so while tile t's softmax works on S_t(j) the tensor pipe runs the other
// tile's P.V and next S. S_t = Q_t K_j^T lands in TMEM; the softmax warps of
// tile t read it (one thread per row), keep a reference max m (log2 domain),
// post the row's rescale factor to the correction warp of its rows through
// a named barrier, and write P = exp2(c log2e S - m) back over S as packed
// bf16; O_t += P V_j takes P straight from TMEM (the A-from-TMEM form of
// tcgen05.mma). P.V over the first 96 keys starts when three of P's four
// fragments are stored. The commit that signals S_t(j) also covers
// PV_t(j-1), so a rescale of O_t never races an MMA. O_t is rescaled only
// when a row max passes the reference by more than 2^64.
//
// Warp roles (512 threads): warps 0-3 softmax of tile 0, 4-7 of tile 1 (warp
// w owns TMEM lanes 32(w%4)..+32), 8-11 correction (O rescales, then the
// epilogue O / l -> swizzled smem -> TMA store, off the softmax's path),
// warp 12 TMEM allocator + MMA issuer, warp 13 TMA producer, 14-15 idle.
// setmaxnreg moves registers from the producer and correction warpgroups to
// the softmax warpgroups, so a thread holds its whole 128-key S row.
// TMEM: S/P_0 [0,128) S/P_1 [128,256) O_0 [256,256+D) O_1 [256+D,256+2D).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "attn_sm100.h"
#include "ptx.cuh"

namespace ed {

namespace {

constexpr int BQ = 128;   // query rows per tile (TMEM lanes)
constexpr int BKV = 128;  // keys per block
constexpr int kThreads = 512;  // four warpgroups
constexpr int kCorrWarp0 = 8, kMmaWarp = 12, kTmaWarp = 13;
// register split (setmaxnreg): 2 x 128 x 184 + 128 x 96 + 128 x 48 <= 64K
#ifndef ED_ATTN_SREGS
#define ED_ATTN_SREGS 184
#define ED_ATTN_PREGS 48
#define ED_ATTN_CREGS 96
#endif
constexpr int kSoftmaxRegs = ED_ATTN_SREGS, kProducerRegs = ED_ATTN_PREGS, kCorrectionRegs = ED_ATTN_CREGS;
// the softmax warpgroups can only take what the others give back from the
// launch allocation (65536 / threads per thread), or setmaxnreg.inc never returns
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;
static_assert(2 * (kSoftmaxRegs - kLaunchRegs) <= (kLaunchRegs - kProducerRegs) + (kLaunchRegs - kCorrectionRegs),
              "setmaxnreg split exceeds the launch allocation");
// lazy rescale (log2 units): P = 2^(x - m) may reach 2^kRescale before O is
// rescaled, and a rescale sets m = row max + kHeadroom. bf16 / fp32 keep full
// relative precision over that span; O = sum P V keeps 2^64 / 4096 of headroom
// for |V|, and keys more than ~2^-78 below the row max underflow to 0.
constexpr float kRescale = 64.0f, kHeadroom = 48.0f;
// exp2 pairs q with bit q % 8 set run on the FMA pipe (exp2_poly2), the rest on MUFU
// (attn_big: 1 of 8 on the FMA pipe 0.2378 ms, none 0.2390, 2 of 8 0.2482, 3 of 8 0.268)
#ifndef ED_ATTN_POLY
#define ED_ATTN_POLY 0x80
#endif
constexpr int kPolyPairs = ED_ATTN_POLY;
// P fragments (32 keys each) stored before P.V over them may start
#ifndef ED_ATTN_SPLIT
#define ED_ATTN_SPLIT 3
#endif
constexpr int kSplitFr = ED_ATTN_SPLIT;
static_assert(kSplitFr >= 1 && kSplitFr <= 3, "P.V starts after 1-3 of the 4 P fragments");

template <int D>
struct ACfg {
  static constexpr int Q_BYTES = BQ * D * 2;    // D/64 K-major chunks of 16 KiB
  static constexpr int KV_BYTES = BKV * D * 2;  // K: D/64 K-major chunks; V: D/64 MN atoms of 128 key-rows x 128 B
  static constexpr int KV_STAGES = D == 64 ? 6 : 3;
  static constexpr int STG_BYTES = 4096;        // per correction warp, two of them: 32 rows x 128 B
  static constexpr int SMEM = 2 * Q_BYTES + KV_STAGES * KV_BYTES + 8 * STG_BYTES + 1024 + 512 + 2048;
  static constexpr int TMEM_COLS = 512;
  __host__ __device__ static constexpr int s_col(int t) { return t * BKV; }
  __host__ __device__ static constexpr int o_col(int t) { return 2 * BKV + t * D; }
};
static_assert(ACfg<128>::SMEM <= 232448 && ACfg<64>::SMEM <= 232448, "shared memory");

struct Job {
  int region, h, s0, two;
};

// Jobs [0, n_pair) are tile pairs (2q, 2q+1) of a head; the remaining pair
// units are split into single tiles, then the odd last tile of every head.
__device__ __forceinline__ Job job_of(const AttnLaunch& p, int j) {
  const int tph = p.S / BQ, pph = tph / 2;
  const int units = p.n_regions * p.H * pph;
  int rh, tile, two;
  if (j < p.n_pair_jobs) {
    rh = j / pph;
    tile = 2 * (j % pph);
    two = 1;
  } else {
    const int s = j - p.n_pair_jobs, split = 2 * (units - p.n_pair_jobs);
    two = 0;
    if (s < split) {
      const int u = p.n_pair_jobs + s / 2;
      rh = u / pph;
      tile = 2 * (u % pph) + (s & 1);
    } else {
      rh = s - split;
      tile = tph - 1;
    }
  }
  Job r;
  r.region = rh / p.H;
  r.h = rh % p.H;
  r.s0 = tile * BQ;
  r.two = two;
  return r;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32x2 FMA-pipe ops (FFMA2 / FADD2): two lanes per instruction
__device__ __forceinline__ unsigned long long f2_bits(float2 a) {
  return (unsigned long long)__float_as_uint(a.x) | ((unsigned long long)__float_as_uint(a.y) << 32);
}
__device__ __forceinline__ float2 bits_f2(unsigned long long b) {
  return make_float2(__uint_as_float(uint32_t(b)), __uint_as_float(uint32_t(b >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}

// 2^x for two lanes without MUFU: x = j + r (j = rint(x) via the 1.5*2^23
// shifter, r in [-1/2, 1/2]), 2^r by a degree-3 minimax polynomial (max rel
// err 7.5e-5, far below the bf16 rounding P gets), j added to the exponent.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);  // keeps 2^j * p (p >= 2^-1/2) a normal number
  x.y = fmaxf(x.y, -125.f);
  const float2 sh = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 jf = fadd2(sh, make_float2(-12582912.f, -12582912.f));
  const float2 r = ffma2(jf, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(r, make_float2(0.055171654f, 0.055171654f), make_float2(0.24261114f, 0.24261114f));
  p = ffma2(p, r, make_float2(0.69326097f, 0.69326097f));
  p = ffma2(p, r, make_float2(0.99992806f, 0.99992806f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(sh.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(sh.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int D, int kPoly>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(const __grid_constant__ AttnLaunch p) {
  using C_ = ACfg<D>;
  constexpr int NS = C_::KV_STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                           // [2] tiles
  uint8_t* sKV = sQ + 2 * C_::Q_BYTES;          // [NS] ring: K0, V0, K1, V1, ...
  uint8_t* sStg = sKV + NS * C_::KV_BYTES;      // [4 correction warps][2] epilogue staging
  uint64_t* bar = reinterpret_cast<uint64_t*>(sStg + 8 * C_::STG_BYTES);
  uint64_t* q_full = bar + 0;     // [tile] TMA -> MMA
  uint64_t* q_empty = bar + 2;    // [tile] MMA -> TMA
  uint64_t* s_full = bar + 4;     // [tile] MMA -> softmax: S_t(j) in TMEM (and PV_t(j-1) done)
  uint64_t* p_part = bar + 6;     // [tile] softmax -> MMA: P over the first 3/4 of the keys stored
  uint64_t* p_full = bar + 8;     // [tile] softmax -> MMA: all of P stored
  uint64_t* o_ok = bar + 10;      // [tile] correction -> MMA: O_t rescaled for this block
  uint64_t* o_full = bar + 12;    // [tile] MMA -> correction: last PV_t of the job done
  uint64_t* o_empty = bar + 14;   // [tile] correction -> MMA: epilogue has read O_t
  uint64_t* l_ready = bar + 16;   // [tile] softmax -> correction: row sums of the job posted
  uint64_t* kv_full = bar + 18;   // [NS]
  uint64_t* kv_empty = bar + 18 + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18 + 2 * NS);
  float* scl = reinterpret_cast<float*>(bar + 20 + 2 * NS);  // [tile][row] rescale factor of the block
  float* lbuf = scl + 2 * BQ;                                // [tile][row] row sum of the job

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = p.T / BKV;
  const int jobs = p.n_jobs;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_part[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_ok[i], 4);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 4);
      mbar_init(&l_ready[i], 4);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc<C_::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // the prologue above overlapped the previous kernel (PDL)

  if (warp >= kCorrWarp0 && warp < kCorrWarp0 + 4) {
    // ---------------- correction warpgroup: O rescales and the epilogue ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCorrectionRegs));
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    uint8_t* stg = sStg + wq * 2 * C_::STG_BYTES;
    int ln[2] = {0, 0}, sb = 0;
    for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
      const Job J = job_of(p, jb);
      for (int j = 0; j < nb; ++j)
        for (int t = 0; t <= J.two; ++t) {
          named_sync(1 + t * 4 + wq, 64);  // the softmax warp of these rows posted its factor
          const float f = scl[t * BQ + row];
          if (__any_sync(0xffffffffu, f != 1.f)) {
            // PV_t(j-1) is complete: the softmax saw S_t(j), committed after it
            tc_fence_after();
            const float2 f2 = make_float2(f, f);
            const uint32_t o_addr = tmem + lane_base + uint32_t(C_::o_col(t));
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(o_addr + uint32_t(c * 32), o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float2 r = fmul2(make_float2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), f2);
                o[e] = __float_as_uint(r.x);
                o[e + 1] = __float_as_uint(r.y);
              }
              tmem_st_32x32b_x32(o_addr + uint32_t(c * 32), o);
            }
            tmem_st_wait();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&o_ok[t]);
        }
      // ---- epilogue: O_t / l -> swizzled staging -> TMA store (32 rows per warp)
      for (int t = 0; t <= J.two; ++t) {
        mbar_wait(&l_ready[t], ln[t] & 1);
        const float inv = 1.0f / lbuf[t * BQ + row];
        mbar_wait(&o_full[t], ln[t] & 1);  // both complete once per job of this tile
        ++ln[t];
        tc_fence_after();
        const uint32_t o_addr = tmem + lane_base + uint32_t(C_::o_col(t));
        const int row0 = J.s0 + t * BQ + wq * 32;
        for (int pass = 0; pass < 2; ++pass) {
          const int cm = pass == 0 ? p.regions[J.region].o32 : p.regions[J.region].o16;
          if (cm < 0) continue;
          const int cols = pass == 0 ? 32 : 64;
#pragma unroll 1
          for (int c = 0; c < D / cols; ++c) {
            uint32_t v[64];
            tmem_ld_32x32b_x32(o_addr + uint32_t(c * cols), *reinterpret_cast<uint32_t(*)[32]>(v));
            if (pass == 1) tmem_ld_32x32b_x32(o_addr + uint32_t(c * cols + 32), *reinterpret_cast<uint32_t(*)[32]>(v + 32));
            tmem_ld_wait();
            uint8_t* buf = stg + (sb & 1) * C_::STG_BYTES;
            if (lane == 0) bulk_wait_read<1>();  // the store that last read this buffer is done
            __syncwarp();
            uint8_t* rowp = buf + lane * 128;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              uint4 q4;
              if (pass == 0) {
                q4 = make_uint4(__float_as_uint(__uint_as_float(v[4 * g]) * inv),
                                __float_as_uint(__uint_as_float(v[4 * g + 1]) * inv),
                                __float_as_uint(__uint_as_float(v[4 * g + 2]) * inv),
                                __float_as_uint(__uint_as_float(v[4 * g + 3]) * inv));
              } else {
                q4 = make_uint4(pack_bf16(__uint_as_float(v[8 * g]) * inv, __uint_as_float(v[8 * g + 1]) * inv),
                                pack_bf16(__uint_as_float(v[8 * g + 2]) * inv, __uint_as_float(v[8 * g + 3]) * inv),
                                pack_bf16(__uint_as_float(v[8 * g + 4]) * inv, __uint_as_float(v[8 * g + 5]) * inv),
                                pack_bf16(__uint_as_float(v[8 * g + 6]) * inv, __uint_as_float(v[8 * g + 7]) * inv));
              }
              *reinterpret_cast<uint4*>(rowp + ((g ^ (lane & 7)) << 4)) = q4;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(p.maps + cm, buf, c * cols, row0, J.h);
              bulk_commit();
            }
            ++sb;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[t]);
      }
    }
    if (lane == 0) bulk_wait<0>();
  } else if (warp >= 12) {
    // producer warpgroup: hands registers to the softmax warpgroups
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    if (warp == kTmaWarp && lane == 0) {
      // ---------------- TMA producer: Q tiles, then the K/V ring K0 V0 K1 V1 ... ----------------
      int kvn = 0, qn0 = 0, qn1 = 0;
      for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
        if (jb + int(gridDim.x) >= jobs) griddep_launch();  // last job: the next kernel may launch
        const Job J = job_of(p, jb);
        const AttnRegion R = p.regions[J.region];
        const CUtensorMap* mq = p.maps + R.q;
        auto src_map = [&](const AttnSrc& a, int key, int dcol) {
          return p.maps + a.base + (key / a.keys) * a.nd + dcol / a.dw;
        };
        for (int t = 0; t <= J.two; ++t) {
          int& qn = t ? qn1 : qn0;
          mbar_wait(&q_empty[t], (qn & 1) ^ 1);
          ++qn;
          mbar_expect_tx(&q_full[t], C_::Q_BYTES);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sQ + t * C_::Q_BYTES + c * 16384, mq, &q_full[t], c * 64, J.s0 + t * BQ, J.h);
        }
        for (int j = 0; j < nb; ++j) {
          for (int kv = 0; kv < 2; ++kv) {
            const int st = kvn % NS;
            mbar_wait(&kv_empty[st], ((kvn / NS) & 1) ^ 1);
            ++kvn;
            mbar_expect_tx(&kv_full[st], C_::KV_BYTES);
            uint8_t* dst = sKV + st * C_::KV_BYTES;
            const AttnSrc& a = kv ? R.v : R.k;
#pragma unroll
            for (int c = 0; c < D / 64; ++c)
              tma_load_3d(dst + c * 16384, src_map(a, j * BKV, c * 64), &kv_full[st], (c * 64) % a.dw,
                          (j * BKV) % a.keys, J.h + a.hoff);
          }
        }
      }
    } else if (warp == kMmaWarp) {
      // ---------------- MMA issuer: PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) ----------------
      // The whole warp runs this loop (uniform values); one elected lane issues.
      // One thread, fixed order: each tile's P.V goes in as soon as its P is
      // stored, its next S right behind it (in issue order after the P.V that
      // reads P, so S may overwrite P's columns), while the other tile's
      // softmax works on its own S.
      const uint32_t idesc_s = umma_idesc(1u, BQ, BKV, 0u, 0u);  // Q, K both K-major (d)
      const uint32_t idesc_o = umma_idesc(1u, BQ, D, 0u, 1u);    // P from TMEM (keys), V MN-major (d)
      int kvn = 0, qn0 = 0, qn1 = 0, pn0 = 0, pn1 = 0, on0 = 0, on1 = 0;
      // Descriptors are built once per operand base; a K step adds its byte
      // offset / 16 to the start-address field (no carry below 256 KiB).
      // (attn_big: 0.2350 vs 0.2373 ms rebuilding them per MMA; TMEM
      // addresses as compile-time constants instead of the allocated base
      // measured slower still, 0.2434.)
      auto issue_s = [&](int t, int kst) {
        const uint64_t qd = umma_desc_sw128(smem_u32(sQ + t * C_::Q_BYTES), 16, 1024);
        const uint64_t kd = umma_desc_sw128(smem_u32(sKV + kst * C_::KV_BYTES), 16, 1024);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t off = uint64_t(((k / 4) * 16384 + (k % 4) * 32) >> 4);
          mma_f16_warp(tmem + C_::s_col(t), qd + off, kd + off, idesc_s, k != 0);
        }
        mma_commit_warp(&s_full[t]);
      };
      auto issue_pv = [&](int t, uint32_t va, int k0, int k1, bool fresh) {
        const uint64_t vd = umma_desc_sw128(va, BKV * 128, 1024);
#pragma unroll
        for (int k = k0; k < k1; ++k)
          mma_f16_ts_warp(tmem + C_::o_col(t), tmem + C_::s_col(t) + k * 8, vd + uint64_t((k * 2048) >> 4), idesc_o,
                          !(fresh && k == 0));
      };
      auto take = [&]() {  // next ring stage, full
        const int st = kvn % NS;
        mbar_wait(&kv_full[st], (kvn / NS) & 1);
        ++kvn;
        return st;
      };
      for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
        const Job J = job_of(p, jb);
        const int two = J.two;
        int kst = take();
        for (int t = 0; t <= two; ++t) {
          int& qn = t ? qn1 : qn0;
          mbar_wait(&q_full[t], qn & 1);
          ++qn;
          tc_fence_after();
          issue_s(t, kst);
          if (nb == 1) mma_commit_warp(&q_empty[t]);
        }
        mma_commit_warp(&kv_empty[kst]);
        for (int j = 0; j < nb; ++j) {
          const int vst = take();
          const uint32_t va = smem_u32(sKV + vst * C_::KV_BYTES);
          for (int t = 0; t <= two; ++t) {
            int& pn = t ? pn1 : pn0;
            if (j == 0) {  // the previous job's epilogue has read O_t
              int& on = t ? on1 : on0;
              mbar_wait(&o_empty[t], (on & 1) ^ 1);
              ++on;
            }
            mbar_wait(&o_ok[t], pn & 1);
            mbar_wait(&p_part[t], pn & 1);
            tc_fence_after();
            issue_pv(t, va, 0, kSplitFr * 2, j == 0);
            mbar_wait(&p_full[t], pn & 1);
            ++pn;
            tc_fence_after();
            issue_pv(t, va, kSplitFr * 2, BKV / 16, false);
            if (t == two) mma_commit_warp(&kv_empty[vst]);
            if (j == nb - 1) {
              mma_commit_warp(&o_full[t]);
            } else {
              if (t == 0) {
                kst = take();
                tc_fence_after();
              }
              issue_s(t, kst);
              if (j + 1 == nb - 1) mma_commit_warp(&q_empty[t]);
              if (t == two) mma_commit_warp(&kv_empty[kst]);
            }
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
    // ---------------- softmax (tile t = warp / 4, one thread per row) ----------------
    const int t = warp >> 2, wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + uint32_t(C_::s_col(t));
    const float sc2 = p.scale * 1.4426950408889634f;  // c * log2(e)
    int sn = 0;
    for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
      const Job J = job_of(p, jb);
      if (t > J.two) continue;
      float m = 0.f, l = 0.f;  // reference max (log2 domain) and row sum
      for (int j = 0; j < nb; ++j) {
        mbar_wait(&s_full[t], sn & 1);
        ++sn;
        tc_fence_after();
        uint32_t v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tmem_ld_32x32b_x32(s_addr + uint32_t(c * 32), *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
        tmem_ld_wait();
        // row max of c*log2e*S: four independent chains
        float mx;
        {
          float a0, a1, a2, a3;
          if (sc2 >= 0.f) {
            a0 = a1 = a2 = a3 = -INFINITY;
#pragma unroll
            for (int e = 0; e < 128; e += 4) {
              a0 = fmaxf(a0, __uint_as_float(v[e]));
              a1 = fmaxf(a1, __uint_as_float(v[e + 1]));
              a2 = fmaxf(a2, __uint_as_float(v[e + 2]));
              a3 = fmaxf(a3, __uint_as_float(v[e + 3]));
            }
            mx = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)) * sc2;
          } else {
            a0 = a1 = a2 = a3 = INFINITY;
#pragma unroll
            for (int e = 0; e < 128; e += 4) {
              a0 = fminf(a0, __uint_as_float(v[e]));
              a1 = fminf(a1, __uint_as_float(v[e + 1]));
              a2 = fminf(a2, __uint_as_float(v[e + 2]));
              a3 = fminf(a3, __uint_as_float(v[e + 3]));
            }
            mx = fminf(fminf(a0, a1), fminf(a2, a3)) * sc2;
          }
        }
        // reference max with hysteresis: when a row's max passes m + kRescale
        // the new reference is max + kHeadroom, so P spans [2^-kHeadroom,
        // 2^kRescale] at the row max and rescales stay rare
        float f = 1.f;
        if (j == 0) {
          m = mx + kHeadroom;
        } else if (mx > m + kRescale) {
          const float mn = mx + kHeadroom;
          f = ex2(m - mn);
          m = mn;
        }
        scl[t * BQ + row] = f;
        named_arrive(1 + t * 4 + wq, 64);  // the correction warp of these rows takes the factor
        // P = exp2(c log2e S - m), packed bf16 over S's first 64 columns, in
        // four fragments of 32 keys; the first three are published together
        // so P.V over 96 keys starts while the last fragment is computed
        const float2 sc2v = make_float2(sc2, sc2), nm = make_float2(-m, -m);
#pragma unroll
        for (int fr = 0; fr < 4; ++fr) {
          uint32_t w[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int e = fr * 32 + 2 * q;
            const float2 x = ffma2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), sc2v, nm);
            float2 y;
            if ((kPoly >> ((fr * 16 + q) & 7)) & 1) {
              y = exp2_poly2(x);
            } else {
              y.x = ex2(x.x);
              y.y = ex2(x.y);
            }
            v[e] = __float_as_uint(y.x);
            v[e + 1] = __float_as_uint(y.y);
            w[q] = pack_bf16(y.x, y.y);
          }
          tmem_st_32x32b_x16(s_addr + uint32_t(fr * 16), w);
          if (fr == kSplitFr - 1 || fr == 3) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(fr == kSplitFr - 1 ? &p_part[t] : &p_full[t]);
          }
        }
        // row sum off the critical path (P is already with the tensor pipe)
        float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0, acc2 = acc0, acc3 = acc0;
#pragma unroll
        for (int e = 0; e < 128; e += 8) {
          acc0 = fadd2(acc0, make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
          acc1 = fadd2(acc1, make_float2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3])));
          acc2 = fadd2(acc2, make_float2(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5])));
          acc3 = fadd2(acc3, make_float2(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7])));
        }
        acc0 = fadd2(fadd2(acc0, acc1), fadd2(acc2, acc3));
        l = l * f + (acc0.x + acc0.y);
      }
      lbuf[t * BQ + row] = l;
      __syncwarp();
      if (lane == 0) mbar_arrive(&l_ready[t]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<C_::TMEM_COLS>(tmem);
  }
}

template <int D>
cudaError_t launch_d(const AttnLaunch& p0, int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_kernel<D, kPolyPairs>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<D>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  AttnLaunch p = p0;
  attn_schedule(p, num_sms);

  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_jobs < num_sms ? p.n_jobs : num_sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = ACfg<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, attn_kernel<D, kPolyPairs>, p);
  return e;
}

}  // namespace

void attn_schedule(AttnLaunch& p, int num_sms) {
  // waves of tile pairs, then one wave mixing pairs and single tiles so every
  // CTA ends at about the same time
  const int tph = p.S / BQ, pph = tph / 2;
  const long long tiles = (long long)p.n_regions * p.H * tph;
  const long long units = (long long)p.n_regions * p.H * pph;
  const long long G = num_sms;
  long long np = 0;
  if (tiles > G) {
    const long long w = tiles / (2 * G), r = tiles - 2 * w * G;
    np = w * G + (r > G ? r - G : 0);
  }
  if (np > units) np = units;
  p.n_pair_jobs = int(np);
  p.n_jobs = int(tiles - np);
}

cudaError_t attn_prepare() {
  cudaError_t e =
      cudaFuncSetAttribute(attn_kernel<64, kPolyPairs>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<64>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_kernel<128, kPolyPairs>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              ACfg<128>::SMEM);
}

bool attn_supported(int S, int T, int D) { return (D == 64 || D == 128) && S % BQ == 0 && T % BKV == 0 && T > 0; }

cudaError_t launch_attn(const AttnLaunch& p, int num_sms, cudaStream_t s) {
  if (p.D == 128) return launch_d<128>(p, num_sms, s);
  if (p.D == 64) return launch_d<64>(p, num_sms, s);
  return cudaErrorInvalidValue;
}

}  // namespace ed
