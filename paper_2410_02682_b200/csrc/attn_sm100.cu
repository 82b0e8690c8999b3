// Fused attention block: T1 = QK^T (+ fused scale), the five-vertex row
// softmax, and O = T3 V — three einsums of the plan executed as one tcgen05
// kernel, so the [h, s, s2] logits and probabilities never reach HBM.
//
// A job is a pair of 128-row query tiles of one head (or a single tile in
// the last wave, to fill the grid): K_j and V_j are loaded once per pair.
// Each tile runs its own chain on the tensor pipe,
//
//   S_t(j) -> softmax_t(j) -> PV_t(j) -> S_t(j+1) -> ...
//
// issued by its own MMA thread; tile 1 starts half a step late so one
// tile's softmax overlaps the other tile's MMAs.
//
// S_t = Q_t K_j^T lands in TMEM; the softmax warps of tile t read it (one
// thread per row), keep a reference max m (log2 domain) and sum l, write
// P = exp2(c log2e S - m) back over S as packed bf16, and O_t += P V_j takes
// P straight from TMEM (the A-from-TMEM form of tcgen05.mma), so P never
// touches shared memory. O_t is rescaled in TMEM only when a row's max
// passes the reference by more than 2^64 (P stays far inside the bf16 /
// fp32 range); the commit that signals S_t(j) also covers PV_t(j-1), so the
// rescale never races an MMA. Epilogue: O / l -> swizzled smem -> TMA store.
//
// Warp roles (512 threads, four warpgroups): warps 0-3 softmax + epilogue
// of tile 0, warps 4-7 of tile 1 (warp w owns TMEM lanes 32(w%4)..+32),
// warp 8 TMA producer, warp 9 TMEM allocator + MMA issuer of tile 0, warp
// 10 MMA issuer of tile 1, warp 11 idle, warps 12-15 the correction
// warpgroup (O rescales, off the softmax's path). setmaxnreg moves
// registers from the producer and correction warpgroups to the softmax
// warpgroups, so a thread can hold its whole 128-key S row.
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
constexpr int kTmaWarp = 8, kMmaWarp = 9;
// register split (setmaxnreg): 2 x 128 x 200 + 128 x 48 + 128 x 56 <= 64K
constexpr int kSoftmaxRegs = 200, kProducerRegs = 48, kCorrectionRegs = 56;
// the softmax warpgroups can only take what the others give back from the
// launch allocation (65536 / threads per thread), or setmaxnreg.inc never returns
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;
static_assert(2 * (kSoftmaxRegs - kLaunchRegs) <= (kLaunchRegs - kProducerRegs) + (kLaunchRegs - kCorrectionRegs),
              "setmaxnreg split exceeds the launch allocation");
constexpr int kCorrWarp0 = 12;  // warps 12-15: O rescale (correction) warpgroup
// lazy rescale (log2 units): P = 2^(x - m) may reach 2^kRescale before O is
// rescaled, and a rescale sets m = row max + kHeadroom. bf16 / fp32 keep full
// relative precision over that span; O = sum P V keeps 2^64 / 4096 of headroom
// for |V|, and keys more than ~2^-78 below the row max underflow to 0.
constexpr float kRescale = 64.0f, kHeadroom = 48.0f;
// exp2 pairs q with bit q % 8 set run on the FMA pipe (measured: 2 of 8 is
// ~2% faster than MUFU only; more is slower, the kernel is not MUFU-bound)
constexpr int kPolyPairs = 0x88;
// 1: the two MMA threads take turns (PV_t(j) + S_t(j+1) groups alternate on
// the tensor pipe), so the tiles' softmaxes run in anti-phase. Measured
// slower (0.346 vs 0.32 ms on attn_big): each group then waits a whole
// softmax for its turn, and the TS-form PV MMAs still slow down under the
// other tile's TMEM stores (profiles/r01b_micro_tcgen05.md). Off by default.
#ifndef ED_ATTN_ALT
#define ED_ATTN_ALT 0
#endif
constexpr bool kAlternate = ED_ATTN_ALT;

template <int D>
struct ACfg {
  static constexpr int Q_BYTES = BQ * D * 2;   // D/64 K-major chunks of 16 KiB
  static constexpr int K_BYTES = BKV * D * 2;
  static constexpr int V_BYTES = BKV * D * 2;  // D/64 MN atoms of 128 key-rows x 128 B
  static constexpr int STG_BYTES = 4096;       // per softmax warp: 32 rows x 128 B
  static constexpr int SMEM = 2 * Q_BYTES + 2 * K_BYTES + 2 * V_BYTES + 8 * STG_BYTES + 1024 + 256 + 1088;
  static constexpr int TMEM_COLS = 512;
  __host__ __device__ static constexpr int s_col(int t) { return t * BKV; }
  __host__ __device__ static constexpr int o_col(int t) { return 2 * BKV + t * D; }
};

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

// debug tracing (ED_ATTN_TRACE=1, profile runs only): clock64 at pipeline
// events of the first job of CTA 0, [event][tile][block]
#define ATTN_TRACE(ev, t, j)                                                                     \
  do {                                                                                           \
    if (p.trace && blockIdx.x == 0 && jb == 0 && (j) < 64)                                       \
      p.trace[((ev) * 2 + (t)) * 64 + (j)] = clock64();                                         \
  } while (0)

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

template <int D, int kPoly>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(const __grid_constant__ AttnLaunch p) {
  using C_ = ACfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                          // [2] tiles
  uint8_t* sK = sQ + 2 * C_::Q_BYTES;          // [2] stages
  uint8_t* sV = sK + 2 * C_::K_BYTES;          // [2] stages
  uint8_t* sStg = sV + 2 * C_::V_BYTES;        // [8] softmax warps
  uint64_t* bar = reinterpret_cast<uint64_t*>(sStg + 8 * C_::STG_BYTES);
  uint64_t* q_full = bar + 0;    // [tile]
  uint64_t* q_empty = bar + 2;   // [tile]
  uint64_t* k_full = bar + 4;    // [stage]
  uint64_t* k_empty = bar + 6;   // [stage]
  uint64_t* v_full = bar + 8;    // [stage]
  uint64_t* v_empty = bar + 10;  // [stage]
  uint64_t* s_full = bar + 12;   // [tile]
  uint64_t* p_full = bar + 14;   // [tile]
  uint64_t* o_full = bar + 16;   // [tile]
  uint64_t* o_empty = bar + 18;  // [tile]
  uint64_t* p_half = bar + 20;   // [tile]: first 64 keys of P published
  uint64_t* t1_go = bar + 22;    // tile 1 starts half a step behind tile 0
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 23);
  uint64_t* corr_req = bar + 24;   // [tile] softmax -> correction: factors posted
  uint64_t* corr_done = bar + 26;  // [tile] correction -> MMA: O_t rescaled
  uint64_t* turn = bar + 28;       // [tile] the tensor pipe alternates PV+S groups between tiles
  float* fac = reinterpret_cast<float*>(bar + 32);      // [tile][row] rescale factor
  int* fac_any = reinterpret_cast<int*>(fac + 2 * BQ);  // [tile][lane quarter] any row grew

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = p.T / BKV;
  const int jobs = p.n_jobs;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 2);  // one arrival per MMA thread
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 2);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_half[i], 4);
      if (i == 0) mbar_init(t1_go, 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 4);
      mbar_init(&corr_req[i], 4);
      mbar_init(&corr_done[i], 4);
      mbar_init(&turn[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc<C_::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // the prologue above overlapped the previous kernel (PDL)

  if (warp >= kCorrWarp0) {
    // ---------------- O rescale (correction) warpgroup ----------------
    // Off the softmax's path: the softmax posts per-row factors right after
    // its row max and goes on with exp2; this warp rescales its 32 rows of
    // O_t in TMEM (only if one of them grew) and releases PV_t(j).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCorrectionRegs));
    const int wq = warp & 3;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    int cn0 = 0, cn1 = 0;
    for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
      const Job J = job_of(p, jb);
      for (int j = 0; j < nb; ++j)
        for (int t = 0; t <= J.two; ++t) {
          int& cn = t ? cn1 : cn0;
          mbar_wait(&corr_req[t], cn & 1);
          ++cn;
          if (fac_any[t * 4 + wq]) {
            // PV_t(j-1) is complete: the softmax posted after S_t(j)'s commit
            tc_fence_after();
            const float f = fac[t * BQ + wq * 32 + lane];
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
          if (lane == 0) mbar_arrive(&corr_done[t]);
        }
    }
  } else if (warp >= 8) {
    // producer warpgroup: hand registers to the softmax warpgroups
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    if (warp == kTmaWarp) {
      // ---------------- TMA producer ----------------
      if (lane == 0) {
        int kc = 0, vc = 0, qn0 = 0, qn1 = 0;
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
            int st = kc & 1;
            mbar_wait(&k_empty[st], ((kc >> 1) & 1) ^ 1);
            ++kc;
            mbar_expect_tx(&k_full[st], C_::K_BYTES);
  #pragma unroll
            for (int c = 0; c < D / 64; ++c)
              tma_load_3d(sK + st * C_::K_BYTES + c * 16384, src_map(R.k, j * BKV, c * 64), &k_full[st],
                          (c * 64) % R.k.dw, (j * BKV) % R.k.keys, J.h + R.k.hoff);
            st = vc & 1;
            mbar_wait(&v_empty[st], ((vc >> 1) & 1) ^ 1);
            ++vc;
            mbar_expect_tx(&v_full[st], C_::V_BYTES);
  #pragma unroll
            for (int a = 0; a < D / 64; ++a)
              tma_load_3d(sV + st * C_::V_BYTES + a * (BKV * 128), src_map(R.v, j * BKV, a * 64), &v_full[st],
                          (a * 64) % R.v.dw, (j * BKV) % R.v.keys, J.h + R.v.hoff);
          }
        }
      }
    } else if (warp == kMmaWarp || warp == kMmaWarp + 1) {
      // ---------------- MMA issuers: one thread per tile ----------------
      // Each tile's chain (S_t(j) -> softmax -> PV_t(j) -> S_t(j+1)) is issued
      // by its own thread, so one tile's MMAs never wait behind the other
      // tile's softmax; K/V stages are released by both (count 2).
      const int t = warp - kMmaWarp;
      if (lane == 0) {
        const uint32_t idesc_s = umma_idesc(1u, BQ, BKV, 0u, 0u);  // Q, K both K-major (d)
        const uint32_t idesc_o = umma_idesc(1u, BQ, D, 0u, 1u);    // P from TMEM (keys), V MN-major (d)
        const uint32_t qa = smem_u32(sQ + t * C_::Q_BYTES);
        int kc = 0, vc = 0, qn = 0, pn = 0, on = 0, gn = 0, tn = 0;
        auto issue_s = [&](int kst) {
          const uint32_t ka = smem_u32(sK + kst * C_::K_BYTES);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k / 4) * 16384 + (k % 4) * 32;
            mma_f16(tmem + C_::s_col(t), umma_desc_sw128(qa + off, 16, 1024), umma_desc_sw128(ka + off, 16, 1024),
                    idesc_s, k != 0);
          }
          mma_commit(&s_full[t]);
        };
        for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
          const Job J = job_of(p, jb);
          if (t > J.two) {  // single-tile job: tile 0's thread releases the stages twice
            kc += nb;
            vc += nb;
            continue;
          }
          const int rel = J.two ? 1 : 2;  // k_empty / v_empty arrivals this thread owes
          mbar_wait(&q_full[t], qn & 1);
          ++qn;
          if (t == 1) {
            // stagger: tile 1's chain starts once tile 0's first PV is issued,
            // so each tile's softmax overlaps the other tile's MMAs
            mbar_wait(t1_go, gn & 1);
            ++gn;
          }
          int kst = kc & 1;
          mbar_wait(&k_full[kst], (kc >> 1) & 1);
          ++kc;
          tc_fence_after();
          issue_s(kst);
          ATTN_TRACE(5, t, 0);
          if (nb == 1) mma_commit(&q_empty[t]);
          for (int r = 0; r < rel; ++r) mma_commit(&k_empty[kst]);
          for (int j = 0; j < nb; ++j) {
            const int vst = vc & 1;
            mbar_wait(&v_full[vst], (vc >> 1) & 1);
            ++vc;
            const uint32_t va = smem_u32(sV + vst * C_::V_BYTES);
            mbar_wait(&p_half[t], pn & 1);
            mbar_wait(&corr_done[t], pn & 1);
            if (kAlternate && J.two) {  // tile 0 holds the first turn
              mbar_wait(&turn[t], (tn & 1) ^ (t == 0 ? 1 : 0));
              ++tn;
            }
            ATTN_TRACE(3, t, j);
            if (j == 0) {  // the last job's epilogue has drained O_t
              mbar_wait(&o_empty[t], (on & 1) ^ 1);
              ++on;
            }
            tc_fence_after();
            // PV over the first 64 keys while the softmax finishes the rest
#pragma unroll
            for (int k = 0; k < BKV / 32; ++k)
              mma_f16_ts(tmem + C_::o_col(t), tmem + C_::s_col(t) + k * 8,
                         umma_desc_sw128(va + k * 2048, BKV * 128, 1024), idesc_o, (j | k) != 0);
            if (t == 0 && j == 0 && J.two) mbar_arrive(t1_go);
            mbar_wait(&p_full[t], pn & 1);
            ++pn;
            ATTN_TRACE(4, t, j);
            tc_fence_after();
#pragma unroll
            for (int k = BKV / 32; k < BKV / 16; ++k)
              mma_f16_ts(tmem + C_::o_col(t), tmem + C_::s_col(t) + k * 8,
                         umma_desc_sw128(va + k * 2048, BKV * 128, 1024), idesc_o, 1u);
            for (int r = 0; r < rel; ++r) mma_commit(&v_empty[vst]);
            if (j == nb - 1) mma_commit(&o_full[t]);
            if (j + 1 < nb) {
              kst = kc & 1;
              ATTN_TRACE(9, t, j + 1);
              mbar_wait(&k_full[kst], (kc >> 1) & 1);
              ++kc;
              tc_fence_after();
              issue_s(kst);  // in issue order after PV_t(j): overwrites P_t(j) only once it is read
              ATTN_TRACE(5, t, j + 1);
              if (j + 1 == nb - 1) mma_commit(&q_empty[t]);
              for (int r = 0; r < rel; ++r) mma_commit(&k_empty[kst]);
            }
            if (kAlternate && J.two) mbar_arrive(&turn[t ^ 1]);
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
    // ---------------- softmax + epilogue (tile t = warp / 4) ----------------
    const int t = warp >> 2, wq = warp & 3;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + uint32_t(C_::s_col(t));
    const uint32_t o_addr = tmem + lane_base + uint32_t(C_::o_col(t));
    const float sc2 = p.scale * 1.4426950408889634f;  // c * log2(e)
    uint8_t* stg = sStg + warp * C_::STG_BYTES;
    int sn = 0, on = 0;
    for (int jb = blockIdx.x; jb < jobs; jb += gridDim.x) {
      const Job J = job_of(p, jb);
      if (t > J.two) continue;
      float m = 0.f, l = 0.f;  // reference max (log2 domain) and row sum
      for (int j = 0; j < nb; ++j) {
        mbar_wait(&s_full[t], sn & 1);
        if (lane == 0 && wq == 0) ATTN_TRACE(0, t, j);
        ++sn;
        tc_fence_after();
        uint32_t v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tmem_ld_32x32b_x32(s_addr + uint32_t(c * 32), *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
        tmem_ld_wait();
        if (lane == 0 && wq == 0) ATTN_TRACE(6, t, j);
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
        if (lane == 0 && wq == 0) ATTN_TRACE(7, t, j);
        if (lane == 0 && wq != 0) ATTN_TRACE(12 + wq, t, j);
        // reference max with hysteresis: when a row's max passes m + kRescale
        // the new reference is max + kHeadroom, so P spans [2^-kHeadroom,
        // 2^kRescale] at the row max and rescales stay rare
        bool grow = false;
        float f = 1.f;
        if (j == 0) {
          m = mx + kHeadroom;
        } else if (mx > m + kRescale) {
          grow = true;
          const float mn = mx + kHeadroom;
          f = ex2(m - mn);
          m = mn;
        }
        // post this row's factor to the correction warp of its lane quarter
        {
          const bool wgrow = __any_sync(0xffffffffu, grow);
          fac[t * BQ + wq * 32 + lane] = f;
          if (lane == 0) fac_any[t * 4 + wq] = wgrow;
          __syncwarp();
          if (lane == 0) mbar_arrive(&corr_req[t]);
        }
        // P = exp2(c log2e S - m), packed bf16, written over S in two halves
        // of 64 keys (the S values of a half are in registers before its
        // P columns, which alias S columns [0, 64), are stored); the first
        // half is published at once so PV over it starts early. One pair in
        // four is evaluated on the FMA pipe (exp2_poly2) to unload MUFU.
        const float2 sc2v = make_float2(sc2, sc2), nm = make_float2(-m, -m);
        float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t w[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int e = hh * 64 + 2 * q;
            const float2 x = ffma2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), sc2v, nm);
            float2 y;
            if ((kPoly >> (q & 7)) & 1) {
              y = exp2_poly2(x);
            } else {
              y.x = ex2(x.x);
              y.y = ex2(x.y);
            }
            if (q & 1) acc1 = fadd2(acc1, y);
            else acc0 = fadd2(acc0, y);
            w[q] = pack_bf16(y.x, y.y);
          }
          tmem_st_32x32b_x32(s_addr + uint32_t(hh * 32), w);
          if (lane == 0 && wq == 0 && hh == 0) ATTN_TRACE(8, t, j);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(hh == 0 ? &p_half[t] : &p_full[t]);
          if (lane == 0 && wq == 0) ATTN_TRACE(1 + hh, t, j);
          if (lane == 0 && wq != 0 && hh == 1) ATTN_TRACE(9 + wq, t, j);
        }
        acc0 = fadd2(acc0, acc1);
        l = l * f + (acc0.x + acc0.y);
      }
      // ---- epilogue: O_t / l -> swizzled staging -> TMA store (32 rows per warp)
      mbar_wait(&o_full[t], on & 1);
      ++on;
      tc_fence_after();
      const float inv = 1.0f / l;
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
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          uint8_t* rowp = stg + lane * 128;
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
            tma_store_3d(p.maps + cm, stg, c * cols, row0, J.h);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[t]);
    }
    if (lane == 0) bulk_wait<0>();
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

  static const bool trace = std::getenv("ED_ATTN_TRACE") != nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (trace && cs == cudaStreamCaptureStatusNone) {
    cudaMalloc(&p.trace, 16 * 2 * 64 * sizeof(long long));
    cudaMemsetAsync(p.trace, 0, 16 * 2 * 64 * sizeof(long long), s);
  }
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
  if (p.trace) {
    long long h[16 * 2 * 64];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(p.trace);
    const long long t0 = h[5 * 128];
    const char* names[16] = {"s_ready", "p_half", "p_full", "mma_got_half", "mma_got_full", "s_issued", "s_loaded", "max_done", "half0_stored", "pvb_issued", "p_full_w1", "p_full_w2", "p_full_w3", "max_w1", "max_w2", "max_w3"};
    for (int ev = 0; ev < 16; ++ev)
      for (int t = 0; t < 2; ++t) {
        std::fprintf(stderr, "attn_trace %-13s t%d:", names[ev], t);
        for (int j = 0; j < 33; ++j) std::fprintf(stderr, " %lld", h[(ev * 2 + t) * 64 + j] ? h[(ev * 2 + t) * 64 + j] - t0 : -1);
        std::fprintf(stderr, "\n");
      }
  }
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
