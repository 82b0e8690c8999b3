// Fused attention block in the fp32-accurate mode (fp32x3): T1 = QK^T (+ its
// fused scale), the row softmax and O = T3 V as one tcgen05 kernel, every
// contraction as three TF32 products hi*hi + hi*lo + lo*hi (lo = x - tf32(x),
// the shadows the producers write beside Q, K and V), P computed and kept in
// fp32. The [h, s, s2] logits never reach HBM (the unfused fp32x3 path moves
// them through HBM five times: T1, softmax in/out, its lo shadow, O's reads).
//
// A job is one 128-row query tile of one head. TMEM (512 columns):
//   Q [0,128) (fp32: the MMA reads it as Q_hi)  O_j [128,256)  R(b, part) = 256 + 128 b + 64 part, b = block parity:
//   part 0 holds S_j, then P_j (fp32, the hi operand: the MMA drops its low
//   13 bits), part 1 holds P_j - tf32(P_j).
// Q_lo sits in shared memory (64 KiB), so only Q_lo K_hi reads its A operand
// from shared memory (shared-memory bandwidth bounds this kernel: per key
// block the MMAs read ~260 KiB of operands and TMA writes 128 KiB); K_j and V_j (64 keys) stream through a
// ring of ten 16 KiB slots (half a block's lo or hi copy each) in the order
// the MMA consumes them: K0 | K1 V0 | K2 V1 | ...  Within S_j all Q_hi K_lo
// products go first and within PV_j all P_hi V_lo ones, so slots are
// released an eighth of a block at a time and the loads run well ahead.
//
// One warp issues the MMAs in the order S_0 | S_1 PV_0 | S_2 PV_1 | ..., so
// S_{j+1} runs while the softmax works on S_j; the two S/P buffers alternate.
// Promoted accumulation: every PV_j starts a fresh TMEM accumulator O_j, and
// the correction warps fold it into fp32 running sums in registers with
// IEEE operations, O = f_j O + O_j (the tensor core's truncating accumulation
// is confined to the 192 products of one key block, as in the x3 GEMM). The
// softmax keeps the exact running row max m (log2 domain, rounded up to an
// integer), so P <= 1 and the rescale factor f_j = 2^(m_{j-1} - m_j) is an
// exact power of two.
//
// Warps: 0-3 softmax (warp w: TMEM lanes 32w..32w+31, one thread per row),
// 4-7 correction + epilogue (same rows), 8 TMEM allocator + MMA issuer, 9 TMA,
// 10-11 idle.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "attn_sm100.h"
#include "ptx.cuh"

namespace ed {

namespace {

constexpr int XQ = 128;   // query rows per job
constexpr int XKV = 64;   // keys per block
constexpr int XD = 128;   // head dim
constexpr int kXThreads = 384;  // three warpgroups: one warp of each on every 16K-register sub-partition
constexpr int kXCorrWarp0 = 4, kXMmaWarp = 8, kXTmaWarp = 9;
// setmaxnreg: the correction warpgroup holds each row's 128 running sums;
// the producer warpgroup (MMA, TMA, two idle warps) gives registers back.
// Per sub-partition: 168 (softmax) + 232 + 96 <= 512 per lane.
constexpr int kXCorrRegs = 232, kXProdRegs = 96;
constexpr int XQ_BYTES = XQ * XD * 4;   // 4 K-major chunks of 128 rows x 128 B
// a slot holds half of one key block's K or V copy: K, two K-major chunks of
// 64 rows x 128 B (32 of the 128 d); V, the 4 MN atoms of 32 keys x 128 B
constexpr int XSLOT = XKV * XD * 2;
constexpr int XNSLOT = 10;
constexpr int XBAR_BYTES = 512;
constexpr int XSMEM = XQ_BYTES + XNSLOT * XSLOT + XBAR_BYTES + 3 * XQ * 4 + 1024;
static_assert(XSMEM <= 232448, "shared memory");
constexpr uint32_t T_Q = 0, T_O = 128;
__device__ __forceinline__ uint32_t t_r(int b, int part) { return 256u + uint32_t(b) * 128u + uint32_t(part) * 64u; }

struct XJob {
  int region, h, s0;
};

__device__ __forceinline__ XJob xjob_of(const AttnLaunch& p, int j) {
  const int tph = p.S / XQ;
  const int rh = j / tph;
  XJob r;
  r.region = rh / p.H;
  r.h = rh % p.H;
  r.s0 = (j % tph) * XQ;
  return r;
}

__device__ __forceinline__ float xex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lo_part(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// 2^k for an integer-valued k <= 0 (0 below the normal range)
__device__ __forceinline__ float pow2i(float k) {
  return k < -126.f ? 0.f : __int_as_float((127 + int(k)) << 23);
}

__global__ void __launch_bounds__(kXThreads, 1) attn_x3_kernel(const __grid_constant__ AttnLaunch p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + XQ_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sKV + XNSLOT * XSLOT);
  uint64_t* q_full = bar + 0;      // TMA -> MMA: Q_lo in smem
  uint64_t* q_empty = bar + 1;     // MMA -> TMA: the job's last S done
  uint64_t* qt_full = bar + 2;     // softmax -> MMA: Q in TMEM
  uint64_t* s_full = bar + 3;      // [2] MMA -> softmax: S_j in R(j & 1)
  // [2] softmax -> MMA: P_j stored. Per block parity: a softmax warp may
  // finish block j+1 (S_{j+1} is ready early) before another warp has
  // finished block j, so one barrier could complete on the wrong arrivals.
  uint64_t* p_full = bar + 5;
  uint64_t* sc_full = bar + 7;     // [2] softmax -> correction: f_j posted
  uint64_t* pv_done = bar + 9;     // MMA -> softmax, correction: PV_j in O_j
  uint64_t* o_free = bar + 10;     // correction -> MMA: O_j folded into the running sums
  uint64_t* l_ready = bar + 11;    // softmax -> correction: the job's row sums posted
  uint64_t* slot_full = bar + 12;  // [XNSLOT]
  uint64_t* slot_empty = slot_full + XNSLOT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slot_empty + XNSLOT);
  static_assert((12 + 2 * XNSLOT) * 8 + 4 <= XBAR_BYTES, "barrier space");
  float* scl = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bar) + XBAR_BYTES);  // [2][XQ] f_j per row
  float* lbuf = scl + 2 * XQ;                                                           // [XQ] row sums

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = p.T / XKV;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(qt_full, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&sc_full[i], 4);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_free, 4);
    mbar_init(l_ready, 4);
    for (int i = 0; i < XNSLOT; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kXMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();

  if (warp >= kXMmaWarp) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kXProdRegs));
  if (warp >= kXMmaWarp + 2) {
    // idle
  } else if (warp == kXTmaWarp) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int sn = 0, qn = 0;
      auto slot_get = [&]() {
        const int st = sn % XNSLOT;
        mbar_wait(&slot_empty[st], ((sn / XNSLOT) & 1) ^ 1);
        ++sn;
        return st;
      };
      for (int jb = blockIdx.x; jb < p.n_jobs; jb += gridDim.x) {
        if (jb + int(gridDim.x) >= p.n_jobs) griddep_launch();
        const XJob J = xjob_of(p, jb);
        const AttnRegion& R = p.regions[J.region];
        auto src_map = [&](const AttnSrc& a, int key, int dcol) {
          return p.maps + a.base + (key / a.keys) * a.nd + dcol / a.dw;
        };
        mbar_wait(q_empty, (qn & 1) ^ 1);
        ++qn;
        mbar_expect_tx(q_full, XQ_BYTES);
#pragma unroll
        for (int c = 0; c < XD / 32; ++c) tma_load_3d(sQ + c * 16384, p.maps + R.q, q_full, c * 32, J.s0, J.h);
        auto load_k = [&](int j) {
          for (int part = 1; part >= 0; --part)  // lo first: consumed first
            for (int hf = 0; hf < 2; ++hf) {     // d chunks 2 hf, 2 hf + 1
              const int st = slot_get();
              uint8_t* dst = sKV + st * XSLOT;
              mbar_expect_tx(&slot_full[st], XSLOT);
#pragma unroll
              for (int c = 2 * hf; c < 2 * hf + 2; ++c)
                tma_load_3d(dst + (c - 2 * hf) * 8192, src_map(R.k, j * XKV, c * 32) + part * R.k.lo, &slot_full[st],
                            (c * 32) % R.k.dw, (j * XKV) % R.k.keys, J.h + R.k.hoff);
            }
        };
        auto load_v = [&](int j) {
          for (int part = 1; part >= 0; --part)
            for (int kb = 0; kb < 2; ++kb) {  // keys 32 kb .. 32 kb + 31 of the block
              const int st = slot_get();
              uint8_t* dst = sKV + st * XSLOT;
              mbar_expect_tx(&slot_full[st], XSLOT);
              const int key = j * XKV + kb * 32;
#pragma unroll
              for (int a = 0; a < XD / 32; ++a)
                tma_load_3d(dst + a * 4096, src_map(R.v, key, a * 32) + part * R.v.lo, &slot_full[st],
                            (a * 32) % R.v.dw, key % R.v.keys, J.h + R.v.hoff);
            }
        };
        load_k(0);
        for (int j = 0; j < nb; ++j) {
          if (j + 1 < nb) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp == kXMmaWarp) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    const uint32_t idesc_s = umma_idesc(2u, XQ, XKV, 0u, 0u);  // Q, K both K-major (d)
    const uint32_t idesc_o = umma_idesc(2u, XQ, XD, 0u, 1u);   // P from TMEM (keys), V MN-major (d)
    int sn = 0, qn = 0, pn0 = 0, pn1 = 0, on = 0;
#if X3_PROF
    long long prof[4] = {0, 0, 0, 0};  // wait K slots, issue S, wait P / O free / V slots, issue PV
    long long t0 = 0;
#define MPROF(i)                    \
  {                                 \
    const long long t1 = clock64(); \
    prof[i] += t1 - t0;             \
    t0 = t1;                        \
  }
#else
#define MPROF(i)
#endif
    auto take = [&]() {
      const int st = sn % XNSLOT;
      mbar_wait(&slot_full[st], (sn / XNSLOT) & 1);
      ++sn;
      return st;
    };
    const uint64_t qd = umma_desc_sw128(smem_u32(sQ), 16, 1024);
    auto issue_s = [&](int b) {
      const uint32_t d = tmem + t_r(b, 0);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // Q_hi K_lo over d chunks 2 hf, 2 hf + 1
        const int kl = take();
        MPROF(0)
        const uint64_t kld = umma_desc_sw128(smem_u32(sKV + kl * XSLOT), 16, 1024);
#pragma unroll
        for (int k = 8 * hf; k < 8 * hf + 8; ++k) {
          const uint64_t ko = uint64_t(((k / 4 - 2 * hf) * 8192 + (k % 4) * 32) >> 4);
          mma_tf32_ts_warp(d, tmem + T_Q + uint32_t(k * 8), kld + ko, idesc_s, k != 0);
        }
        mma_commit_warp(&slot_empty[kl]);
      }
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // Q_lo K_hi + Q_hi K_hi
        const int kh = take();
        MPROF(0)
        const uint64_t khd = umma_desc_sw128(smem_u32(sKV + kh * XSLOT), 16, 1024);
#pragma unroll
        for (int k = 8 * hf; k < 8 * hf + 8; ++k) {
          const uint64_t qo = uint64_t(((k / 4) * 16384 + (k % 4) * 32) >> 4);
          const uint64_t ko = uint64_t(((k / 4 - 2 * hf) * 8192 + (k % 4) * 32) >> 4);
          mma_tf32_warp(d, qd + qo, khd + ko, idesc_s, 1u);
          mma_tf32_ts_warp(d, tmem + T_Q + uint32_t(k * 8), khd + ko, idesc_s, 1u);
        }
        mma_commit_warp(&slot_empty[kh]);
      }
      mma_commit_warp(&s_full[b]);
      MPROF(1)
    };
    auto issue_pv = [&](int b) {
      const uint32_t ph = tmem + t_r(b, 0), pl = tmem + t_r(b, 1);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {  // P_hi V_lo over keys 32 kb.., a fresh O_j
        const int vl = take();
        MPROF(2)
        const uint64_t vld = umma_desc_sw128(smem_u32(sKV + vl * XSLOT), 4096, 512, 1);
#pragma unroll
        for (int k = 4 * kb; k < 4 * kb + 4; ++k)
          mma_tf32_ts_warp(tmem + T_O, ph + uint32_t(k * 8), vld + uint64_t(((k % 4) * 1024) >> 4), idesc_o, k != 0);
        mma_commit_warp(&slot_empty[vl]);
      }
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {  // P_lo V_hi + P_hi V_hi
        const int vh = take();
        MPROF(2)
        const uint64_t vhd = umma_desc_sw128(smem_u32(sKV + vh * XSLOT), 4096, 512, 1);
#pragma unroll
        for (int k = 4 * kb; k < 4 * kb + 4; ++k) {
          const uint64_t vo = uint64_t(((k % 4) * 1024) >> 4);
          mma_tf32_ts_warp(tmem + T_O, pl + uint32_t(k * 8), vhd + vo, idesc_o, 1u);
          mma_tf32_ts_warp(tmem + T_O, ph + uint32_t(k * 8), vhd + vo, idesc_o, 1u);
        }
        mma_commit_warp(&slot_empty[vh]);
      }
      mma_commit_warp(pv_done);
      MPROF(3)
    };
    for (int jb = blockIdx.x; jb < p.n_jobs; jb += gridDim.x) {
      mbar_wait(q_full, qn & 1);
      mbar_wait(qt_full, qn & 1);
      ++qn;
      tc_fence_after();
#if X3_PROF
      t0 = clock64();
#endif
      issue_s(0);
      if (nb == 1) mma_commit_warp(q_empty);
      for (int j = 0; j < nb; ++j) {
        const int b = j & 1;
        if (j + 1 < nb) {
          // S_{j+1} overwrites the buffer PV_{j-1} read: issued after it, so in order
          issue_s(b ^ 1);
          if (j + 1 == nb - 1) mma_commit_warp(q_empty);
        }
        int& pn = b ? pn1 : pn0;
        mbar_wait(&p_full[b], pn & 1);
        ++pn;
        if (on > 0) mbar_wait(o_free, (on - 1) & 1);  // the correction warps have read O_{j-1}
        ++on;
        tc_fence_after();
        issue_pv(b);
      }
    }
#if X3_PROF
    if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
      printf("cta %d mma cycles: wait K %lld issue S %lld wait P/O/V %lld issue PV %lld\n", blockIdx.x, prof[0],
             prof[1], prof[2], prof[3]);
#endif
  } else if (warp >= kXCorrWarp0) {
    // ---------------- correction: O = f_j O + O_j in registers, then the epilogue ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kXCorrRegs));
    const int wq = warp - kXCorrWarp0;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    int pvn = 0, sc0 = 0, sc1 = 0, ln = 0;
    for (int jb = blockIdx.x; jb < p.n_jobs; jb += gridDim.x) {
      const XJob J = xjob_of(p, jb);
      const AttnRegion& R = p.regions[J.region];
      float o[XD];
#pragma unroll
      for (int e = 0; e < XD; ++e) o[e] = 0.f;
      for (int j = 0; j < nb; ++j) {
        const int b = j & 1;
        int& sc = b ? sc1 : sc0;
        mbar_wait(&sc_full[b], sc & 1);
        ++sc;
        const float f = scl[b * XQ + row];
        mbar_wait(pv_done, uint32_t(pvn) & 1);
        ++pvn;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < XD / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + lane_base + T_O + uint32_t(c * 32), r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            o[c * 32 + e] = fmaf(o[c * 32 + e], f, __uint_as_float(r[e]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);
      }
      // ---- epilogue: O / l (and its lo shadow) -> HBM, one row per thread
      mbar_wait(l_ready, ln & 1);
      ++ln;
      const float inv = 1.0f / lbuf[row];
      float* out = R.o + J.h * R.o_hs + (long long)(J.s0 + row) * R.o_rs;
      float* ol = R.o_lo ? R.o_lo + J.h * R.o_hs + (long long)(J.s0 + row) * R.o_rs : nullptr;
#pragma unroll
      for (int g = 0; g < XD / 4; ++g) {
        const float4 y = make_float4(o[4 * g] * inv, o[4 * g + 1] * inv, o[4 * g + 2] * inv, o[4 * g + 3] * inv);
        __stcs(reinterpret_cast<float4*>(out + 4 * g), y);
        if (ol)
          __stcs(reinterpret_cast<float4*>(ol + 4 * g),
                 make_float4(lo_part(y.x), lo_part(y.y), lo_part(y.z), lo_part(y.w)));
      }
    }
  } else {
    // ---------------- softmax (one thread per row) ----------------
    const int row = warp * 32 + lane;
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    const float sc2 = p.scale * 1.4426950408889634f;  // c * log2(e)
    int sn0 = 0, sn1 = 0, pvn = 0;
#if X3_PROF
    long long sp[4] = {0, 0, 0, 0};  // wait S + load, compute P, wait PV_{j-1}, store
    long long ts = clock64();
#define SPROF(i)                    \
  {                                 \
    const long long t1 = clock64(); \
    sp[i] += t1 - ts;               \
    ts = t1;                        \
  }
#else
#define SPROF(i)
#endif
    for (int jb = blockIdx.x; jb < p.n_jobs; jb += gridDim.x) {
      const XJob J = xjob_of(p, jb);
      const AttnRegion& R = p.regions[J.region];
      {
        // Q row -> TMEM (the previous job's last PV has completed: waited below)
        const float4* src = reinterpret_cast<const float4*>(R.q_tm + J.h * R.q_hs + (long long)(J.s0 + row) * R.q_rs);
#pragma unroll
        for (int c = 0; c < XD / 32; ++c) {
          uint32_t w[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 v = __ldg(src + c * 8 + q);
            w[4 * q] = __float_as_uint(v.x);
            w[4 * q + 1] = __float_as_uint(v.y);
            w[4 * q + 2] = __float_as_uint(v.z);
            w[4 * q + 3] = __float_as_uint(v.w);
          }
          tmem_st_32x32b_x32(tmem + lane_base + T_Q + uint32_t(c * 32), w);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(qt_full);
      }
      float m = 0.f, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        const int b = j & 1;
        int& sn = b ? sn1 : sn0;
        mbar_wait(&s_full[b], sn & 1);
        ++sn;
        tc_fence_after();
        uint32_t v[64];
        tmem_ld_32x32b_x32(tmem + lane_base + t_r(b, 0), *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld_32x32b_x32(tmem + lane_base + t_r(b, 0) + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_ld_wait();
        SPROF(0)
        float mx;
        {
          float a0, a1, a2, a3;
          if (sc2 >= 0.f) {
            a0 = a1 = a2 = a3 = -INFINITY;
#pragma unroll
            for (int e = 0; e < 64; e += 4) {
              a0 = fmaxf(a0, __uint_as_float(v[e]));
              a1 = fmaxf(a1, __uint_as_float(v[e + 1]));
              a2 = fmaxf(a2, __uint_as_float(v[e + 2]));
              a3 = fmaxf(a3, __uint_as_float(v[e + 3]));
            }
            mx = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)) * sc2;
          } else {
            a0 = a1 = a2 = a3 = INFINITY;
#pragma unroll
            for (int e = 0; e < 64; e += 4) {
              a0 = fminf(a0, __uint_as_float(v[e]));
              a1 = fminf(a1, __uint_as_float(v[e + 1]));
              a2 = fminf(a2, __uint_as_float(v[e + 2]));
              a3 = fminf(a3, __uint_as_float(v[e + 3]));
            }
            mx = fminf(fminf(a0, a1), fminf(a2, a3)) * sc2;
          }
        }
        // the running max, rounded up to an integer: P <= 1, f exact
        const float mn = j == 0 ? ceilf(mx) : fmaxf(m, ceilf(mx));
        const float f = j == 0 ? 1.f : pow2i(m - mn);
        m = mn;
        // P = 2^(c log2e S - m) in fp32 (registers), P - tf32(P) beside it
        float2 s0 = make_float2(0.f, 0.f), s1 = s0;
        uint32_t lo[64];
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          const float y0 = xex2(fmaf(__uint_as_float(v[e]), sc2, -m));
          const float y1 = xex2(fmaf(__uint_as_float(v[e + 1]), sc2, -m));
          v[e] = __float_as_uint(y0);
          v[e + 1] = __float_as_uint(y1);
          lo[e] = __float_as_uint(lo_part(y0));
          lo[e + 1] = __float_as_uint(lo_part(y1));
          if (e & 2) s1 = make_float2(s1.x + y0, s1.y + y1);
          else s0 = make_float2(s0.x + y0, s0.y + y1);
        }
        l = fmaf(l, f, (s0.x + s0.y) + (s1.x + s1.y));
        SPROF(1)
        // The TMEM stores wait for PV_{j-1}: measured on B200 (tools/x3_attn_debug.py),
        // tcgen05.st of P_j issued while the A-from-TMEM kind::tf32 PV_{j-1}
        // runs leaves PV_{j-1} reading stale A columns (S_{j-1} instead of
        // P_{j-1}) although the columns are disjoint; with the stores held
        // until PV_{j-1} completes every size checked is correct. TMEM loads
        // alongside it are harmless, so S_j is read and P_j computed meanwhile.
        if (j > 0) {
          mbar_wait(pv_done, uint32_t(pvn + j - 1) & 1);
          tc_fence_after();
        }
        SPROF(2)
        scl[b * XQ + row] = f;  // correction of block j-2 read it before PV_{j-1} was issued
        tmem_st_32x32b_x32(tmem + lane_base + t_r(b, 0), *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_st_32x32b_x32(tmem + lane_base + t_r(b, 0) + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_st_32x32b_x32(tmem + lane_base + t_r(b, 1), *reinterpret_cast<uint32_t(*)[32]>(lo));
        tmem_st_32x32b_x32(tmem + lane_base + t_r(b, 1) + 32u, *reinterpret_cast<uint32_t(*)[32]>(lo + 32));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&p_full[b]);
          mbar_arrive(&sc_full[b]);
        }
        SPROF(3)
      }
      lbuf[row] = l;  // the correction warps read the previous job's sums before its last o_free
      __syncwarp();
      if (lane == 0) mbar_arrive(l_ready);
      // the next job's Q store waits for this job's last PV (see above)
      mbar_wait(pv_done, uint32_t(pvn + nb - 1) & 1);
      pvn += nb;
      tc_fence_after();
    }
#if X3_PROF
    if (row == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
      printf("cta %d softmax cycles: wait S %lld compute %lld wait PV %lld store %lld\n", blockIdx.x, sp[0], sp[1],
             sp[2], sp[3]);
#endif
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kXMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

bool attn_x3_supported(int S, int T, int D) { return D == XD && S % XQ == 0 && T % XKV == 0 && T > 0; }

cudaError_t attn_x3_prepare() {
  return cudaFuncSetAttribute(attn_x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, XSMEM);
}

cudaError_t launch_attn_x3(const AttnLaunch& p0, int num_sms, cudaStream_t s) {
  AttnLaunch p = p0;
  p.n_pair_jobs = 0;
  p.n_jobs = p.n_regions * p.H * (p.S / XQ);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_jobs < num_sms ? p.n_jobs : num_sms);
  cfg.blockDim = dim3(kXThreads);
  cfg.dynamicSmemBytes = XSMEM;
  cfg.stream = s;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_x3_kernel, p);
}

}  // namespace ed
