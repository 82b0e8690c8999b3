// Fused attention block in the fp32-accurate mode (fp32x3): T1 = QK^T (+ its
// fused scale), the row softmax and O = T3 V as one tcgen05 kernel, every
// contraction as three TF32 products hi*hi + hi*lo + lo*hi (lo = x - tf32(x),
// the shadows the producers write beside Q, K and V), P computed and kept in
// fp32. The [h, s, s2] logits never reach HBM (the unfused fp32x3 path moves
// them through HBM five times: T1, softmax in/out, its lo shadow, O's reads).
//
// A job is one 128-row query tile of one head; with kCta = 2 a cluster of two
// CTAs takes two tiles of one head and the leader issues cta_group::2 MMAs
// (M = 256), each CTA loading half of every K block (its 64 keys) and half of
// every V block (64 of the d columns). Key blocks of 128 keep every MMA N = 128
// wide. Q_hi (Q itself: the MMA drops the low 13 bits) and Q_lo sit in shared
// memory (128 KiB); K_j and V_j stream through three 32 KiB slots, lo and hi
// copies in separate slots, in the order the MMA consumes them:
// K0 | K1 V0 | K2 V1 | ...  TMEM (512 columns) per CTA:
//   O_j [0,128)   S/P buffer 0 [128,256)   S/P buffer 1 [256,384)   P - tf32(P) [384,512)
// The MMAs run S_0 | S_1 PV_0 | S_2 PV_1 | ..., so S_{j+1} lands while the
// softmax works on S_j; the softmax writes P_j over S_j's columns at once and
// P_j - tf32(P_j) (one buffer) once PV_{j-1} has read the previous one.
// Promoted accumulation: every PV_j starts a fresh TMEM accumulator O_j, and
// the correction warps fold it into fp32 running sums in registers with IEEE
// operations, O = f_j O + O_j (the tensor core's truncating accumulation is
// confined to one key block's products, as in the x3 GEMM). The softmax keeps
// the exact running row max m (log2 domain, rounded up to an integer), so
// P <= 1 and f_j = 2^(m_{j-1} - m_j) is exact.
//
// Warps: 0-3 softmax (warp w: TMEM lanes 32w..32w+31, one thread per row),
// 4-7 correction + epilogue (same rows), 8 TMEM allocator + MMA issuer, 9 TMA,
// 10-11 idle.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "attn_sm100.h"
#include "ptx.cuh"

namespace ed {

namespace {

constexpr int XQ = 128;   // query rows per CTA
constexpr int XKV = 128;  // keys per block
constexpr int XD = 128;   // head dim
constexpr int kXThreads = 384;  // three warpgroups: one warp of each on every 16K-register sub-partition
constexpr int kXCorrWarp0 = 4, kXMmaWarp = 8, kXTmaWarp = 9;
// setmaxnreg: the correction warpgroup holds each row's 128 running sums;
// the producer warpgroup (MMA, TMA, two idle warps) gives registers back.
// Per sub-partition: 168 (softmax) + 232 + 96 <= 512 per lane.
constexpr int kXCorrRegs = 232, kXProdRegs = 96;
constexpr int XQ_BYTES = XQ * XD * 4;   // per Q copy: 4 K-major chunks of 128 rows x 128 B
// a slot: kCta 1, half of one block's K or V copy (K: d chunks 2h, 2h+1 of the
// 128 keys; V: keys 64h.. for all d); kCta 2, this CTA's whole half of a copy
// (K: its 64 keys, all d; V: all 128 keys, its 64 d)
constexpr int XSLOT = 32768;
constexpr int XNSLOT = 3;
constexpr int XBAR_BYTES = 256;
constexpr int XSMEM = 2 * XQ_BYTES + XNSLOT * XSLOT + XBAR_BYTES + 3 * XQ * 4 + 1024;
static_assert(XSMEM <= 232448, "shared memory");
constexpr uint32_t T_O = 0, T_PL = 384;
__device__ __forceinline__ uint32_t t_s(int b) { return 128u + 128u * uint32_t(b); }

struct XJob {
  int region, h, s0;
};

// job j: kCta consecutive 128-row query tiles of one head, CTA `rank` of the
// cluster taking tile rank
template <int kCta>
__device__ __forceinline__ XJob xjob_of(const AttnLaunch& p, int j, uint32_t rank) {
  const int jph = p.S / (XQ * kCta);
  const int rh = j / jph;
  XJob r;
  r.region = rh / p.H;
  r.h = rh % p.H;
  r.s0 = (j % jph) * XQ * kCta + int(rank) * XQ;
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

template <int kCta>
__global__ void __launch_bounds__(kXThreads, 1) attn_x3_kernel(const __grid_constant__ AttnLaunch p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;             // Q_lo
  uint8_t* sQh = sQ + XQ_BYTES;   // Q (the hi operand)
  uint8_t* sKV = sQh + XQ_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sKV + XNSLOT * XSLOT);
  uint64_t* q_full = bar + 0;      // TMA -> MMA: Q_lo and Q in smem
  uint64_t* q_empty = bar + 1;     // MMA -> TMA: the job's last S done
  uint64_t* s_full = bar + 2;      // [2] MMA -> softmax: S_j in buffer j & 1
  // [2] softmax -> MMA: P_j stored (block parity: a softmax warp may finish
  // block j+1 before another has finished block j)
  uint64_t* p_full = bar + 4;
  uint64_t* sc_full = bar + 6;     // [2] softmax -> correction: f_j posted (block parity)
  uint64_t* pv_done = bar + 8;     // MMA -> softmax, correction: P V_j in O_j
  uint64_t* o_free = bar + 9;      // correction -> MMA: O_j folded into the running sums
  uint64_t* l_ready = bar + 10;    // softmax -> correction: the job's row sums posted
  uint64_t* slot_full = bar + 11;  // [XNSLOT]
  uint64_t* slot_empty = slot_full + XNSLOT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slot_empty + XNSLOT);
  static_assert((11 + 2 * XNSLOT) * 8 + 4 <= XBAR_BYTES, "barrier space");
  float* scl = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bar) + XBAR_BYTES);  // [2][XQ] f_j per row
  float* lbuf = scl + 2 * XQ;                                                           // [XQ] row sums

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = p.T / XKV;
  const uint32_t rank = kCta == 2 ? cluster_ctarank() : 0;
  const int first = blockIdx.x / kCta, stride = gridDim.x / kCta;
  // arrive on the leader CTA's copy of a barrier (the MMA issuer's)
  auto arrive_leader = [&](uint64_t* b) {
    if (kCta == 2) mbar_arrive_cluster(mapa(smem_u32(b), 0));
    else mbar_arrive(b);
  };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4 * kCta);
      mbar_init(&sc_full[i], 4);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_free, 4 * kCta);
    mbar_init(l_ready, 4);
    for (int i = 0; i < XNSLOT; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kXMmaWarp) tmem_alloc<512, kCta>(tmem_slot);
  tc_fence_before();
  if (kCta == 2) cluster_sync();
  else __syncthreads();
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
      // kCta = 2: data lands in this CTA's smem, the bytes count on the leader's barrier
      auto load = [&](void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
        if (kCta == 2) tma_load_3d_2sm(dst, m, b, c0, c1, c2);
        else tma_load_3d(dst, m, b, c0, c1, c2);
      };
      for (int jb = first; jb < p.n_jobs; jb += stride) {
        if (jb + stride >= p.n_jobs) griddep_launch();
        const XJob J = xjob_of<kCta>(p, jb, rank);
        const AttnRegion& R = p.regions[J.region];
        auto src_map = [&](const AttnSrc& a, int key, int dcol) {
          return p.maps + a.base + (key / a.keys) * a.nd + dcol / a.dw;
        };
        mbar_wait(q_empty, (qn & 1) ^ 1);
        ++qn;
        if (rank == 0) mbar_expect_tx(q_full, 2 * XQ_BYTES * kCta);
#pragma unroll
        for (int c = 0; c < XD / 32; ++c) {
          load(sQ + c * 16384, p.maps + R.q, q_full, c * 32, J.s0, J.h);
          load(sQh + c * 16384, p.maps + R.q + 1, q_full, c * 32, J.s0, J.h);
        }
        auto load_k = [&](int j) {
          // K_j: lo then hi. kCta 1: two slots per copy, d chunks {0,1} / {2,3} of the
          // 128 keys (16 KiB each); kCta 2: one slot, this CTA's 64 keys, all four chunks (8 KiB)
          for (int part = 1; part >= 0; --part)
            for (int hf = 0; hf < 2 / kCta; ++hf) {
              const int st = slot_get();
              uint8_t* dst = sKV + st * XSLOT;
              if (rank == 0) mbar_expect_tx(&slot_full[st], XSLOT * kCta);
              const int key = j * XKV + int(rank) * (XKV / kCta);
#pragma unroll
              for (int c = 0; c < 2 * kCta; ++c) {
                const int dc = kCta == 1 ? 2 * hf + c : c;
                load(dst + c * (XSLOT / (2 * kCta)), src_map(R.k, key, dc * 32) + part * R.k.lo, &slot_full[st],
                     (dc * 32) % R.k.dw, key % R.k.keys, J.h + R.k.hoff);
              }
            }
        };
        auto load_v = [&](int j) {
          // V_j: lo then hi, MN atoms of 32 keys x 32 d. kCta 1: two slots per copy
          // (keys 64 hf..: 2 quarters x 4 atoms); kCta 2: one slot (4 quarters x this CTA's 2 atoms)
          for (int part = 1; part >= 0; --part)
            for (int hf = 0; hf < 2 / kCta; ++hf) {
              const int st = slot_get();
              uint8_t* dst = sKV + st * XSLOT;
              if (rank == 0) mbar_expect_tx(&slot_full[st], XSLOT * kCta);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int quarter = kCta == 1 ? 2 * hf + i / 4 : i / 2;
                const int a = kCta == 1 ? i % 4 : int(rank) * 2 + i % 2;
                const int key = j * XKV + quarter * 32;
                load(dst + i * 4096, src_map(R.v, key, a * 32) + part * R.v.lo, &slot_full[st], (a * 32) % R.v.dw,
                     key % R.v.keys, J.h + R.v.hoff);
              }
            }
        };
        load_k(0);  // the MMA's consumption order: K0 | K1 V0 | K2 V1 | ...
        for (int j = 0; j < nb; ++j) {
          if (j + 1 < nb) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp == kXMmaWarp) {
    if (rank != 0) goto done;  // the pair's MMAs are issued by the leader
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    const uint32_t idesc_s = umma_idesc(2u, XQ * kCta, XKV, 0u, 0u);  // Q, K both K-major (d)
    const uint32_t idesc_o = umma_idesc(2u, XQ * kCta, XD, 0u, 1u);   // P from TMEM (keys), V MN-major (d)
    auto mma_ss = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
      if (kCta == 2) mma_tf32_2sm_warp(d, a, b, id, acc);
      else mma_tf32_warp(d, a, b, id, acc);
    };
    auto mma_ts = [&](uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
      if (kCta == 2) mma_tf32_ts_2sm_warp(d, a, b, id, acc);
      else mma_tf32_ts_warp(d, a, b, id, acc);
    };
    auto commit = [&](uint64_t* b) {
      if (kCta == 2) mma_commit_2sm_warp(b);
      else mma_commit_warp(b);
    };
    auto wait_arrivals = [&](uint64_t* b, uint32_t ph) {  // arrivals from both CTAs' warps
      if (kCta == 2) mbar_wait_cluster(b, ph);
      else mbar_wait(b, ph);
    };
    int sn = 0, qn = 0, pn0 = 0, pn1 = 0, on = 0;
    auto take = [&]() {
      const int st = sn % XNSLOT;
      mbar_wait(&slot_full[st], (sn / XNSLOT) & 1);
      ++sn;
      return st;
    };
    const uint64_t qd = umma_desc_sw128(smem_u32(sQ), 16, 1024);    // Q_lo
    const uint64_t qhd = umma_desc_sw128(smem_u32(sQh), 16, 1024);  // Q (hi)
    // K slot: kCta 1, two chunks of 128 keys x 128 B (16 KiB) of d chunks 2 hf, 2 hf + 1;
    // kCta 2, four chunks of 64 keys x 128 B (8 KiB). A K step = 8 d = 32 B of a chunk row.
    constexpr int KCH = XSLOT / (2 * kCta);
    auto k_off = [&](int k, int hf) { return uint64_t((((k / 4) - 2 * hf) * KCH + (k % 4) * 32) >> 4); };
    constexpr int KSTEPS = XD / 8 / (2 / kCta);  // K steps per K slot
    auto issue_s = [&](int b) {
      const uint32_t d = tmem + t_s(b);
#pragma unroll
      for (int hf = 0; hf < 2 / kCta; ++hf) {  // Q_hi K_lo
        const int kl = take();
        tc_fence_after();
        const uint64_t kld = umma_desc_sw128(smem_u32(sKV + kl * XSLOT), 16, 1024);
#pragma unroll
        for (int k = KSTEPS * hf; k < KSTEPS * (hf + 1); ++k) {
          const uint64_t qo = uint64_t(((k / 4) * 16384 + (k % 4) * 32) >> 4);
          mma_ss(d, qhd + qo, kld + k_off(k, kCta == 1 ? hf : 0), idesc_s, k != 0);
        }
        commit(&slot_empty[kl]);
      }
#pragma unroll
      for (int hf = 0; hf < 2 / kCta; ++hf) {  // Q_lo K_hi + Q_hi K_hi
        const int kh = take();
        tc_fence_after();
        const uint64_t khd = umma_desc_sw128(smem_u32(sKV + kh * XSLOT), 16, 1024);
#pragma unroll
        for (int k = KSTEPS * hf; k < KSTEPS * (hf + 1); ++k) {
          const uint64_t qo = uint64_t(((k / 4) * 16384 + (k % 4) * 32) >> 4);
          const uint64_t ko = k_off(k, kCta == 1 ? hf : 0);
          mma_ss(d, qd + qo, khd + ko, idesc_s, 1u);
          mma_ss(d, qhd + qo, khd + ko, idesc_s, 1u);
        }
        commit(&slot_empty[kh]);
      }
      commit(&s_full[b]);
    };
    // V slot: 8 MN atoms of 32 keys x 128 B. kCta 1: [key quarter (2)][d atom (4)];
    // kCta 2: [key quarter (4)][this CTA's d atom (2)]. A K step = 8 keys.
    constexpr int QB = kCta == 1 ? 16384 : 8192;  // bytes per key quarter in a slot
    constexpr int VSTEPS = XKV / 8 / (2 / kCta);  // K steps per V slot
    auto v_off = [&](int k) { return uint64_t((((k % VSTEPS) / 4) * QB + (k % 4) * 1024) >> 4); };
    auto issue_pv = [&](int b) {
      const uint32_t ph = tmem + t_s(b), pl = tmem + T_PL;
#pragma unroll
      for (int hf = 0; hf < 2 / kCta; ++hf) {  // P_hi V_lo, a fresh O_j
        const int vl = take();
        tc_fence_after();
        const uint64_t vld = umma_desc_sw128(smem_u32(sKV + vl * XSLOT), 4096, 512, 1);
#pragma unroll
        for (int k = VSTEPS * hf; k < VSTEPS * (hf + 1); ++k)
          mma_ts(tmem + T_O, ph + uint32_t(k * 8), vld + v_off(k), idesc_o, k != 0);
        commit(&slot_empty[vl]);
      }
#pragma unroll
      for (int hf = 0; hf < 2 / kCta; ++hf) {  // P_lo V_hi + P_hi V_hi
        const int vh = take();
        tc_fence_after();
        const uint64_t vhd = umma_desc_sw128(smem_u32(sKV + vh * XSLOT), 4096, 512, 1);
#pragma unroll
        for (int k = VSTEPS * hf; k < VSTEPS * (hf + 1); ++k) {
          mma_ts(tmem + T_O, pl + uint32_t(k * 8), vhd + v_off(k), idesc_o, 1u);
          mma_ts(tmem + T_O, ph + uint32_t(k * 8), vhd + v_off(k), idesc_o, 1u);
        }
        commit(&slot_empty[vh]);
      }
      commit(pv_done);
    };
    for (int jb = first; jb < p.n_jobs; jb += stride) {
      mbar_wait(q_full, qn & 1);
      ++qn;
      tc_fence_after();
      issue_s(0);
      if (nb == 1) commit(q_empty);
      for (int j = 0; j < nb; ++j) {
        const int b = j & 1;
        if (j + 1 < nb) {
          // S_{j+1} overwrites the buffer PV_{j-1} read: issued after it, so in order
          issue_s(b ^ 1);
          if (j + 1 == nb - 1) commit(q_empty);
        }
        int& pn = b ? pn1 : pn0;
        wait_arrivals(&p_full[b], pn & 1);
        ++pn;
        if (on > 0) wait_arrivals(o_free, (on - 1) & 1);  // the correction warps have read O_{j-1}
        ++on;
        tc_fence_after();
        issue_pv(b);
      }
    }
  } else if (warp >= kXCorrWarp0) {
    // ---------------- correction: O = f_j O + O_j in registers, then the epilogue ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kXCorrRegs));
    const int wq = warp - kXCorrWarp0;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    int pvn = 0, sc0 = 0, sc1 = 0, ln = 0;
    for (int jb = first; jb < p.n_jobs; jb += stride) {
      const XJob J = xjob_of<kCta>(p, jb, rank);
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
        if (lane == 0) arrive_leader(o_free);
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
    for (int jb = first; jb < p.n_jobs; jb += stride) {
      float m = 0.f, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        const int b = j & 1;
        int& sn = b ? sn1 : sn0;
        mbar_wait(&s_full[b], sn & 1);
        ++sn;
        tc_fence_after();
        const uint32_t ts = tmem + lane_base + t_s(b);
        // row max of c log2e S over the 128 keys, 32 columns at a time
        float mx = sc2 >= 0.f ? -INFINITY : INFINITY;
#pragma unroll 1
        for (int c = 0; c < XKV / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ts + uint32_t(c * 32), v);
          tmem_ld_wait();
          float a0 = __uint_as_float(v[0]), a1 = __uint_as_float(v[1]);
#pragma unroll
          for (int e = 2; e < 32; e += 2) {
            a0 = sc2 >= 0.f ? fmaxf(a0, __uint_as_float(v[e])) : fminf(a0, __uint_as_float(v[e]));
            a1 = sc2 >= 0.f ? fmaxf(a1, __uint_as_float(v[e + 1])) : fminf(a1, __uint_as_float(v[e + 1]));
          }
          mx = sc2 >= 0.f ? fmaxf(mx, fmaxf(a0, a1)) : fminf(mx, fminf(a0, a1));
        }
        mx *= sc2;
        // the running max, rounded up to an integer: P <= 1, f exact
        const float mn = j == 0 ? ceilf(mx) : fmaxf(m, ceilf(mx));
        const float f = j == 0 ? 1.f : pow2i(m - mn);
        m = mn;
        // P = 2^(c log2e S - m) in fp32 over S's columns (its own buffer: at once)
        float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll 1  // one 32-column slice live at a time
        for (int c = 0; c < XKV / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ts + uint32_t(c * 32), v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float y0 = xex2(fmaf(__uint_as_float(v[e]), sc2, -m));
            const float y1 = xex2(fmaf(__uint_as_float(v[e + 1]), sc2, -m));
            v[e] = __float_as_uint(y0);
            v[e + 1] = __float_as_uint(y1);
            if (e & 2) s1 = make_float2(s1.x + y0, s1.y + y1);
            else s0 = make_float2(s0.x + y0, s0.y + y1);
          }
          tmem_st_32x32b_x32(ts + uint32_t(c * 32), v);
        }
        l = fmaf(l, f, (s0.x + s0.y) + (s1.x + s1.y));
        // P - tf32(P) goes to the one P_lo buffer, which PV_{j-1} reads
        if (j > 0 || jb != first) {
          mbar_wait(pv_done, uint32_t(pvn - 1) & 1);
          tc_fence_after();
        }
        tmem_st_wait();
#pragma unroll 1
        for (int c = 0; c < XKV / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ts + uint32_t(c * 32), v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(lo_part(__uint_as_float(v[e])));
          tmem_st_32x32b_x32(tmem + lane_base + T_PL + uint32_t(c * 32), v);
        }
        ++pvn;
        scl[b * XQ + row] = f;  // the correction of block j-2 read it before PV_{j-1} was issued
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          arrive_leader(&p_full[b]);
          mbar_arrive(&sc_full[b]);
        }
      }
      lbuf[row] = l;  // the correction warps read the previous job's sums before its last o_free
      __syncwarp();
      if (lane == 0) mbar_arrive(l_ready);
    }
  }

done:
  tc_fence_before();
  if (kCta == 2) cluster_sync();
  else __syncthreads();
  if (warp == kXMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512, kCta>(tmem);
  }
}

}  // namespace

bool attn_x3_supported(int S, int T, int D) { return D == XD && S % XQ == 0 && T % XKV == 0 && T > 0; }

int attn_x3_cta(int S) {
  static const int force = [] {
    const char* e = std::getenv("ED_ATTN_X3_CTA");
    return e ? std::atoi(e) : 0;
  }();
  if (force == 1) return 1;
  return S % (2 * XQ) == 0 ? 2 : 1;
}

cudaError_t attn_x3_prepare() {
  cudaError_t e = cudaFuncSetAttribute(attn_x3_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, XSMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_x3_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, XSMEM);
}

cudaError_t launch_attn_x3(const AttnLaunch& p0, int num_sms, cudaStream_t s) {
  AttnLaunch p = p0;
  const int cta = attn_x3_cta(p.S);
  p.n_pair_jobs = 0;
  p.n_jobs = p.n_regions * p.H * (p.S / (XQ * cta));  // one job per cluster: cta query tiles
  const int clusters = p.n_jobs < num_sms / cta ? p.n_jobs : num_sms / cta;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * cta);
  cfg.blockDim = dim3(kXThreads);
  cfg.dynamicSmemBytes = XSMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cta;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cta == 2 ? cudaLaunchKernelEx(&cfg, attn_x3_kernel<2>, p) : cudaLaunchKernelEx(&cfg, attn_x3_kernel<1>, p);
}

}  // namespace ed
