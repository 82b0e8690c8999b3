// Block contractions of mul/sum joins on the 5th-gen tensor cores.
//
// Replaces kernel_eval's mul/sum case (kernel.cc:48-65). One persistent
// launch covers every output region of one einsum on this rank; each region
// is C = sum_s A_s * B_s over its aggregation siblings s (the join tuples its
// refinement folds, runtime.cc:242-261), K-concatenated so the fold happens
// in the TMEM accumulator and no partial ever reaches HBM.
//
// Label permutations are folded into 3-D TMA tensor maps {inner, outer,
// batch} — K-major or MN-major per operand — so no transpose copy runs.
// kCta = 2 pairs two SMs as one cluster (tcgen05 cta_group::2): a 256xBN
// tile per pair, each CTA loading half of A and half of B, so per-SM operand
// traffic drops by a third. BN = 256, or 128 for launches too small to
// fill half the grid with 256-wide tiles (gemm_pick_bn).
// Warp roles (192 threads, 1 CTA per SM):
//   warp 0     TMA producer over a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  epilogue: TMEM -> registers -> HBM (fp32 and/or bf16 shadow)
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap
// the MMAs of tile i+1. Tiles are scheduled round-robin over the grid.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "gemm_sm100.h"
#include "ptx.cuh"

namespace ed {

namespace {

constexpr int BM = 128;  // accumulator rows per CTA (TMEM lanes)
// accumulator columns per tile (BN): 256, or 128 for launches too small to
// fill half the grid (gemm_pick_bn)
constexpr int kThreads = 192;
constexpr int kAccStages = 2;

template <bool kBF16, int kCta, int BN, bool kX3 = false>
struct Cfg {
  static constexpr int ES = kBF16 ? 2 : 4;          // element bytes
  static constexpr int BK = 128 / ES;               // one 128-byte swizzle row of K
  static constexpr int UMMA_K = kBF16 ? 16 : 8;     // 32 bytes of K per MMA
  static constexpr int TILE_M = BM * kCta;          // output rows per cluster tile
  static constexpr int B_ROWS = BN / kCta;          // B rows (N) loaded per CTA
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = B_ROWS * 128;
  // kX3 (fp32-accurate 3xTF32): a stage holds A_hi | B_hi | A_lo | B_lo and
  // feeds three products hi*hi + hi*lo + lo*hi into the same accumulator
  static constexpr int LO_OFF = A_BYTES + B_BYTES;  // offset of the lo copies in a stage
  static constexpr int NPROD = kX3 ? 3 : 1;
  static constexpr int NMAP = kX3 ? 4 : 2;          // tensor maps per sibling
  static constexpr int STAGE_BYTES = (kX3 ? 2 : 1) * (A_BYTES + B_BYTES);
  static constexpr int STAGES = 196608 / STAGE_BYTES > 8 ? 8 : 196608 / STAGE_BYTES;  // 192 KiB ring
  static constexpr int STORE_BYTES = 4 * 2 * 4096;  // 4 epilogue warps x 2 staging tiles of 32x128 B
  static constexpr int SMEM = STAGES * STAGE_BYTES + STORE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int MN_ATOM = 128 / ES;          // MN elements per 128-byte atom
  static_assert(SMEM <= 232448, "shared memory");
};

struct TileCoord {
  int region, b, m0, n0;
};

template <int TILE_M, int BN>
__device__ __forceinline__ TileCoord tile_coord(const GemmLaunch& p, int t, int tiles_m, int tiles_n) {
  TileCoord c;
  const int per_batch = tiles_m * tiles_n;
  int r;
  if (p.region_inner) {
    // batch-major over the regions: the regions' tiles of one batch run
    // together, so a B operand all regions share (C2's repartitioned Z2
    // reading W) leaves HBM once per batch instead of once per region
    const int per_b = per_batch * p.n_regions;
    c.b = t / per_b;
    r = t - c.b * per_b;
    c.region = r / per_batch;
    r -= c.region * per_batch;
  } else {
    const int per_region = per_batch * p.batch;
    c.region = t / per_region;
    r = t - c.region * per_region;
    c.b = r / per_batch;
    r -= c.b * per_batch;
  }
  // grouped raster: kGroupM tile rows advance together along N, so one wave
  // of ~74 cluster tiles touches ~8 A panels + ~9 B panels instead of
  // 3 + tiles_n, and the panels it shares stay in L2 (hoc: 8192^2 tiles)
  const int kGroupM = p.group_m;
  const int g = r / (kGroupM * tiles_n);
  const int gm0 = g * kGroupM;
  const int gsz = tiles_m - gm0 < kGroupM ? tiles_m - gm0 : kGroupM;
  const int rg = r - g * kGroupM * tiles_n;
  c.m0 = (gm0 + rg % gsz) * TILE_M;
  c.n0 = (rg / gsz) * BN;
  return c;
}

// unary map of a fused consumer vertex (ops.cc:18-28) on 32 accumulator
// values; the op is uniform, so branch once outside the unrolled loops.
__device__ __forceinline__ void epi32(const GemmLaunch& p, uint32_t* r) {
  const int op = p.epi_map;
  const float c = p.epi_c;
  if (op == 0) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float x = __uint_as_float(r[j]);
      r[j] = __float_as_uint(x > 0.0f ? x : 0.0f);
    }
  } else if (op == 2) {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] ^= 0x80000000u;
  } else if (op == 3) {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(c * __uint_as_float(r[j]));
  }
}

// Loose lockstep of the TMA producers (GemmLaunch::sync): before issuing its
// K block k, a CTA announces the epoch it finished (sync_g K blocks each) and
// waits until every CTA of the grid has issued epoch e - sync_lag, so the
// grid's CTAs stay within ~sync_lag epochs of each other along K and the A /
// B panels one wave shares are still in L2 when the slower CTAs read them
// (hoc fp32x3: DRAM reads 89 -> 37 GB per launch). A wait that exceeds 200 us
// (CTAs not co-resident, e.g. other kernels on the SMs) switches the wait
// off for the rest of the launch: a hint, never a hang.
__device__ __forceinline__ void producer_lockstep(const GemmLaunch& p, int k, bool& on) {
  if (k % p.sync_g) return;
  const int e = k / p.sync_g;
  if (e > 0) atomicAdd(&p.sync[e - 1], 1u);  // this CTA has issued epoch e - 1
  if (!on || e < p.sync_lag) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sync + (e - p.sync_lag)) : "memory");
    if (v >= gridDim.x) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 200000ull) {
      on = false;
      return;
    }
    __nanosleep(64);
  }
}

// After the producer's last load: epochs this CTA never issues count as
// issued; the last CTA out re-zeroes the counters for the op's next launch.
__device__ __forceinline__ void producer_lockstep_exit(const GemmLaunch& p, int issued) {
  for (int e = (issued + p.sync_g - 1) / p.sync_g - 1; e < p.sync_epochs; ++e)
    if (e >= 0) atomicAdd(&p.sync[e], 1u);
  if (atomicAdd(&p.sync[p.sync_epochs], 1u) == gridDim.x - 1) {
    __threadfence();
    for (int e = 0; e <= p.sync_epochs; ++e) atomicExch(&p.sync[e], 0u);
  }
}

// kMc = 2: two 2-SM pairs form one 4-CTA cluster over a 256 x 2BN tile; they
// share the A panel, each pair loading half of every A box and multicasting it
// to both pairs, so each A byte leaves L2 once per cluster instead of twice.
template <bool kBF16, int kCta, int BN, bool kX3, int kMc>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmLaunch p) {
  using C_ = Cfg<kBF16, kCta, BN, kX3>;
  static_assert(kMc == 1 || kCta == 2, "A multicast pairs 2-SM tiles");
  constexpr int kClu = kCta * kMc;  // CTAs per cluster
  constexpr int STAGES = C_::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_out = smem + STAGES * C_::STAGE_BYTES;  // epilogue staging (1024-aligned)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stage_out + C_::STORE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* acc_full = empty_bar + STAGES;
  uint64_t* acc_empty = acc_full + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kAccStages);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = kClu > 1 ? cluster_ctarank() : 0;
  const uint32_t rank = kCta == 2 ? (crank & 1u) : 0u;  // CTA within its MMA pair
  const uint32_t q = kCta == 2 ? (crank >> 1) : 0u;     // pair within the cluster (kMc)
  const int tiles_m = (p.M + C_::TILE_M - 1) / C_::TILE_M;
  const int tiles_n = (p.N + BN * kMc - 1) / (BN * kMc);  // cluster tiles along N
  const int total = tiles_m * tiles_n * p.batch * p.n_regions;
  const int kblocks = (p.K + C_::BK - 1) / C_::BK;
  const int first = blockIdx.x / kClu, stride = gridDim.x / kClu;
  auto coord = [&](int t) {
    TileCoord c = tile_coord<C_::TILE_M, BN * kMc>(p, t, tiles_m, tiles_n);
    c.n0 += int(q) * BN;
    return c;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kMc);  // one MMA commit per pair reading this stage
    }
    for (int s = 0; s < kAccStages; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4 * kCta);  // one arrive per epilogue warp of the pair
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kAccStages * BN, kCta>(tmem_slot);
  tc_fence_before();
  if (kClu > 1) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // everything above overlaps the previous kernel's tail (PDL); operands and
  // outputs are touched only after it has completed
  griddep_wait();

  if (warp == 0) {
    // ---- TMA producer (both CTAs of a pair load their halves) ----
    if (lane == 0) {
      int it = 0, ti = 0;
      bool sync_on = p.sync != nullptr;
      for (int t = first; t < total; t += stride, ++ti) {
        if (t + stride >= total) griddep_launch();  // last tile: the next kernel may launch
        const TileCoord tc = coord(t);
        const bool back = p.serp && (ti & 1);  // serpentine K (see gemm_x3_kernel)
        const GemmRegion reg = p.regions[tc.region];
        const int am = tc.m0 + int(rank) * BM, bn = tc.n0 + int(rank) * C_::B_ROWS;
        // kMc: CTAs with the same rank in both pairs hold the same A rows
        const uint16_t a_mask = uint16_t((1u << rank) | (1u << (2 + rank)));
        // batch coordinates of A and B (a batch-segmented operand: its segment's)
        const int bseg_i = reg.bseg ? tc.b / reg.bseg : 0;
        const int ba = reg.bseg && !reg.bseg_b ? tc.b % reg.bseg : tc.b;
        const int bb = reg.bseg && reg.bseg_b ? tc.b % reg.bseg : tc.b;
        for (int si = 0; si < reg.n_sib; ++si) {
          const int sib = back ? reg.n_sib - 1 - si : si;
          const CUtensorMap* ma = p.maps + reg.map0 + C_::NMAP * (bseg_i * reg.n_sib + sib);
          const CUtensorMap* mb = ma + 1;
          for (int kq = 0; kq < kblocks; ++kq, ++it) {
            const int kb = back ? kblocks - 1 - kq : kq;
            if (p.sync) producer_lockstep(p, it, sync_on);
            const int s = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            mbar_wait(&empty_bar[s], ph ^ 1);
            const int k0 = kb * C_::BK;
            uint8_t* sa = smem + s * C_::STAGE_BYTES;
            uint8_t* sb = sa + C_::A_BYTES;
            if (rank == 0) mbar_expect_tx(&full_bar[s], C_::STAGE_BYTES * kCta);
            auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1, int cb) {
              if (kCta == 2) tma_load_3d_2sm(dst, m, &full_bar[s], c0, c1, cb);
              else tma_load_3d(dst, m, &full_bar[s], c0, c1, cb);
            };
#pragma unroll
            for (int part = 0; part < (kX3 ? 2 : 1); ++part) {  // hi, then (kX3) lo copies
              uint8_t* pa = sa + part * C_::LO_OFF;
              uint8_t* pb = sb + part * C_::LO_OFF;
              const CUtensorMap* pma = ma + 2 * part;
              const CUtensorMap* pmb = mb + 2 * part;
              if (kMc == 2) {
                // this pair's half of the A box, multicast to both pairs (K-major:
                // 64 of the 128 rows; MN-major: half of the 128-byte MN atoms)
                if (!p.a_mn) {
                  tma_load_3d_2sm_mc(pa + q * (BM / 2) * 128, pma, &full_bar[s], k0, am + int(q) * (BM / 2), ba,
                                     a_mask);
                } else {
                  constexpr int NA = BM / C_::MN_ATOM;
#pragma unroll
                  for (int i = int(q) * NA / 2; i < (int(q) + 1) * NA / 2; ++i)
                    tma_load_3d_2sm_mc(pa + i * C_::BK * 128, pma, &full_bar[s], am + i * C_::MN_ATOM, k0, ba,
                                       a_mask);
                }
              } else if (!p.a_mn) {
                load(pa, pma, k0, am, ba);
              } else {
#pragma unroll
                for (int i = 0; i < BM / C_::MN_ATOM; ++i) load(pa + i * C_::BK * 128, pma, am + i * C_::MN_ATOM, k0, ba);
              }
              if (!p.b_mn) {
                load(pb, pmb, k0, bn, bb);
              } else {
#pragma unroll
                for (int i = 0; i < C_::B_ROWS / C_::MN_ATOM; ++i)
                  load(pb + i * C_::BK * 128, pmb, bn + i * C_::MN_ATOM, k0, bb);
              }
            }
          }
        }
      }
      if (p.sync) producer_lockstep_exit(p, it);
    }
  } else if (warp == 1) {
    // ---- MMA issuer (the leader CTA's warp 1; one elected lane issues) ----
    if (rank == 0) {  // the whole warp runs the loop (uniform values), one elected lane issues
      const uint32_t idesc = umma_idesc(kBF16 ? 1u : 2u, BM * kCta, BN, p.a_mn, p.b_mn);
      // K-major: 8-row x 128-byte swizzle atoms stacked along MN (SBO 1024),
      // K advances 32 bytes per MMA inside the atom.
      // MN-major: 128-byte MN atoms of BK K-rows (LBO = BK*128), 8-row K
      // groups (SBO 1024), K advances UMMA_K rows per MMA.
      // MN-major tf32 uses the 32B-atom swizzle: K groups of 4 rows (SBO 512).
      const uint32_t a_lbo = p.a_mn ? C_::BK * 128 : 16, b_lbo = p.b_mn ? C_::BK * 128 : 16;
      const uint32_t a_step = p.a_mn ? C_::UMMA_K * 128 : 32, b_step = p.b_mn ? C_::UMMA_K * 128 : 32;
      const uint32_t a_lt = (!kBF16 && p.a_mn) ? 1u : 2u, b_lt = (!kBF16 && p.b_mn) ? 1u : 2u;
      const uint32_t a_sbo = a_lt == 1 ? 512u : 1024u, b_sbo = b_lt == 1 ? 512u : 1024u;
      int it = 0, local = 0;
      for (int t = first; t < total; t += stride, ++local) {
        const TileCoord tc = coord(t);
        const int n_sib = p.regions[tc.region].n_sib;
        const int as = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        if (kCta == 2) mbar_wait_cluster(&acc_empty[as], aph ^ 1);
        else mbar_wait(&acc_empty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(as * BN);
        const int iters = kblocks * n_sib;
        for (int i = 0; i < iters; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * C_::STAGE_BYTES);
          const uint32_t sb = sa + C_::A_BYTES;
#pragma unroll
          for (int k = 0; k < C_::NPROD * (C_::BK / C_::UMMA_K); ++k) {
            // kX3: k-steps of hi*hi, then hi*lo, then lo*hi over the same stage
            const int prod = k / (C_::BK / C_::UMMA_K), kk = k % (C_::BK / C_::UMMA_K);
            const uint32_t oa = prod == 2 ? uint32_t(C_::LO_OFF) : 0u, ob = prod == 1 ? uint32_t(C_::LO_OFF) : 0u;
            const uint64_t ad = umma_desc_sw128(sa + oa + kk * a_step, a_lbo, a_sbo, a_lt);
            const uint64_t bd = umma_desc_sw128(sb + ob + kk * b_step, b_lbo, b_sbo, b_lt);
            const uint32_t acc = (i | k) != 0;
            if (kCta == 2) {
              if (kBF16) mma_f16_2sm_warp(d_tmem, ad, bd, idesc, acc);
              else mma_tf32_2sm_warp(d_tmem, ad, bd, idesc, acc);
            } else {
              if (kBF16) mma_f16_warp(d_tmem, ad, bd, idesc, acc);
              else mma_tf32_warp(d_tmem, ad, bd, idesc, acc);
            }
          }
          // the stage is free once every pair that reads it has consumed it
          if (kCta == 2) mma_commit_2sm_warp(&empty_bar[s], kMc == 2 ? 0xF : 0x3);
          else mma_commit_warp(&empty_bar[s]);
        }
        if (kCta == 2) mma_commit_2sm_warp(&acc_full[as], uint16_t(0x3u << (2 * q)));
        else mma_commit_warp(&acc_full[as]);
      }
    }
  } else {
    // ---- epilogue: TMEM -> registers -> HBM (each CTA its 128 rows) ----
    const int wq = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t empty_leader = kCta == 2 ? mapa(smem_u32(acc_empty), 2 * q) : 0;
    int local = 0;
    uint32_t stage_ctr = 0;
    for (int t = first; t < total; t += stride, ++local) {
      const TileCoord tc = coord(t);
      const GemmRegion reg = p.regions[tc.region];
      const int as = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&acc_full[as], aph);
      tc_fence_after();
      const int row = tc.m0 + int(rank) * BM + wq * 32 + lane;
      const long long base = (long long)tc.b * p.c_sb + (long long)row * p.c_sm;
      float* c32 = reg.c32 ? reg.c32 + base : nullptr;
      __nv_bfloat16* c16 = reg.c16 ? static_cast<__nv_bfloat16*>(reg.c16) + base : nullptr;
      const uint32_t tbase = tmem + (uint32_t(wq * 32) << 16) + uint32_t(as * BN);
      if (reg.cmap32 >= 0 || reg.cmap16 >= 0) {
        // TMEM -> registers -> 128B-swizzled smem tile -> TMA store (full lines,
        // clipped at the region bounds); two staging tiles per warp alternate.
        const int trow = tc.m0 + int(rank) * BM + wq * 32;
        for (int pass = 0; pass < 2; ++pass) {
          const int cm = pass == 0 ? reg.cmap32 : reg.cmap16;
          if (cm < 0) continue;
          const int cols = pass == 0 ? 32 : 64;  // 128 bytes of fp32 / bf16
#pragma unroll 1
          for (int c = 0; c < BN / cols; ++c) {
            uint32_t r[64];
            tmem_ld_32x32b_x32(tbase + uint32_t(c * cols), *reinterpret_cast<uint32_t(*)[32]>(r));
            if (pass == 1) tmem_ld_32x32b_x32(tbase + uint32_t(c * cols + 32), *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            tmem_ld_wait();
            if (p.epi_map >= 0) {
              epi32(p, r);
              if (pass == 1) epi32(p, r + 32);
            }
            uint8_t* tile = stage_out + (wq * 2 + (stage_ctr & 1)) * 4096;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* rowp = tile + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint4 v;
              if (pass == 0) {
                v = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
              } else {
                __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(r[8 * j]), __uint_as_float(r[8 * j + 1]));
                __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3]));
                __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5]));
                __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7]));
                v.x = *reinterpret_cast<uint32_t*>(&h0);
                v.y = *reinterpret_cast<uint32_t*>(&h1);
                v.z = *reinterpret_cast<uint32_t*>(&h2);
                v.w = *reinterpret_cast<uint32_t*>(&h3);
              }
              *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4)) = v;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              // outputs stream out: keep L2 for the operand tiles other CTAs re-read
              tma_store_3d_hint(p.maps + cm, tile, tc.n0 + c * cols, trow, tc.b, policy_evict_first());
              bulk_commit();
            }
            ++stage_ctr;
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + uint32_t(c * 32), r);
          tmem_ld_wait();
          if (p.epi_map >= 0) epi32(p, r);
          const int col = tc.n0 + c * 32;
          if (row >= p.M || col >= p.N) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {  // constant indices keep r[] in registers
            if (col + j >= p.N) break;
            if (c32) c32[col + j] = __uint_as_float(r[j]);
            if (c16) c16[col + j] = __float2bfloat16_rn(__uint_as_float(r[j]));
          }
        }
      }
      // this warp is done reading accumulator `as` (tell the leader's MMA issuer)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kCta == 2) mbar_arrive_cluster(empty_leader + uint32_t(as * sizeof(uint64_t)));
        else mbar_arrive(&acc_empty[as]);
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  if (kClu > 1) cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kAccStages * BN, kCta>(tmem);
  }
}

// ---- fp32x3 with promoted accumulation --------------------------------------
// The tensor core adds each MMA's result into its fp32 accumulator with
// truncation, so over a long K loop a 3xTF32 product loses ~K/8 half-ulps of
// the running sum (measured: 256 x K x 256, U[-1,1): mean error / sum|x||y|
// 1.4e-7 at K = 32, 9.7e-7 at K = 16384; sequential fp32 rounding-to-nearest,
// the reference's f32 mode, stays at 1.7e-8). Here the MMAs accumulate only
// `chunk` K blocks (default 4) at a time into one of two TMEM buffers, and eight epilogue
// warps add each finished chunk into a running sum held in registers with
// IEEE fp32 adds (round to nearest) — the promotion DeepSeek-V3 uses for FP8,
// applied to TF32. The chunk drains overlap the next chunk's MMAs (two
// buffers), so the tensor pipe never waits for them.
// Warps: 0-7 epilogue (warp w: TMEM lane quarter w % 4, column half w / 4),
// 8 TMA producer, 9 TMEM allocator + MMA issuer, 10-11 idle. Warps are dealt
// to the SM's four 16K-register sub-partitions round-robin, so twelve warps
// (three per sub-partition) leave 168 registers per thread — room for each
// epilogue thread's BN / 2 running sums (ten warps would put three on some
// sub-partitions all the same).
constexpr int kX3Threads = 384;

// x - tf32(x): the part of an fp32 value a kind::tf32 MMA drops (its 13 low
// mantissa bits); the x3 kernel writes it as the "lo" shadow of its output
// when a later fp32x3 contraction reads that output (split_lo_kernel's value)
__device__ __forceinline__ float lo_of(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ float epi_f(int op, float c, float x) {
  if (op == 0) return x > 0.0f ? x : 0.0f;
  if (op == 2) return -x;
  if (op == 3) return c * x;
  return x;
}

// Work units of the x3 kernel: every tile, except that the last `split`
// tiles (the partial last wave) are each cut into two halves of their
// (sibling, K block) sequence, run by two clusters of that wave: half 0 leaves
// its fp32 running sums in a workspace, half 1 adds them to its own and stores.
struct X3Unit {
  int t, part;  // tile, -1 whole / 0 first half / 1 second half
};
__device__ __forceinline__ X3Unit x3_unit(const GemmLaunch& p, int u, int total) {
  const int whole = total - p.split;
  X3Unit r;
  r.t = u < whole ? u : whole + (u - whole) / 2;
  r.part = u < whole ? -1 : (u - whole) % 2;
  return r;
}
// the unit's range [q0, q1) of its tile's (sibling, K block) iterations
__device__ __forceinline__ void x3_range(const X3Unit& U, int iters, int& q0, int& q1) {
  q0 = U.part == 1 ? iters / 2 : 0;
  q1 = U.part == 0 ? iters / 2 : iters;
}

template <int kCta, int BN>
__global__ void __launch_bounds__(kX3Threads, 1) gemm_x3_kernel(const __grid_constant__ GemmLaunch p) {
  using C_ = Cfg<false, kCta, BN, true>;
  constexpr int STAGES = C_::STAGES;
  constexpr int HALF = BN / 2;  // running-sum columns per epilogue thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_out = smem + STAGES * C_::STAGE_BYTES;  // 8 warps x one 32 x 128 B staging tile
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stage_out + C_::STORE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* part_full = empty_bar + STAGES;  // chunk partial ready in TMEM buffer b
  uint64_t* part_empty = part_full + 2;      // chunk partial drained into the running sums
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(part_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = kCta == 2 ? cluster_ctarank() : 0;
  const int tiles_m = (p.M + C_::TILE_M - 1) / C_::TILE_M;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int total = tiles_m * tiles_n * p.batch * p.n_regions;
  const int units = total + p.split;
  const int kblocks = (p.K + C_::BK - 1) / C_::BK;
  const int first = blockIdx.x / kCta, stride = gridDim.x / kCta;
  const int chunk = p.chunk > 0 ? p.chunk : 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&part_full[b], 1);
      mbar_init(&part_empty[b], 8 * kCta);  // every epilogue warp of the pair
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<2 * BN, kCta>(tmem_slot);
  tc_fence_before();
  if (kCta == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();

  if (warp == 8) {
    // ---- TMA producer: A_hi | B_hi | A_lo | B_lo per stage ----
    if (lane == 0) {
      int it = 0, ti = 0;
      bool sync_on = p.sync != nullptr;
      for (int u = first; u < units; u += stride, ++ti) {
        if (u + stride >= units) griddep_launch();
        const X3Unit U = x3_unit(p, u, total);
        const TileCoord tc = tile_coord<C_::TILE_M, BN>(p, U.t, tiles_m, tiles_n);
        const GemmRegion reg = p.regions[tc.region];
        int q0, q1;
        x3_range(U, kblocks * reg.n_sib, q0, q1);
        const int am = tc.m0 + int(rank) * BM, bn = tc.n0 + int(rank) * C_::B_ROWS;
        const int bseg_i = reg.bseg ? tc.b / reg.bseg : 0;
        const int ba = reg.bseg && !reg.bseg_b ? tc.b % reg.bseg : tc.b;
        const int bb = reg.bseg && reg.bseg_b ? tc.b % reg.bseg : tc.b;
        // serpentine K: every other wave walks (sibling, K block) backwards, so it
        // starts on the panel slices the previous wave left in L2 (the grouped
        // raster keeps a wave's A panels for the next few waves)
        const bool back = p.serp && (ti & 1) && U.part < 0;
        for (int q = q0; q < q1; ++q, ++it) {
          const int si = q / kblocks, kq = q % kblocks;
          {
            const int sib = back ? reg.n_sib - 1 - si : si;
            const CUtensorMap* ma = p.maps + reg.map0 + C_::NMAP * (bseg_i * reg.n_sib + sib);
            const int kb = back ? kblocks - 1 - kq : kq;
            if (p.sync) producer_lockstep(p, it, sync_on);
            const int s = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            mbar_wait(&empty_bar[s], ph ^ 1);
            const int k0 = kb * C_::BK;
            uint8_t* sa = smem + s * C_::STAGE_BYTES;
            uint8_t* sb = sa + C_::A_BYTES;
            if (rank == 0) mbar_expect_tx(&full_bar[s], C_::STAGE_BYTES * kCta);
            auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1, int cb) {
              if (kCta == 2) tma_load_3d_2sm(dst, m, &full_bar[s], c0, c1, cb);
              else tma_load_3d(dst, m, &full_bar[s], c0, c1, cb);
            };
#pragma unroll
            for (int part = 0; part < 2; ++part) {
              uint8_t* pa = sa + part * C_::LO_OFF;
              uint8_t* pb = sb + part * C_::LO_OFF;
              const CUtensorMap* pma = ma + 2 * part;
              const CUtensorMap* pmb = ma + 1 + 2 * part;
              if (!p.a_mn) {
                load(pa, pma, k0, am, ba);
              } else {
#pragma unroll
                for (int i = 0; i < BM / C_::MN_ATOM; ++i) load(pa + i * C_::BK * 128, pma, am + i * C_::MN_ATOM, k0, ba);
              }
              if (!p.b_mn) {
                load(pb, pmb, k0, bn, bb);
              } else {
#pragma unroll
                for (int i = 0; i < C_::B_ROWS / C_::MN_ATOM; ++i)
                  load(pb + i * C_::BK * 128, pmb, bn + i * C_::MN_ATOM, k0, bb);
              }
            }
          }
        }
      }
      if (p.sync) producer_lockstep_exit(p, it);
    }
  } else if (warp == 9) {
    // ---- MMA issuer: chunks of `chunk` K blocks into alternating buffers ----
    if (rank == 0) {  // the whole warp runs the loop (uniform values), one elected lane issues
      const uint32_t idesc = umma_idesc(2u, BM * kCta, BN, p.a_mn, p.b_mn);
      const uint32_t a_lbo = p.a_mn ? C_::BK * 128 : 16, b_lbo = p.b_mn ? C_::BK * 128 : 16;
      const uint32_t a_step = p.a_mn ? C_::UMMA_K * 128 : 32, b_step = p.b_mn ? C_::UMMA_K * 128 : 32;
      const uint32_t a_lt = p.a_mn ? 1u : 2u, b_lt = p.b_mn ? 1u : 2u;
      const uint32_t a_sbo = a_lt == 1 ? 512u : 1024u, b_sbo = b_lt == 1 ? 512u : 1024u;
      int it = 0, nchunk = 0;
      for (int u = first; u < units; u += stride) {
        const X3Unit U = x3_unit(p, u, total);
        const TileCoord tc = tile_coord<C_::TILE_M, BN>(p, U.t, tiles_m, tiles_n);
        int q0, q1;
        x3_range(U, kblocks * p.regions[tc.region].n_sib, q0, q1);
        const int iters = q1 - q0;
        for (int i = 0; i < iters; ++nchunk) {
          const int b = nchunk & 1;
          const uint32_t bph = (nchunk >> 1) & 1;
          if (kCta == 2) mbar_wait_cluster(&part_empty[b], bph ^ 1);
          else mbar_wait(&part_empty[b], bph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem + uint32_t(b * BN);
          const int n = iters - i < chunk ? iters - i : chunk;
          for (int q = 0; q < n; ++q, ++i, ++it) {
            const int s = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * C_::STAGE_BYTES);
            const uint32_t sb = sa + C_::A_BYTES;
#pragma unroll
            for (int k = 0; k < 3 * (C_::BK / C_::UMMA_K); ++k) {
              const int prod = k / (C_::BK / C_::UMMA_K), kk = k % (C_::BK / C_::UMMA_K);
              const uint32_t oa = prod == 2 ? uint32_t(C_::LO_OFF) : 0u, ob = prod == 1 ? uint32_t(C_::LO_OFF) : 0u;
              const uint64_t ad = umma_desc_sw128(sa + oa + kk * a_step, a_lbo, a_sbo, a_lt);
              const uint64_t bd = umma_desc_sw128(sb + ob + kk * b_step, b_lbo, b_sbo, b_lt);
              const uint32_t acc = (q | k) != 0;  // each chunk starts a fresh partial
              if (kCta == 2) mma_tf32_2sm_warp(d_tmem, ad, bd, idesc, acc);
              else mma_tf32_warp(d_tmem, ad, bd, idesc, acc);
            }
            if (kCta == 2) mma_commit_2sm_warp(&empty_bar[s]);
            else mma_commit_warp(&empty_bar[s]);
          }
          if (kCta == 2) mma_commit_2sm_warp(&part_full[b]);
          else mma_commit_warp(&part_full[b]);
        }
      }
    }
  } else if (warp < 8) {
    // ---- epilogue: promote every chunk partial into fp32 running sums ----
    const int wq = warp & 3, hh = warp >> 2;
    const uint32_t empty_leader = kCta == 2 ? mapa(smem_u32(part_empty), 0) : 0;
    uint8_t* tile = stage_out + warp * 4096;
    int nchunk = 0;
    for (int u = first; u < units; u += stride) {
      const X3Unit U = x3_unit(p, u, total);
      const TileCoord tc = tile_coord<C_::TILE_M, BN>(p, U.t, tiles_m, tiles_n);
      const GemmRegion reg = p.regions[tc.region];
      int q0, q1;
      x3_range(U, kblocks * reg.n_sib, q0, q1);
      const int iters = q1 - q0;
      const int nch = (iters + chunk - 1) / chunk;
      float acc[HALF];
      for (int c = 0; c < nch; ++c, ++nchunk) {
        const int b = nchunk & 1;
        const uint32_t bph = (nchunk >> 1) & 1;
        mbar_wait(&part_full[b], bph);
        tc_fence_after();
        const uint32_t tb = tmem + (uint32_t(wq * 32) << 16) + uint32_t(b * BN + hh * HALF);
#pragma unroll
        for (int j = 0; j < HALF / 16; ++j) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tb + uint32_t(j * 16), r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            acc[j * 16 + e] = c == 0 ? __uint_as_float(r[e]) : __fadd_rn(acc[j * 16 + e], __uint_as_float(r[e]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kCta == 2) mbar_arrive_cluster(empty_leader + uint32_t(b * sizeof(uint64_t)));
          else mbar_arrive(&part_empty[b]);
        }
      }
      if (U.part >= 0) {
        // split tile: this thread's row segment of the running sums in the workspace
        const int si = U.t - (total - p.split);
        float* ws = p.split_ws + ((size_t(si) * kCta + rank) * BM + size_t(wq * 32 + lane)) * BN + hh * HALF;
        unsigned int* cnt = p.split_cnt + si;
        if (U.part == 0) {
#pragma unroll
          for (int e = 0; e < HALF; e += 4)
            __stcg(reinterpret_cast<float4*>(ws + e), make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]));
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(cnt, 1u);  // 8 * kCta warps: the first half is in place
          continue;
        }
        if (lane == 0) {
          unsigned int v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
          } while (v < 8u * kCta);
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < HALF; e += 4) {
          const float4 f = __ldcg(reinterpret_cast<const float4*>(ws + e));
          acc[e] = __fadd_rn(f.x, acc[e]);
          acc[e + 1] = __fadd_rn(f.y, acc[e + 1]);
          acc[e + 2] = __fadd_rn(f.z, acc[e + 2]);
          acc[e + 3] = __fadd_rn(f.w, acc[e + 3]);
        }
        __syncwarp();
        if (lane == 0 && atomicAdd(cnt, 1u) == 16u * kCta - 1u) atomicExch(cnt, 0u);  // last reader re-arms
      }
      if (p.epi_map >= 0) {
#pragma unroll
        for (int e = 0; e < HALF; ++e) acc[e] = epi_f(p.epi_map, p.epi_c, acc[e]);
      }
      const int row0 = tc.m0 + int(rank) * BM + wq * 32;
      const int col0 = tc.n0 + hh * HALF;
      if (reg.cmap32 >= 0 || reg.cmap16 >= 0) {
        // registers -> 128B-swizzled staging tile -> TMA store (clipped at the region bounds)
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int cm = pass == 0 ? reg.cmap32 : reg.cmap16;
          if (cm < 0) continue;
          constexpr int kSlices = HALF / 32;
#pragma unroll
          for (int sl = 0; sl < kSlices; ++sl) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            uint8_t* rowp = tile + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int e = sl * 32 + 4 * j;
              const uint4 v = pass == 0 ? make_uint4(__float_as_uint(acc[e]), __float_as_uint(acc[e + 1]),
                                                     __float_as_uint(acc[e + 2]), __float_as_uint(acc[e + 3]))
                                        : make_uint4(__float_as_uint(lo_of(acc[e])), __float_as_uint(lo_of(acc[e + 1])),
                                                     __float_as_uint(lo_of(acc[e + 2])), __float_as_uint(lo_of(acc[e + 3])));
              *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4)) = v;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d_hint(p.maps + cm, tile, col0 + sl * 32, row0, tc.b, policy_evict_first());
              bulk_commit();
            }
          }
        }
      } else {
        const int row = row0 + lane;
        const long long base = (long long)tc.b * p.c_sb + (long long)row * p.c_sm;
        float* c32 = reg.c32 ? reg.c32 + base : nullptr;
        float* clo = reg.c16 ? static_cast<float*>(reg.c16) + base : nullptr;
        if (row < p.M) {
#pragma unroll
          for (int e = 0; e < HALF; ++e) {
            if (col0 + e < p.N) {
              if (c32) c32[col0 + e] = acc[e];
              if (clo) clo[col0 + e] = lo_of(acc[e]);
            }
          }
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  if (kCta == 2) cluster_sync();
  else __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<2 * BN, kCta>(tmem);
  }
}

template <int kCta, int BN>
cudaError_t prepare_x3() {
  return cudaFuncSetAttribute(gemm_x3_kernel<kCta, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Cfg<false, kCta, BN, true>::SMEM);
}

template <int kCta, int BN>
cudaError_t launch_x3(const GemmLaunch& p, int num_sms, cudaStream_t stream) {
  using C_ = Cfg<false, kCta, BN, true>;
  const long long tiles =
      (long long)((p.M + C_::TILE_M - 1) / C_::TILE_M) * ((p.N + BN - 1) / BN) * p.batch * p.n_regions + p.split;
  const int clusters = int(tiles < num_sms / kCta ? tiles : num_sms / kCta);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * kCta);
  cfg.blockDim = dim3(kX3Threads);
  cfg.dynamicSmemBytes = C_::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemm_x3_kernel<kCta, BN>, p);
}

// co-resident clusters per kernel variant (clusters never span a GPC, so
// 4-CTA clusters may leave SMs idle): measured once by the occupancy API
template <bool kBF16, int kCta, int BN, bool kX3, int kMc>
int& max_clusters() {
  static int n = 0;
  return n;
}

template <bool kBF16, int kCta, int BN, bool kX3 = false, int kMc = 1>
cudaError_t prepare_t() {
  using C_ = Cfg<kBF16, kCta, BN, kX3>;
  auto kern = gemm_kernel<kBF16, kCta, BN, kX3, kMc>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
  if (e != cudaSuccess || kMc == 1) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCta * kMc);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C_::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCta * kMc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  max_clusters<kBF16, kCta, BN, kX3, kMc>() = n;
  return e;
}

template <bool kBF16, int kCta, int BN, bool kX3 = false, int kMc = 1>
cudaError_t launch_t(const GemmLaunch& p, int num_sms, cudaStream_t stream) {
  using C_ = Cfg<kBF16, kCta, BN, kX3>;
  constexpr int kClu = kCta * kMc;
  const long long tiles = (long long)((p.M + C_::TILE_M - 1) / C_::TILE_M) * ((p.N + BN * kMc - 1) / (BN * kMc)) *
                          p.batch * p.n_regions;
  int cap = num_sms / kClu;
  const int resident = max_clusters<kBF16, kCta, BN, kX3, kMc>();
  if (kMc > 1 && resident > 0 && resident < cap) cap = resident;
  const int clusters = int(tiles < cap ? tiles : cap);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * kClu);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C_::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClu;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemm_kernel<kBF16, kCta, BN, kX3, kMc>, p);
}

}  // namespace

int gemm_bk(bool bf16) { return bf16 ? 64 : 32; }
int gemm_bm() { return BM; }
bool gemm_paired(int M) { return M > BM; }
int gemm_b_box(int M, int bn) { return gemm_paired(M) ? bn / 2 : bn; }

bool gemm_use_mc(int M, int N, int bn) {
  // A multicast over two 2-SM pairs: 256-row tiles, 256-wide, and at least
  // two N tiles so the second pair has work of its own
  static const int env = [] {
    const char* e = std::getenv("ED_GEMM_MC");
    return e ? std::atoi(e) : 0;  // opt-in: measured slower (4-CTA clusters fit only 132 of 148 SMs)
  }();
  return env != 0 && gemm_paired(M) && bn == 256 && N > 256;
}
int gemm_a_box_rows(bool mc) { return mc ? BM / 2 : BM; }

int gemm_x3_split(const GemmLaunch& p, int num_sms) {
  if (!p.x3) return 0;
  if (const char* e = std::getenv("ED_GEMM_X3_SPLIT"))
    if (e[0] == '0') return 0;
  const int kcta = gemm_paired(p.M) ? 2 : 1;
  const long long tiles =
      (long long)((p.M + BM * kcta - 1) / (BM * kcta)) * ((p.N + p.bn - 1) / p.bn) * p.batch * p.n_regions;
  const long long clusters = num_sms / kcta;
  const long long rem = tiles % clusters;
  // at least one full wave before it, and both halves of every split tile in the last one
  if (tiles < clusters || rem == 0 || 2 * rem > clusters) return 0;
  return int(rem);
}

int gemm_sync_epochs(const GemmLaunch& p, int num_sms, int max_sib) {
  const int kcta = gemm_paired(p.M) ? 2 : 1;
  const int tile_m = BM * kcta;
  const long long tiles = (long long)((p.M + tile_m - 1) / tile_m) * ((p.N + p.bn - 1) / p.bn) * p.batch * p.n_regions;
  const long long clusters = tiles < num_sms / kcta ? tiles : num_sms / kcta;
  const long long per_cta = (tiles + clusters - 1) / clusters;
  const long long kblocks = (p.K + gemm_bk(p.bf16) - 1) / gemm_bk(p.bf16);
  return int((per_cta * kblocks * max_sib + p.sync_g - 1) / p.sync_g + 1);
}

int gemm_pick_bn(int M, int N, int batch, int n_regions, int num_sms) {
  // 128-wide tiles need 1.5x the L2->SMEM bytes per flop of 256-wide ones,
  // which a full grid cannot feed (measured on chain3: 0.094 -> 0.14 ms per
  // GEMM), so they are used only when a single partial wave of 256-wide
  // tiles would leave more than half of the SMs idle
  const int cta = gemm_paired(M) ? 2 : 1;
  const long long clusters = num_sms / cta;
  const long long tiles256 =
      (long long)((M + BM * cta - 1) / (BM * cta)) * ((N + 255) / 256) * batch * n_regions;
  return 2 * tiles256 <= clusters && N > 128 ? 128 : 256;
}

cudaError_t gemm_prepare() {
  cudaError_t e;
  if ((e = prepare_t<true, 1, 256>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 1, 256>()) != cudaSuccess) return e;
  if ((e = prepare_t<true, 2, 256>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 2, 256>()) != cudaSuccess) return e;
  if ((e = prepare_t<true, 1, 128>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 1, 128>()) != cudaSuccess) return e;
  if ((e = prepare_t<true, 2, 128>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 2, 128>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 1, 256, true>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 2, 256, true>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 1, 128, true>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 2, 128, true>()) != cudaSuccess) return e;
  if ((e = prepare_x3<1, 256>()) != cudaSuccess) return e;
  if ((e = prepare_x3<2, 256>()) != cudaSuccess) return e;
  if ((e = prepare_x3<1, 128>()) != cudaSuccess) return e;
  if ((e = prepare_x3<2, 128>()) != cudaSuccess) return e;
  if ((e = prepare_t<true, 2, 256, false, 2>()) != cudaSuccess) return e;
  if ((e = prepare_t<false, 2, 256, false, 2>()) != cudaSuccess) return e;
  return prepare_t<false, 2, 256, true, 2>();
}

cudaError_t launch_gemm(const GemmLaunch& p, int num_sms, cudaStream_t stream) {
  // pair SMs when the output has rows for both halves of a 256-row tile
  const bool pair = gemm_paired(p.M);
  const bool narrow = p.bn == 128;
  if (p.x3 && p.chunk > 0) {  // fp32x3 with promoted (round-to-nearest) accumulation
    if (narrow) return pair ? launch_x3<2, 128>(p, num_sms, stream) : launch_x3<1, 128>(p, num_sms, stream);
    return pair ? launch_x3<2, 256>(p, num_sms, stream) : launch_x3<1, 256>(p, num_sms, stream);
  }
  if (p.mc && pair && !narrow) {  // 4-CTA clusters sharing A (gemm_use_mc)
    if (p.bf16) return launch_t<true, 2, 256, false, 2>(p, num_sms, stream);
    if (p.x3) return launch_t<false, 2, 256, true, 2>(p, num_sms, stream);
    return launch_t<false, 2, 256, false, 2>(p, num_sms, stream);
  }
  if (p.bf16) {
    if (narrow) return pair ? launch_t<true, 2, 128>(p, num_sms, stream) : launch_t<true, 1, 128>(p, num_sms, stream);
    return pair ? launch_t<true, 2, 256>(p, num_sms, stream) : launch_t<true, 1, 256>(p, num_sms, stream);
  }
  if (p.x3) {
    if (narrow)
      return pair ? launch_t<false, 2, 128, true>(p, num_sms, stream) : launch_t<false, 1, 128, true>(p, num_sms, stream);
    return pair ? launch_t<false, 2, 256, true>(p, num_sms, stream) : launch_t<false, 1, 256, true>(p, num_sms, stream);
  }
  if (narrow) return pair ? launch_t<false, 2, 128>(p, num_sms, stream) : launch_t<false, 1, 128>(p, num_sms, stream);
  return pair ? launch_t<false, 2, 256>(p, num_sms, stream) : launch_t<false, 1, 256>(p, num_sms, stream);
}

}  // namespace ed
