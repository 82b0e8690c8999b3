// Block contraction of a mul/sum join on the 5th-gen tensor cores.
//
// Replaces kernel_eval's mul/sum case (kernel.cc:48-65) for one output
// region: C = sum_s A_s * B_s over the aggregation siblings s of the region
// (the join tuples folded by the region's refinement, runtime.cc:242-261),
// concatenated along K so the fold happens in the TMEM accumulator.
//
// Label permutations are folded into 3-D TMA tensor maps (inner dim, outer
// dim, batch) — K-major or MN-major per operand — so no transpose copy ever
// runs. Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + single-
// thread tcgen05.mma issuer, warps 2-5 epilogue (TMEM -> registers -> HBM),
// STAGES-deep smem ring with full/empty mbarriers.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm_sm100.h"
#include "ptx.cuh"

namespace ed {

namespace {

constexpr int BM = 128;
constexpr int STAGES = 4;
constexpr int kThreads = 192;

template <bool kBF16, int BN>
struct Cfg {
  static constexpr int ES = kBF16 ? 2 : 4;          // element bytes
  static constexpr int BK = 128 / ES;               // one 128-byte swizzle row of K
  static constexpr int UMMA_K = kBF16 ? 16 : 8;     // 32 bytes of K per MMA
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int MN_ATOM = 128 / ES;          // MN elements per 128-byte atom
};

template <bool kBF16, int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmParams p) {
  using C_ = Cfg<kBF16, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C_::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tmem_full = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * BM;
  const int bz = blockIdx.z;
  const int kblocks = (p.K + C_::BK - 1) / C_::BK;
  const int iters = kblocks * p.n_sib;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.n_sib; ++s) {
      tma_prefetch(&p.a[s]);
      tma_prefetch(&p.b[s]);
    }
  }
  if (warp == 1) tmem_alloc<BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      for (int it = 0; it < iters; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty_bar[s], ph ^ 1);
        const int sib = it / kblocks;
        const int k0 = (it % kblocks) * C_::BK;
        uint8_t* sa = smem + s * C_::STAGE_BYTES;
        uint8_t* sb = sa + C_::A_BYTES;
        mbar_expect_tx(&full_bar[s], C_::STAGE_BYTES);
        if (!p.a_mn) {
          tma_load_3d(sa, &p.a[sib], &full_bar[s], k0, m0, bz);
        } else {
          for (int i = 0; i < BM / C_::MN_ATOM; ++i)
            tma_load_3d(sa + i * C_::BK * 128, &p.a[sib], &full_bar[s], m0 + i * C_::MN_ATOM, k0, bz);
        }
        if (!p.b_mn) {
          tma_load_3d(sb, &p.b[sib], &full_bar[s], k0, n0, bz);
        } else {
          for (int i = 0; i < BN / C_::MN_ATOM; ++i)
            tma_load_3d(sb + i * C_::BK * 128, &p.b[sib], &full_bar[s], n0 + i * C_::MN_ATOM, k0, bz);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (one thread) ----
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(kBF16 ? 1u : 2u, BM, BN, p.a_mn, p.b_mn);
      // K-major: 8-row x 128-byte swizzle atoms stacked along MN (SBO 1024),
      // K advances 32 bytes per MMA inside the atom.
      // MN-major: 128-byte MN atoms of BK K-rows (LBO = BK*128), 8-row K
      // groups (SBO 1024), K advances UMMA_K rows per MMA.
      const uint32_t a_lbo = p.a_mn ? C_::BK * 128 : 16, b_lbo = p.b_mn ? C_::BK * 128 : 16;
      const uint32_t a_step = p.a_mn ? C_::UMMA_K * 128 : 32, b_step = p.b_mn ? C_::UMMA_K * 128 : 32;
      for (int it = 0; it < iters; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * C_::STAGE_BYTES);
        const uint32_t sb = sa + C_::A_BYTES;
#pragma unroll
        for (int k = 0; k < C_::BK / C_::UMMA_K; ++k) {
          const uint64_t ad = umma_desc_sw128(sa + k * a_step, a_lbo, 1024);
          const uint64_t bd = umma_desc_sw128(sb + k * b_step, b_lbo, 1024);
          if (kBF16) mma_f16(tmem, ad, bd, idesc, (it | k) != 0);
          else mma_tf32(tmem, ad, bd, idesc, (it | k) != 0);
        }
        mma_commit(&empty_bar[s]);
      }
      mma_commit(tmem_full);
    }
  } else {
    // ---- epilogue: TMEM -> registers -> HBM ----
    const int wq = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + wq * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    float* c32 = p.c32 ? p.c32 + (long long)bz * p.c_sb + (long long)row * p.c_sm : nullptr;
    __nv_bfloat16* c16 = p.c16 ? static_cast<__nv_bfloat16*>(p.c16) + (long long)bz * p.c_sb + (long long)row * p.c_sm : nullptr;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (uint32_t(wq * 32) << 16) + uint32_t(c * 32), r);
      tmem_ld_wait();
      const int col = n0 + c * 32;
      if (row >= p.M || col >= p.N) continue;
      const bool full = col + 32 <= p.N && p.vec_ok;
      if (c32) {
        if (full) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(c32 + col + j) =
                make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                            __uint_as_float(r[j + 3]));
        } else {
          for (int j = 0; j < 32 && col + j < p.N; ++j) c32[col + j] = __uint_as_float(r[j]);
        }
      }
      if (c16) {
        if (full) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            __nv_bfloat162 h[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              h[q] = __floats2bfloat162_rn(__uint_as_float(r[j + 2 * q]), __uint_as_float(r[j + 2 * q + 1]));
            *reinterpret_cast<uint4*>(c16 + col + j) = *reinterpret_cast<uint4*>(h);
          }
        } else {
          for (int j = 0; j < 32 && col + j < p.N; ++j) c16[col + j] = __float2bfloat16_rn(__uint_as_float(r[j]));
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<BN>(tmem);
  }
}

template <bool kBF16, int BN>
cudaError_t prepare_t() {
  return cudaFuncSetAttribute(gemm_kernel<kBF16, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Cfg<kBF16, BN>::SMEM);
}

template <bool kBF16, int BN>
cudaError_t launch_t(const GemmParams& p, cudaStream_t stream) {
  using C_ = Cfg<kBF16, BN>;
  auto k = gemm_kernel<kBF16, BN>;
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.batch);
  k<<<grid, kThreads, C_::SMEM, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

int gemm_bn(bool bf16) { (void)bf16; return 256; }
int gemm_bk(bool bf16) { return bf16 ? 64 : 32; }

cudaError_t gemm_prepare() {
  cudaError_t e = prepare_t<true, 256>();
  return e != cudaSuccess ? e : prepare_t<false, 256>();
}

cudaError_t launch_gemm(const GemmParams& p, bool bf16, cudaStream_t stream) {
  return bf16 ? launch_t<true, 256>(p, stream) : launch_t<false, 256>(p, stream);
}

}  // namespace ed
