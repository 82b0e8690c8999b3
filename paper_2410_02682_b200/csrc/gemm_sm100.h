// tcgen05 block-contraction kernel interface (see gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace ed {

constexpr int kMaxSib = 8;  // aggregation siblings folded in one accumulator

// One output region of an einsum: the sum over its aggregation siblings s of
// A_s * B_s (K-concatenated), written to c32 and/or its shadow c16: bf16 in
// the bf16 / tf32 kernels, fp32 x - tf32(x) (the "lo" operand copy a later
// fp32x3 contraction reads) in the x3 kernel.
struct GemmRegion {
  int n_sib;
  int map0;        // maps[map0 + 2*s] = A_s, maps[map0 + 2*s + 1] = B_s; with x3
                   // four per sibling: A_s, B_s, A_s lo, B_s lo
  int cmap32;      // output tensor map for TMA stores (-1: direct stores)
  int cmap16;
  float* c32;
  void* c16;
  // batch-segmented operand (bseg > 0): the operand (A if bseg_b == 0, else
  // B) of batch b is read in place from segment b / bseg at batch coordinate
  // b % bseg; segment s has its own sibling maps at map0 + NMAP * n_sib * s
  int bseg, bseg_b;
};

// One launch: every region of one einsum on this rank (same chunk shapes).
struct GemmLaunch {
  const CUtensorMap* maps;    // device array, 64-byte aligned
  const GemmRegion* regions;  // device array
  int n_regions;
  int M, N, K, batch;
  int a_mn, b_mn;             // 1: operand is MN-major (M or N contiguous)
  int vec_ok;                 // 1: output rows 16-byte aligned (vector stores)
  long long c_sm, c_sb;       // output element strides for M and batch; N stride is 1
  int bf16;                   // operand type: 1 bf16 (kind::f16), 0 fp32 (kind::tf32)
  int epi_map;                // fused map on the accumulator (ed_map_op) or -1
  float epi_c;                // scale constant of a fused scale map
  int bn;                     // tile width: 256 or 128 (gemm_pick_bn)
  int mc;                     // 1: 4-CTA clusters, two 2-SM pairs sharing (multicasting) the A panel
  int group_m;
  int region_inner;           // 1: tiles ordered batch-major across regions (regions share their B operand)
  int chunk;                  // x3: K blocks per TMEM partial promoted into fp32 running sums (0: off)
  // loose lockstep of the producers (experiment, x3 kernel): a CTA issues the
  // loads of epoch e (sync_g K blocks) only once every CTA has issued epoch
  // e - sync_lag, bounding how far the grid's CTAs drift apart along K so
  // the operand panels a wave shares are still in L2. sync: sync_epochs + 1
  // zeroed counters (the kernel re-zeroes them on exit); nullptr: off.
  unsigned int* sync;
  int sync_g, sync_lag, sync_epochs;                // grouped raster: tile rows that advance together along N
  int serp;                   // odd tile iterations walk (sibling, K block) backwards (L2 reuse across waves)
  // x3 kernel: the last `split` tiles (a partial last wave of at most half the
  // clusters) run as two half-K units each; split_ws holds the first halves'
  // running sums (split * TILE_M * BN floats), split_cnt one zeroed counter per tile
  int split;
  float* split_ws;
  unsigned int* split_cnt;
  int x3;                     // fp32-accurate 3xTF32: each stage carries hi and lo operand copies
                              // and feeds hi*hi + hi*lo + lo*hi into one accumulator
};

int gemm_bk(bool bf16);
int gemm_bm();
bool gemm_paired(int M);          // 2-SM (cta_group::2) tiles for this M
int gemm_b_box(int M, int bn);    // B rows (N) one CTA loads per K-major TMA box
// tile width: 128 when 256-wide tiles would leave over half the grid idle, else 256
int gemm_pick_bn(int M, int N, int batch, int n_regions, int num_sms);
bool gemm_use_mc(int M, int N, int bn);  // A multicast across two 2-SM pairs for this launch
int gemm_a_box_rows(bool mc);            // A rows per K-major TMA box (half a pair's rows with multicast)
constexpr int kStoreRows = 32;   // epilogue TMA-store box: 32 rows x 128 bytes
cudaError_t gemm_prepare();  // sets the dynamic-smem attribute (call before capture)
cudaError_t launch_gemm(const GemmLaunch& p, int num_sms, cudaStream_t stream);
// epochs of sync_g K blocks the busiest CTA of this launch issues (x3 kernel)
int gemm_sync_epochs(const GemmLaunch& p, int num_sms, int max_sib);
// x3 kernel: tiles of the partial last wave to split in two along K (0: none)
int gemm_x3_split(const GemmLaunch& p, int num_sms);

}  // namespace ed
