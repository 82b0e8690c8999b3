// Fused attention kernel interface (see attn_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace ed {

// One output region: indices into AttnLaunch::maps.
// K and V may be read in place from a regular grid of producer regions
// (keys x head-dim) instead of a pasted chunk: map index for a 128-key block
// j and 64-wide d slice c is base + (j*128 / keys) * nd + (c*64) / dw, at
// coordinates {(c*64) % dw, (j*128) % keys, h + hoff}.
struct AttnSrc {
  int base, nd, keys, dw, hoff;
  int lo;           // fp32x3: maps[i + lo] is the lo-shadow twin of maps[i]
};

struct AttnRegion {
  int q;            // Q [s,h,d] (K-major, box {64, 128})
  AttnSrc k, v;     // K [s2,h,d] (K-major), V [s2,h,d] (MN-major), boxes {64, 128}
  int o32, o16;     // O [s,h,d] store maps (box {32|64, 32}), -1 if that dtype is not needed
  // fp32x3 kernel (attn_x3_sm100.cu): q maps Q's lo shadow, q + 1 Q itself
  // (box {32, 128} each); q_tm (Q) and O (+ its lo shadow) are plain pointers,
  // [s,h,d] with d contiguous; strides in elements
  const float* q_tm;
  long long q_rs, q_hs;
  float* o;
  float* o_lo;      // nullable
  long long o_rs, o_hs;
};

struct AttnLaunch {
  const CUtensorMap* maps;     // device array
  const AttnRegion* regions;   // device array
  int n_regions;
  int H, S, T, D;              // heads, query rows, keys, head dim (per region)
  float scale;                 // scale of the fused T2 vertex (1 if none)
  int x3;                      // 1: fp32x3 kernel (launch_attn_x3)
  int n_pair_jobs, n_jobs;     // set by attn_schedule (launch_attn calls it)
};

// Split the (region, head, 128-row tile) space into tile-pair jobs and, for
// the last wave, single-tile jobs, so that every CTA of the persistent grid
// finishes at about the same time.
void attn_schedule(AttnLaunch& p, int num_sms);

bool attn_supported(int S, int T, int D);
cudaError_t attn_prepare();
cudaError_t launch_attn(const AttnLaunch& p, int num_sms, cudaStream_t s);

// fp32x3 variant (attn_x3_sm100.cu): fp32 operands with lo shadows, both
// contractions as three TF32 products, P in fp32. Maps: Q box {32, 128},
// K box {32, 64} (K-major), V box {32, 32} (MN-major, 32-byte-atom swizzle).
bool attn_x3_supported(int S, int T, int D);
// CTAs per cluster of the fp32x3 kernel for S query rows (2: cta_group::2 pairs,
// K maps then box {32, 32}; ED_ATTN_X3_CTA=1 forces single CTAs)
int attn_x3_cta(int S);
cudaError_t attn_x3_prepare();
cudaError_t launch_attn_x3(const AttnLaunch& p, int num_sms, cudaStream_t s);

}  // namespace ed
