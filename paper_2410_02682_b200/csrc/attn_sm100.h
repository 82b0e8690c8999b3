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
};

struct AttnRegion {
  int q;            // Q [s,h,d] (K-major, box {64, 128})
  AttnSrc k, v;     // K [s2,h,d] (K-major), V [s2,h,d] (MN-major), boxes {64, 128}
  int o32, o16;     // O [s,h,d] store maps (box {32|64, 32}), -1 if that dtype is not needed
};

struct AttnLaunch {
  const CUtensorMap* maps;     // device array
  const AttnRegion* regions;   // device array
  int n_regions;
  int H, S, T, D;              // heads, query rows, keys, head dim (per region)
  float scale;                 // scale of the fused T2 vertex (1 if none)
  int n_pair_jobs, n_jobs;     // set by attn_schedule (launch_attn calls it)
};

// Split the (region, head, 128-row tile) space into tile-pair jobs and, for
// the last wave, single-tile jobs, so that every CTA of the persistent grid
// finishes at about the same time.
void attn_schedule(AttnLaunch& p, int num_sms);

bool attn_supported(int S, int T, int D);
cudaError_t attn_prepare();
cudaError_t launch_attn(const AttnLaunch& p, int num_sms, cudaStream_t s);

}  // namespace ed
