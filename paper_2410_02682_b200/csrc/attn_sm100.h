// Fused attention kernel interface (see attn_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace ed {

// One output region: indices into AttnLaunch::maps.
struct AttnRegion {
  int q, k, v;      // Q [s,h,d], K [s2,h,d] (K-major, box {64, 128}); V [s2,h,d] (MN-major, box {64, 128})
  int o32, o16;     // O [s,h,d] store maps (box {32|64, 32}), -1 if that dtype is not needed
};

struct AttnLaunch {
  const CUtensorMap* maps;     // device array
  const AttnRegion* regions;   // device array
  int n_regions;
  int H, S, T, D;              // heads, query rows, keys, head dim (per region)
  float scale;                 // scale of the fused T2 vertex (1 if none)
};

bool attn_supported(int S, int T, int D);
cudaError_t attn_prepare();
cudaError_t launch_attn(const AttnLaunch& p, int num_sms, cudaStream_t s);

}  // namespace ed
