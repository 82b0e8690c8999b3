// How many 2-CTA clusters with ~225 KiB of shared memory each can be resident
// at once on this GPU (cudaOccupancyMaxActiveClusters), vs num_SMs / 2.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) k2(int* p) { if (p) p[0] = 1; }
__global__ void k1(int* p) { if (p) p[0] = 1; }
int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  for (int smem : {100 * 1024, 200 * 1024, 230656}) {
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pr.multiProcessorCount);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k2, &cfg);
    std::printf("SMs %d, smem %d: max active 2-CTA clusters %d (%s)\n", pr.multiProcessorCount, smem, n, cudaGetErrorString(e));
  }
  return 0;
}
