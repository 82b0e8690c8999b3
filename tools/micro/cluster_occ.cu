// How many clusters of 2 / 4 / 8 CTAs with ~225 KiB of shared memory each can
// be resident at once on this GPU (cudaOccupancyMaxActiveClusters), vs
// num_SMs / cluster size: clusters must fit inside one GPC, so SMs left over
// in a GPC stay idle for larger clusters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    for (int smem : {100 * 1024, 230656}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(pr.multiProcessorCount / cs * cs);
      cfg.blockDim = dim3(192);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
      std::printf("SMs %d, cluster %d, smem %d: max active clusters %d = %d SMs (%s)\n", pr.multiProcessorCount, cs,
                  smem, n, n * cs, cudaGetErrorString(e));
    }
  }
  return 0;
}
