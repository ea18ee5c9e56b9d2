// Diagnostics: how many clusters of size 4 / 8 / 16 fit on the device at
// once for a 256-thread CTA with the given dynamic shared memory.
#include <cstdio>
__global__ void __launch_bounds__(256, 1) k(int* p) { if (p) p[0] = 1; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {70 * 1024, 133 * 1024, 200 * 1024})
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * 32);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %3d KB cluster %2d: %d clusters (%d CTAs) %s\n", smem / 1024, cs, n, n * cs,
             cudaGetErrorString(e));
    }
  return 0;
}
