// How many thread-block clusters of a given size fit on this GPU at once
// (cudaOccupancyMaxActiveClusters) for the ALS kernels' footprint (1 CTA/SM).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* p) { extern __shared__ double s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int smems[] = {48 * 1024, 100 * 1024, 160 * 1024, 200 * 1024, 227 * 1024};
  for (int sm : smems) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int cs : {1, 2, 4, 8, 12, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 8); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %6d cluster %2d -> max active clusters %3d (%d CTAs) %s\n", sm, cs, n, n * cs,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
