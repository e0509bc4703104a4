#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* o) { extern __shared__ int s[]; s[threadIdx.x] = threadIdx.x; if (threadIdx.x == 0) o[blockIdx.x] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smemkb : {100, 150, 200, 220}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smemkb * 1024);
    for (int cs : {2, 4, 8, 9, 12, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * 16); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smemkb * 1024;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
      printf("smem %3d KB cluster %2d: max active clusters %d (%s) -> CTAs %d\n", smemkb, cs, n, cudaGetErrorString(e), n * cs);
    }
  }
  return 0;
}
