// max active clusters for a 512-thread, ~210 KB-smem kernel at cluster sizes 2..16 (tuning aid)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* o) { extern __shared__ float s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); if (o) o[blockIdx.x] = s[5]; }
int main() {
  for (size_t smem : {100 * 1024, 150 * 1024, 210 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * 32); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %zu KB cluster %2d: max active clusters %d (= %d CTAs) %s\n", smem / 1024, cs, n, n * cs, cudaGetErrorString(e));
    }
  }
  return 0;
}
