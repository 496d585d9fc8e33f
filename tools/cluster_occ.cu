// How many clusters of a given shape can be co-resident (cudaOccupancyMaxActiveClusters)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k256(float* p) { extern __shared__ float s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); if (p) p[threadIdx.x] = s[255 - threadIdx.x]; }
__global__ void __launch_bounds__(512, 1) k512(float* p) { extern __shared__ float s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); if (p) p[threadIdx.x] = s[511 - threadIdx.x]; }
template <typename K>
void q(K kern, int nt, int smem, int C) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  printf("threads %4d smem %6d KB cluster %2d -> max active clusters %3d (%d CTAs) %s\n", nt, smem / 1024, C, n, n * C, cudaGetErrorString(e));
}
int main() {
  for (int C : {2, 4, 8, 16}) {
    q(k256, 256, 96 * 1024, C);
    q(k256, 256, 64 * 1024, C);
    q(k256, 256, 48 * 1024, C);
    q(k512, 512, 192 * 1024, C);
    q(k512, 512, 96 * 1024, C);
  }
}
