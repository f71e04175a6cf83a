#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* x) { extern __shared__ int s[]; if (threadIdx.x == 0 && x) x[blockIdx.x] = s[0]; }
int main() {
  for (int smem : {100 * 1024, 150 * 1024, 200 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(1, 1, 16 * cs); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 1; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = cs;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %d KB cluster %2d: max active clusters %d (%s) -> %d CTAs\n", smem / 1024, cs, n, cudaGetErrorString(e), n * cs);
    }
  }
}
