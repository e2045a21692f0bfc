// Dev: how many 2-CTA clusters of a big-smem kernel fit on this GPU at once.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0]; }
int main() {
  for (int smem : {60 * 1024, 120 * 1024, 200 * 1024}) for (int threads : {256, 512}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = 2; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at; cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("smem %d KB threads %d: max active 2-CTA clusters %d (%s)\n", smem / 1024, threads, n, cudaGetErrorString(e));
  }
}
