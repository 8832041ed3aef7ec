// Can B200 co-schedule clusters of up to 16 CTAs of ~209 KB shared memory each?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) { if (threadIdx.x == 0) out[blockIdx.x] = 1; }
int main() {
  int* out; cudaMalloc(&out, 4096 * 4);
  int smem = 6 * 32768 + 30 * 528 + 1024;  // cluster kernel: 6 stages + 30 push-slot rows + align
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("nonportable attr: %s\n", cudaGetErrorString(e));
  for (int cs = 2; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim = {(unsigned)cs, 1, 1};
    cfg.attrs = &at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t q = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    cudaError_t l = cudaLaunchKernelEx(&cfg, k, out);
    cudaError_t s = cudaDeviceSynchronize();
    printf("cluster %2d: max active clusters %3d (%s), launch of 8 clusters: %s / %s\n", cs, n, cudaGetErrorString(q), cudaGetErrorString(l), cudaGetErrorString(s));
  }
  return 0;
}
