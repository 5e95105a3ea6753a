// Max co-resident clusters per cluster size for a 1-CTA/SM kernel (development tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_clusters.bin tools/probe_clusters.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; s[threadIdx.x] = 0; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C = 1; C <= 16; ++C) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(C * 64);
    c.blockDim = dim3(544);
    c.dynamicSmemBytes = smem;
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = C; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
    c.attrs = &a; c.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &c);
    printf("C=%2d clusters=%3d SMs=%3d %s\n", C, n, n * C, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
