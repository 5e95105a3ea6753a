// Probe: shared-window addressing inside 2-CTA clusters (dynamic smem symbol, constant-address
// LDS/STS, mapa + ld.shared::cluster).  Dev tool: tools/probe_cluster_smem.bin <test>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
extern "C" __shared__ __align__(16) unsigned char probe_dyn[];
__global__ void k(unsigned* out, int test) {
  asm volatile("" ::"l"(probe_dyn));
  unsigned b, r;
  asm("mov.u32 %0, probe_dyn;" : "=r"(b));
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  unsigned v = 0, w = 0;
  if (test >= 1) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(0x400u + 4 * threadIdx.x), "r"(100 + blockIdx.x) : "memory");
    __syncthreads();
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(0x400u + 4 * threadIdx.x) : "memory");
  }
  if (test >= 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned rem;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem) : "r"(0x400u + 4 * threadIdx.x), "r"(r ^ 1));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(w) : "r"(rem) : "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) { out[blockIdx.x * 4] = b; out[blockIdx.x * 4 + 1] = r; out[blockIdx.x * 4 + 2] = v; out[blockIdx.x * 4 + 3] = w; }
}
int main(int argc, char** argv) {
  unsigned* d; cudaMalloc(&d, 64 * 4); unsigned h[64];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  for (int test = 0; test <= 2; ++test)
  for (int cl = 1; cl <= 2; ++cl) {
    if (test == 2 && cl == 1) continue;
    cudaMemset(d, 0, 256);
    cudaLaunchConfig_t c = {}; c.gridDim = 4; c.blockDim = 32; c.dynamicSmemBytes = 80000;
    cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension; a.val.clusterDim.x = cl; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
    c.attrs = &a; c.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&c, k, d, test);
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("test %d cluster %d: launch=%d sync=%s |", test, cl, (int)e, cudaGetErrorString(e2));
    for (int i = 0; i < 4; ++i) printf(" [b=%x r=%u v=%u w=%u]", h[4*i], h[4*i+1], h[4*i+2], h[4*i+3]);
    printf("\n");
    if (e2 != cudaSuccess) return 1;
  }
}
