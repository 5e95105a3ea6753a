// tma_lat.cu -- latency of one 1-D bulk copy (cp.async.bulk) global -> shared vs size, from L2
// and from DRAM, measured with clock64 in one CTA or in every SM at once (dev tool).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_lat.cu -o tools/tma_lat.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
extern __shared__ __align__(128) unsigned char dsm[];
__global__ void k(const uint8_t* src, int bytes, int chunks, long long* out, int stride_ctas) {
  const uint32_t buf = (uint32_t)__cvta_generic_to_shared(dsm), bar = buf + 200 * 1024;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint8_t* s = src + (size_t)blockIdx.x * stride_ctas;
    long long t0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * chunks) : "memory");
    for (int c = 0; c < chunks; ++c)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(buf + c * bytes), "l"(s + (size_t)c * bytes), "r"(bytes), "r"(bar) : "memory");
    uint32_t done = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(bar) : "memory");
    } while (!done);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
}
__global__ void touch(const uint8_t* p, size_t n, unsigned* o) {
  unsigned a = 0;
  for (size_t i = (blockIdx.x * blockDim.x + threadIdx.x) * 16; i < n; i += (size_t)gridDim.x * blockDim.x * 16) a ^= *(const unsigned*)(p + i);
  if (a == 0x1234567) o[0] = a;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t pool = (size_t)1 << 30;
  uint8_t* b; CK(cudaMalloc(&b, pool)); CK(cudaMemset(b, 1, pool));
  long long* o; CK(cudaMalloc(&o, 8 * 1024)); unsigned* so; CK(cudaMalloc(&so, 64));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  std::vector<long long> h(1024);
  size_t off = 0;
  for (int ctas : {1, 148}) for (int l2 : {0, 1}) for (int bytes : {512, 4096, 16384, 24576, 65536}) for (int chunks : {1, 4}) {
    if (bytes * chunks > 196608) continue;
    const size_t span = (size_t)ctas * 262144;
    if (off + span > pool) off = 0;
    const uint8_t* src = b + off;
    if (l2) { touch<<<148, 256>>>(src, span, so); }
    else off += span;
    CK(cudaDeviceSynchronize());
    k<<<ctas, 32, 201 * 1024>>>(src, bytes / chunks, chunks, o, 262144);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), o, 8 * ctas, cudaMemcpyDeviceToHost));
    std::sort(h.begin(), h.begin() + ctas);
    printf("ctas=%3d %s bytes=%6d in %d copies: cycles min %lld med %lld max %lld\n", ctas, l2 ? "L2  " : "DRAM", bytes, chunks,
           h[0], h[ctas / 2], h[ctas - 1]);
  }
  return 0;
}
