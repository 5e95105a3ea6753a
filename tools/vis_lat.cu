// vis_lat.cu -- cross-SM visibility latency of a relaxed.gpu store (writer CTA stores a
// stamped 64-bit word, reader CTA polls it with ld.relaxed.gpu), idle and while the other SMs
// stream HBM through bulk copies (dev tool).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/vis_lat.cu -o tools/vis_lat.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
extern __shared__ __align__(128) unsigned char dsm[];
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
// block 0: writer (after a delay, stores gt() into w[i] for i < n, spaced); block 1: reader
// blocks >= 2: streamers (bulk copies of their chunk, ring of 4 x 32 KB), if load != 0
__global__ void k(unsigned long long* w, unsigned long long* seen, int n, const uint8_t* src, long long per, int load) {
  if (blockIdx.x == 0) {
    if (threadIdx.x != 0) return;
    unsigned long long t = gt();
    while (gt() - t < 20000) {}
    for (int i = 0; i < n; ++i) {
      unsigned long long now = gt();
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(w + i), "l"(now) : "memory");
      while (gt() - now < 2000) {}
    }
    return;
  }
  if (blockIdx.x == 1) {
    if (threadIdx.x != 0) return;
    for (int i = 0; i < n; ++i) {
      unsigned long long v;
      do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w + i) : "memory"); } while (v == 0);
      seen[i] = gt() - v;
    }
    return;
  }
  if (!load || threadIdx.x != 0) return;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(dsm), bar = ring + 4 * 32768;
  for (int j = 0; j < 4; ++j) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8 * j) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint8_t* s = src + (size_t)blockIdx.x * per;
  const int stages = (int)(per / 32768);
  for (int t = 0; t < stages; ++t) {
    const int j = t & 3;
    if (t >= 4) {
      uint32_t done = 0;
      do { asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar + 8 * j), "r"((uint32_t)(((t >> 2) - 1) & 1)) : "memory"); } while (!done);
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar + 8 * j), "r"(32768) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(ring + j * 32768), "l"(s + (size_t)t * 32768), "r"(32768), "r"(bar + 8 * j) : "memory");
  }
  for (int j = 0; j < 4; ++j) {
    uint32_t done = 0;
    const int last = stages - 4 + j;
    do { asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar + 8 * (last & 3)), "r"((uint32_t)((last >> 2) & 1)) : "memory"); } while (!done);
  }
}
int main() {
  const int n = 64;
  unsigned long long *w, *seen; CK(cudaMalloc(&w, 8 * n)); CK(cudaMalloc(&seen, 8 * n));
  const long long per = 4LL << 20;  // 4 MB per streaming CTA
  uint8_t* src; CK(cudaMalloc(&src, per * 148)); CK(cudaMemset(src, 1, per * 148));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 64));
  std::vector<unsigned long long> h(n);
  for (int load = 0; load < 2; ++load) {
    CK(cudaMemset(w, 0, 8 * n));
    k<<<148, 32, 4 * 32768 + 64>>>(w, seen, n, src, per, load);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), seen, 8 * n, cudaMemcpyDeviceToHost));
    double s = 0, mx = 0; for (auto v : h) { s += v; mx = mx > v ? mx : v; }
    printf("load=%d: store->visible avg %.0f ns max %.0f ns (globaltimer)\n", load, s / n, mx);
  }
  return 0;
}
