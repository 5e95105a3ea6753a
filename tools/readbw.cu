// readbw.cu -- streaming-read microbenchmarks on B200 (development tool, not product code).
// Measures which load structure reaches HBM read bandwidth for the LUT-GEMV access pattern:
// a CTA streams one contiguous chunk of 512-byte tiles (one LDG.128 per lane per tile).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/readbw.cu -o /tmp/readbw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_na(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ldg_na256(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ldg_plain(const uint4* p) { return __ldg(p); }

// (1) grid-stride, D independent 16-B loads per thread per iteration
template <int D>
__global__ void k_gridstride(const uint4* __restrict__ a, size_t n16, unsigned* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (D - 1) * stride < n16; i += D * stride) {
    uint4 v[D];
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = ldg_na(a + i + d * stride);
#pragma unroll
    for (int d = 0; d < D; ++d) acc ^= v[d].x ^ v[d].y ^ v[d].z ^ v[d].w;
  }
  for (; i < n16; i += stride) { uint4 v = ldg_na(a + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// (2) chunked: CTA c owns tiles [c*T/G, (c+1)*T/G); warp w takes tiles w, w+NW, ...; each
// warp keeps D tiles in flight (LDG.128 per lane per 512-B tile).  MODE 0: .na, 1: .na.L2::256B
template <int D, int MODE>
__global__ void k_chunk(const uint4* __restrict__ a, long long T, unsigned* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const long long t0 = (blockIdx.x * T) / gridDim.x, t1 = ((blockIdx.x + 1) * T) / gridDim.x;
  uint32_t acc = 0;
  long long t = t0 + warp;
  for (; t + (long long)(D - 1) * NW < t1; t += (long long)D * NW) {
    uint4 v[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const uint4* p = a + (t + (long long)d * NW) * 32 + lane;
      v[d] = MODE == 1 ? ldg_na256(p) : ldg_na(p);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) acc ^= v[d].x ^ v[d].y ^ v[d].z ^ v[d].w;
  }
  for (; t < t1; t += NW) { uint4 v = ldg_na(a + t * 32 + lane); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// (3) chunk + bulk L2 prefetch of the whole remaining window ahead, issued by lane 0 of each warp
template <int D>
__global__ void k_chunk_pf(const uint4* __restrict__ a, long long T, unsigned* out, int pf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const long long t0 = (blockIdx.x * T) / gridDim.x, t1 = ((blockIdx.x + 1) * T) / gridDim.x;
  uint32_t acc = 0;
  long long t = t0 + warp;
  long long p = t;
  for (; t + (long long)(D - 1) * NW < t1; t += (long long)D * NW) {
    const long long lim = min(t1, t + (long long)(D + pf) * NW);
    for (; p < lim; p += NW)
      if (lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;" ::"l"(a + p * 32) : "memory");
    uint4 v[D];
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = ldg_na(a + (t + (long long)d * NW) * 32 + lane);
#pragma unroll
    for (int d = 0; d < D; ++d) acc ^= v[d].x ^ v[d].y ^ v[d].z ^ v[d].w;
  }
  for (; t < t1; t += NW) { uint4 v = ldg_na(a + t * 32 + lane); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) f(i);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) f(i);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes_per = 96ull << 20;   // one "layer" ~ LLaMA-70B MLP matrix
  const int R = 6;                        // rotating copies (> 4 x L2)
  uint8_t* buf; unsigned* out;
  CK(cudaMalloc(&buf, bytes_per * R));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf, 1, bytes_per * R));
  auto A = [&](int i) { return reinterpret_cast<const uint4*>(buf + (size_t)(i % R) * bytes_per); };
  const size_t n16 = bytes_per / 16;
  const long long T = bytes_per / 512;
  auto rep = [&](const char* name, float ms, size_t b) { printf("%-44s %8.2f us  %7.1f GB/s\n", name, ms * 1e3, b / (ms * 1e-3) / 1e9); };
  for (int blocks_per : {1, 2, 4, 8}) {
    for (int thr : {256, 512, 1024}) {
      char nm[96];
      snprintf(nm, sizeof nm, "gridstride D=4 grid=%dx%d thr=%d", sms, blocks_per, thr);
      rep(nm, timeit([&](int i) { k_gridstride<4><<<sms * blocks_per, thr>>>(A(i), n16, out); }, 20), bytes_per);
    }
  }
  for (int nw : {8, 16, 32}) for (int per : {1, 2}) {
    char nm[96];
    snprintf(nm, sizeof nm, "chunk D=1 NW=%d per_sm=%d", nw, per);
    rep(nm, timeit([&](int i) { k_chunk<1, 0><<<sms * per, nw * 32>>>(A(i), T, out); }, 20), bytes_per);
    snprintf(nm, sizeof nm, "chunk D=2 NW=%d per_sm=%d", nw, per);
    rep(nm, timeit([&](int i) { k_chunk<2, 0><<<sms * per, nw * 32>>>(A(i), T, out); }, 20), bytes_per);
    snprintf(nm, sizeof nm, "chunk D=4 NW=%d per_sm=%d", nw, per);
    rep(nm, timeit([&](int i) { k_chunk<4, 0><<<sms * per, nw * 32>>>(A(i), T, out); }, 20), bytes_per);
    snprintf(nm, sizeof nm, "chunk D=4 L2::256B NW=%d per_sm=%d", nw, per);
    rep(nm, timeit([&](int i) { k_chunk<4, 1><<<sms * per, nw * 32>>>(A(i), T, out); }, 20), bytes_per);
    snprintf(nm, sizeof nm, "chunk D=8 NW=%d per_sm=%d", nw, per);
    rep(nm, timeit([&](int i) { k_chunk<8, 0><<<sms * per, nw * 32>>>(A(i), T, out); }, 20), bytes_per);
    for (int pf : {8, 32}) {
      snprintf(nm, sizeof nm, "chunk D=2 +L2pf %d NW=%d per_sm=%d", pf, nw, per);
      rep(nm, timeit([&](int i) { k_chunk_pf<2><<<sms * per, nw * 32>>>(A(i), T, out, pf); }, 20), bytes_per);
    }
  }
  // small transfers: fixed overhead per launch
  for (size_t small : {4ull << 20, 16ull << 20, 32ull << 20}) {
    const long long Ts = small / 512;
    char nm[96];
    snprintf(nm, sizeof nm, "chunk D=4 NW=16 %zu MB", small >> 20);
    rep(nm, timeit([&](int i) { k_chunk<4, 0><<<sms, 512>>>(A(i), Ts, out); }, 50), small);
  }
  printf("empty-ish launch: %8.2f us\n", timeit([&](int i) { k_chunk<1, 0><<<sms, 256>>>(A(i), 0, out); }, 100) * 1e3);
  return 0;
}
