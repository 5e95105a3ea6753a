// latency.cu -- B200 latency microbenchmarks for the split-K / launch design (dev tool).
//   (1) L2-hit and DRAM pointer-chase latency (one thread)
//   (2) grid barrier (red.release + ld.acquire spin) over G CTAs, per barrier
//   (3) back-to-back tiny kernels: stream launches vs CUDA graph vs graph + PDL
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/latency.cu -o tools/latency.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void chase(const unsigned* __restrict__ next, int steps, unsigned* out, long long* cyc) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// `rounds` grid barriers in a row; counter monotonically increases.
__global__ void gbar(unsigned* ctr, int rounds, long long* cyc) {
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      red_rel(ctr, 1u);
      while (ld_acq(ctr) < (unsigned)(r * gridDim.x)) {
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

// B2: relaxed atomic arrival after a fence; the last arriver publishes a generation word
// with st.release; everyone else polls it with ld.acquire (+ short backoff).
__global__ void gbar2(unsigned* ctr, unsigned* flag, int rounds, long long* cyc, int backoff) {
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned old = atomicAdd(ctr, 1u);
      if (old == (unsigned)(r * gridDim.x - 1)) {
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"((unsigned)r) : "memory");
      } else {
        while (ld_acq(flag) < (unsigned)r) {
          if (backoff) __nanosleep(backoff);
        }
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

// B3: as B2, but every CTA polls its own 128-byte flag line; the last arriver's whole CTA
// writes the G flags (one store per thread).
__global__ void gbar3(unsigned* ctr, unsigned* flags, int rounds, long long* cyc) {
  __shared__ int last;
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(ctr, 1u) == (unsigned)(r * gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
      for (int c = threadIdx.x; c < gridDim.x; c += blockDim.x)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + 32 * c), "r"((unsigned)r) : "memory");
    } else if (threadIdx.x == 0) {
      while (ld_acq(flags + 32 * blockIdx.x) < (unsigned)r) {
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

__global__ void tiny(float* p, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[blockIdx.x] += 1.f;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  unsigned *next, *out, *ctr;
  long long* cyc;
  const size_t n_small = 1 << 16, n_big = 1ull << 28;  // 256 KB (L2) and 1 GB (DRAM) rings
  CK(cudaMalloc(&next, n_big * 4));
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&ctr, 64));
  CK(cudaMalloc(&cyc, 64));
  for (int which = 0; which < 2; ++which) {
    const size_t n = which ? n_big : n_small;
    std::vector<unsigned> h(n);
    const size_t stride = which ? 4099 * 32 + 7 : 33;   // hop far (new line / page) each step
    for (size_t i = 0; i < n; ++i) h[i] = (unsigned)((i + stride) % n);
    CK(cudaMemcpy(next, h.data(), n * 4, cudaMemcpyHostToDevice));
    chase<<<1, 1>>>(next, 2000, out, cyc);  // warm
    chase<<<1, 1>>>(next, 2000, out, cyc);
    long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("%s pointer chase: %.0f cycles/load (clock %d MHz nominal)\n", which ? "DRAM" : "L2  ", c / 2000.0, clk_khz / 1000);
  }
  for (int G : {148, 296}) {
    CK(cudaMemset(ctr, 0, 4));
    gbar<<<G, 512>>>(ctr, 100, cyc);
    CK(cudaDeviceSynchronize());
    long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("grid barrier G=%d: %.0f cycles per barrier\n", G, c / 100.0);
  }
  unsigned* flags;
  CK(cudaMalloc(&flags, 4096 * 128));
  for (int G : {148, 296}) {
    for (int bo : {0, 32, 100}) {
      CK(cudaMemset(ctr, 0, 4));
      CK(cudaMemset(flags, 0, 4096 * 128));
      gbar2<<<G, 512>>>(ctr, flags, 100, cyc, bo);
      CK(cudaDeviceSynchronize());
      long long c;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      printf("grid barrier B2 (flag word, backoff %d) G=%d: %.0f cycles\n", bo, G, c / 100.0);
    }
    CK(cudaMemset(ctr, 0, 4));
    CK(cudaMemset(flags, 0, 4096 * 128));
    gbar3<<<G, 512>>>(ctr, flags, 100, cyc);
    CK(cudaDeviceSynchronize());
    long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("grid barrier B3 (per-CTA flags) G=%d: %.0f cycles\n", G, c / 100.0);
  }
  float* p;
  CK(cudaMalloc(&p, 4096 * 4));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 200;
  for (int mode = 0; mode < 3; ++mode) {   // 0 stream, 1 graph, 2 graph+PDL
    cudaGraphExec_t ge = nullptr;
    auto launch = [&](int pdl) {
      cudaLaunchConfig_t c = {};
      c.gridDim = dim3(sms);
      c.blockDim = dim3(256);
      c.stream = s;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      a[0].val.programmaticStreamSerializationAllowed = 1;
      c.attrs = a;
      c.numAttrs = pdl;
      cudaLaunchKernelEx(&c, tiny, p, pdl);
    };
    if (mode > 0) {
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < n; ++i) launch(mode == 2);
      cudaStreamEndCapture(s, &g);
      CK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphLaunch(ge, s);
    } else {
      for (int i = 0; i < n; ++i) launch(0);
    }
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    if (mode > 0) cudaGraphLaunch(ge, s);
    else for (int i = 0; i < n; ++i) launch(0);
    cudaEventRecord(e1, s);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("tiny kernel x%d (%s): %.2f us per kernel\n", n, mode == 0 ? "stream" : mode == 1 ? "graph" : "graph+PDL", ms * 1e3 / n);
  }
  return 0;
}
