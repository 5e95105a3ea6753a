// floor.cu -- B200 floors for one LUT-GEMV call in a PDL chain (development tool, not product).
//  (1) chain: graph of back-to-back kernels with programmatic dependent launch; every kernel
//      triggers its dependents at entry and waits (griddepcontrol.wait) in thread 0.
//      Shapes: small CTAs, one fat CTA per SM, and fat/small alternating (GEMV + reduce).
//  (2) stream: pure weight streaming through a bulk-copy (TMA) ring, no lookups: CTA c copies
//      bytes [c*B/G, (c+1)*B/G) in stages; consumers wait for the PDL dependency before the
//      first stage (as a GEMV must before reading x) then release stages.  Per call time over
//      rotating copies (> 4x L2) for layer sizes of the LLaMA-2 targets; 1 or 2 CTAs per SM.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/floor.cu -o tools/floor.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

extern __shared__ __align__(128) unsigned char dsm[];

__global__ void k_chain(unsigned* sink, int wait_all) {
  pdl_trigger();
  if (threadIdx.x == 0 || wait_all) pdl_wait();
  if (threadIdx.x == 0 && sink && blockIdx.x == 0) sink[0] += 1;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Stream kernel: NW consumer warps + 1 producer warp.  ring bytes = nst * stage.
// trace (optional): per CTA [start, wait_ret, first_full, last_full, end]
__global__ void k_stream(const uint8_t* __restrict__ src, long long bytes, int stage, int nst, int consume,
                         unsigned long long* trace, int pre_stages) {
  const int NW = blockDim.x / 32 - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long t0 = gtimer();
  pdl_trigger();
  const long long b0 = ((long long)blockIdx.x * bytes / gridDim.x) & ~15LL;
  const long long b1 = blockIdx.x + 1 == gridDim.x ? bytes : (((long long)(blockIdx.x + 1) * bytes / gridDim.x) & ~15LL);
  const int nstages = (int)((b1 - b0 + stage - 1) / stage);
  const uint32_t ring = smem_u32(dsm);
  const uint32_t full = ring + nst * stage, empty = full + 8 * 16;
  if (threadIdx.x == 0) {
    for (int j = 0; j < nst; ++j) { mbar_init(full + 8 * j, 1); mbar_init(empty + 8 * j, NW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  unsigned long long tw = 0, tf = 0, tl = 0;
  if (warp == NW) {
    if (lane == 0) {
      const uint64_t pol = pol_ef();
      for (int t = 0; t < nstages; ++t) {
        const int j = t % nst;
        if (t == pre_stages) pdl_wait();
        if (t >= nst) mbar_wait(empty + 8 * j, (uint32_t)((t / nst - 1) & 1));
        const long long a = b0 + (long long)t * stage;
        const uint32_t n = (uint32_t)((b1 - a) < stage ? (b1 - a) : stage);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * j), "r"(n) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(ring + j * stage), "l"(src + a), "r"(n), "r"(full + 8 * j), "l"(pol) : "memory");
      }
    }
  } else {
    pdl_wait();
    tw = gtimer();
    uint32_t acc = 0;
    for (int t = 0; t < nstages; ++t) {
      const int j = t % nst;
      mbar_wait(full + 8 * j, (uint32_t)((t / nst) & 1));
      if (t == 0) tf = gtimer();
      if (t == nstages - 1) tl = gtimer();
      if (consume) {   // every consumer warp reads its share of the stage with LDS.128
        for (int o = (warp * 32 + lane) * 16; o < stage; o += NW * 32 * 16) {
          uint4 v;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "r"(ring + j * stage + o));
          acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
    }
    if (acc == 0x9e3779b9u) asm volatile("trap;");
  }
  __syncthreads();
  if (trace && threadIdx.x == 0) {
    unsigned long long* tr = trace + 8 * blockIdx.x;
    tr[0] = t0; tr[1] = tw; tr[2] = tf; tr[3] = tl; tr[4] = gtimer();
  }
}

// PDL probe: a dependent CTA issues one bulk copy (and one LDG) at entry and records when each
// lands, without calling griddepcontrol.wait first; then waits and records that.
__global__ void k_probe(const uint8_t* __restrict__ src, int bytes, unsigned long long* out, int mode) {
  unsigned long long t0 = gtimer();
  pdl_trigger();
  const uint32_t buf = smem_u32(dsm), bar = buf + 65536;
  unsigned long long t_copy = 0, t_ldg = 0, t_wait = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode & 1) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(buf), "l"(src + (size_t)blockIdx.x * bytes), "r"(bytes), "r"(bar) : "memory");
      mbar_wait(bar, 0);
      t_copy = gtimer();
    }
    if ((mode & 3) == 2 || mode == 3) {
      unsigned v = *(volatile const unsigned*)(src + (size_t)blockIdx.x * bytes + 64 * 1024 * 1024);
      if (v == 0x12345u) asm volatile("trap;");
      t_ldg = gtimer();
    }
    pdl_wait();
    t_wait = gtimer();
    unsigned long long* o = out + 4 * blockIdx.x;
    o[0] = t0; o[1] = t_copy; o[2] = t_ldg; o[3] = t_wait;
  }
}

// small reduce-like kernel (co-resident with fat CTAs)
__global__ void k_small(const float* __restrict__ in, float* __restrict__ out, int n) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] * 2.f;
}

static cudaLaunchAttribute g_attr[1];
template <typename... A>
static void launch(void (*k)(A...), dim3 grid, dim3 block, int smem, cudaStream_t s, bool pdl, A... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = grid; c.blockDim = block; c.dynamicSmemBytes = smem; c.stream = s;
  g_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  g_attr[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = g_attr; c.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&c, k, args...));
}

template <typename F>
static float time_graph(cudaStream_t s, int n, F body, int reps = 5) {
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < n; ++i) body(i);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a, s); CK(cudaGraphLaunch(ge, s)); cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
  }
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  return best * 1000.f / n;   // us per body
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  const int sms = pr.multiProcessorCount;
  printf("device %s, %d SMs, L2 %d MB\n", pr.name, sms, pr.l2CacheSize >> 20);
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  unsigned* sink; CK(cudaMalloc(&sink, 64));
  CK(cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));

  // (1) chains
  struct C { const char* name; int ctas, thr, smem, wait_all; };
  C cs[] = {{"148x32 thr, no smem", sms, 32, 0, 0},
            {"148x544 thr, 200KB smem (1 CTA/SM)", sms, 544, 200 * 1024, 0},
            {"148x544 thr, 200KB, all threads wait", sms, 544, 200 * 1024, 1},
            {"296x288 thr, 100KB (2 CTA/SM)", 2 * sms, 288, 100 * 1024, 0},
            {"120x544 thr, 200KB", 120, 544, 200 * 1024, 0}};
  for (auto& c : cs) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      float us = time_graph(s, 200, [&](int) { launch(k_chain, dim3(c.ctas), dim3(c.thr), c.smem, s, pdl == 1, sink, c.wait_all); });
      printf("chain %-40s pdl=%d : %.3f us/launch\n", c.name, pdl, us);
    }
  }
  float *fa, *fb; CK(cudaMalloc(&fa, 1 << 22)); CK(cudaMalloc(&fb, 1 << 22));
  {
    float us = time_graph(s, 100, [&](int) {
      launch(k_chain, dim3(sms), dim3(544), 200 * 1024, s, true, sink, 0);
      launch(k_small, dim3(sms), dim3(256), 0, s, true, (const float*)fa, fb, 28672 * 8);
    });
    printf("chain fat(200KB)+small(reduce 28672x8 f32) pairs: %.3f us/pair\n", us);
  }

  // (3) does a PDL dependent's bulk copy issued before griddepcontrol.wait land while the
  //     primary still runs?  primary: one long streaming call (93 MB, 2 CTAs/SM of ~100 KB so
  //     the probe's 64 KB CTA fits beside it); probe: copy 16 KB at entry.
  {
    const size_t pbytes = (size_t)512 << 20;
    uint8_t* pb; CK(cudaMalloc(&pb, pbytes)); CK(cudaMemset(pb, 1, pbytes));
    unsigned long long* po; CK(cudaMalloc(&po, 4 * 8 * 2 * sms));
    unsigned long long* tr1; CK(cudaMalloc(&tr1, 8 * 8 * 2 * sms));
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64));
    for (int mode = 1; mode <= 7; ++mode) {
      const long long bytes = 93660000LL & ~15LL;
      if (mode <= 3)
        launch(k_stream, dim3(2 * sms), dim3(9 * 32), 4 * 24 * 1024 + 256, s, false, (const uint8_t*)pb, bytes, 24 * 1024, 4, 0, tr1, 1 << 30);
      else   // one 100 KB CTA per SM: the probe's CTA is co-resident from the start
        launch(k_stream, dim3(sms), dim3(17 * 32), 4 * 24 * 1024 + 256, s, false, (const uint8_t*)pb, bytes, 24 * 1024, 4, 0, tr1, 1 << 30);
      launch(k_probe, dim3(sms), dim3(32), 65536 + 64, s, true, (const uint8_t*)(pb + ((size_t)256 << 20)), 16384, po, mode);
      CK(cudaStreamSynchronize(s));
      std::vector<unsigned long long> h(4 * sms), t(8 * 2 * sms);
      CK(cudaMemcpy(h.data(), po, h.size() * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(t.data(), tr1, t.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long p0 = ~0ull, pend = 0;
      for (int c = 0; c < (mode <= 3 ? 2 : 1) * sms; ++c) { p0 = std::min(p0, t[8 * c]); pend = std::max(pend, t[8 * c + 4]); }
      double a[4] = {0, 0, 0, 0}; int nn = 0;
      for (int c = 0; c < sms; ++c) {
        for (int k = 0; k < 4; ++k) if (h[4 * c + k]) a[k] += (double)(h[4 * c + k] - p0) / 1e3;
        ++nn;
      }
      printf("probe mode %d: primary 0 .. %.2f us; dependent avg: start %.2f copy-landed %.2f ldg-landed %.2f wait-returned %.2f us\n",
             mode, (pend - p0) / 1e3, a[0] / nn, a[1] / nn, a[2] / nn, a[3] / nn);
    }
  }

  // (4) footprint sweep: same 4.47 MB calls over rotating buffers of total footprint F
  if (argc > 1) {
    const long long bytes = 4470000LL & ~15LL;
    const size_t pool4 = (size_t)2 << 30;
    uint8_t* b4; CK(cudaMalloc(&b4, pool4)); CK(cudaMemset(b4, 1, pool4));
    unsigned long long* tr4; CK(cudaMalloc(&tr4, 8 * 8 * sms));
    for (double fmb : {4.47, 64.0, 130.0, 250.0, 540.0, 1000.0, 2000.0}) {
      int R = std::max(1, (int)(fmb * 1e6 / bytes));
      float us = time_graph(s, 240, [&](int i) {
        launch(k_stream, dim3(sms), dim3(17 * 32), 8 * 24 * 1024 + 256, s, true, (const uint8_t*)(b4 + (size_t)(i % R) * bytes),
               bytes, 24 * 1024, 8, 0, (unsigned long long*)nullptr, 1 << 30);
      });
      for (int i = 0; i < 8; ++i)
        launch(k_stream, dim3(sms), dim3(17 * 32), 8 * 24 * 1024 + 256, s, true, (const uint8_t*)(b4 + (size_t)(i % R) * bytes),
               bytes, 24 * 1024, 8, 0, i == 7 ? tr4 : (unsigned long long*)nullptr, 1 << 30);
      CK(cudaStreamSynchronize(s));
      std::vector<unsigned long long> h(8 * sms);
      CK(cudaMemcpy(h.data(), tr4, h.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < sms; ++c) t0 = std::min(t0, h[8 * c]);
      double a[5] = {0};
      for (int c = 0; c < sms; ++c) for (int k = 0; k < 5; ++k) a[k] += (double)(h[8 * c + k] - t0) / 1e3 / sms;
      printf("footprint %7.1f MB (R=%d): %.3f us/call; avg start %.2f wait %.2f first %.2f last %.2f end %.2f\n", fmb, R, us,
             a[0], a[1], a[2], a[3], a[4]);
    }
    return 0;
  }

  // (2) streaming
  const double l2 = pr.l2CacheSize;
  const double sizes_mb[] = {4.47, 6.70, 11.93, 17.90, 22.55, 93.66};
  const size_t pool = (size_t)2 << 30;   // 2 GB of rotating weights
  uint8_t* buf; CK(cudaMalloc(&buf, pool)); CK(cudaMemset(buf, 1, pool));
  unsigned long long* trace; CK(cudaMalloc(&trace, 8 * 8 * 2 * sms * sizeof(unsigned long long)));
  struct V { const char* name; int cpsm, stage, nst, consume, pre; };
  V vs[] = {{"1 CTA/SM ring 8x24KB", 1, 24 * 1024, 8, 0, 1 << 30},
            {"1 CTA/SM ring 8x24KB +LDS", 1, 24 * 1024, 8, 1, 1 << 30},
            {"1 CTA/SM ring 8x16KB", 1, 16 * 1024, 8, 0, 1 << 30},
            {"1 CTA/SM ring 4x32KB", 1, 32 * 1024, 4, 0, 1 << 30},
            {"1 CTA/SM ring 8x24KB pre=1", 1, 24 * 1024, 8, 0, 1},
            {"2 CTA/SM ring 6x16KB", 2, 16 * 1024, 6, 0, 1 << 30},
            {"2 CTA/SM ring 6x16KB +LDS", 2, 16 * 1024, 6, 1, 1 << 30},
            {"2 CTA/SM ring 4x24KB", 2, 24 * 1024, 4, 0, 1 << 30}};
  for (double mb : sizes_mb) {
    const long long bytes = ((long long)(mb * 1e6) + 15) & ~15LL;
    int R = (int)std::max(4.0 * l2 / bytes, 4.0) + 1;
    R = std::min<long long>(R, pool / bytes);
    for (auto& v : vs) {
      const int ctas = v.cpsm * sms;
      const int thr = v.cpsm == 1 ? 17 * 32 : 9 * 32;
      const int smem = v.nst * v.stage + 256;
      float us = time_graph(s, R * 4, [&](int i) {
        launch(k_stream, dim3(ctas), dim3(thr), smem, s, true, (const uint8_t*)(buf + (size_t)(i % R) * bytes), bytes,
               v.stage, v.nst, v.consume, (unsigned long long*)nullptr, v.pre);
      });
      printf("stream %7.2f MB %-30s R=%3d : %7.3f us/call  %7.1f GB/s\n", mb, v.name, R, us, bytes / (us * 1e3));
    }
    // one traced chain (1 CTA/SM ring 8x24KB): per-CTA phase times relative to the call's first CTA start
    {
      const int ctas = sms;
      for (int i = 0; i < 8; ++i)
        launch(k_stream, dim3(ctas), dim3(17 * 32), 8 * 24 * 1024 + 256, s, true,
               (const uint8_t*)(buf + (size_t)(i % R) * bytes), bytes, 24 * 1024, 8, 0, i == 7 ? trace : (unsigned long long*)nullptr, 1 << 30);
      CK(cudaStreamSynchronize(s));
      std::vector<unsigned long long> h(8 * ctas);
      CK(cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull, te = 0;
      for (int c = 0; c < ctas; ++c) { t0 = std::min(t0, h[8 * c]); te = std::max(te, h[8 * c + 4]); }
      double mx[5] = {0}, mn[5] = {1e30, 1e30, 1e30, 1e30, 1e30}, av[5] = {0};
      for (int c = 0; c < ctas; ++c)
        for (int k = 0; k < 5; ++k) {
          double v = (double)(h[8 * c + k] - t0) / 1e3;
          mx[k] = std::max(mx[k], v); mn[k] = std::min(mn[k], v); av[k] += v / ctas;
        }
      const char* nm[5] = {"start", "wait", "first", "last", "end"};
      printf("  trace %.2f MB:", mb);
      for (int k = 0; k < 5; ++k) printf(" %s %.2f/%.2f/%.2f", nm[k], mn[k], av[k], mx[k]);
      printf(" us (min/avg/max)\n");
    }
  }
  printf("done\n");
  return 0;
}
