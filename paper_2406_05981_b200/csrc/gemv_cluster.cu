// gemv_cluster.cu -- batch-1 LUT-GEMV with the K-split reduced inside a thread-block cluster
// (§8 a2-a6), tiled layout: K <= 4096 (clusters of <= 4), and K <= 8192 for layers <= 12 MB.
//
// Same per-byte hot loop as gemv_tiled.cu (rotated 16-row x 256-k tiles, one PRMT + one
// conflict-free LDS + one FADD per key byte, exponent-add shift per 128-k chunk); different
// decomposition of the reduction:
//
//  * A cluster of C = ceil(S / 4) CTAs owns a band of row groups; CTA rank c owns the slices
//    [c*S/C, (c+1)*S/C) -- at most 4 -- and builds all of their LUTs (a2) once, up front, in
//    four 32 KB slots of shared memory (slots 0/1 are the two column halves of the 64 KB slab
//    at kDynBase, slots 2/3 the halves of a second slab 64 KB higher: both bases fit the LDS
//    immediate, so a lookup is still LDS [R + imm]).
//  * The CTA's items (slice t, row group of the band) go round-robin to its 16 warps and
//    stream through a register ring; with every LUT resident there is no barrier in the loop
//    -- each warp runs at its own pace, as in the split-K kernel.  Each item's 16 row sums
//    land in shared memory, part[t][row]; the CTA sums them over t in order.
//  * The C partial sums meet over distributed shared memory (a5): every CTA pushes its row
//    sums into the owning rank's receive buffer (rank c owns rows [c*chunk, (c+1)*chunk) of
//    the band) with DSMEM stores; after one cluster barrier each owner sums ranks 0..C-1 in
//    that order and stores fp16 (RNE).  Deterministic; no workspace, no global atomics.
//  * The grid is (max co-resident clusters) x C, from cudaOccupancyMaxActiveClusters, so it
//    never needs a second wave.
// In a cluster a CTA's shared addresses carry its rank in bits 24+ (a rank-0 address used by
// rank 1 is an illegal instruction -- measured), so the PRMT that forms a lookup address
// takes byte 3 = rank from the constant registers (see step_sel_c).
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace shiftadd {
namespace {

constexpr int kNW = 16;                   // warps per CTA (16 hi nibbles of the LUT build)
constexpr int kMaxSc = 4;                 // resident LUT slots (slices per CTA)
constexpr int kMaxC = 8;                  // portable cluster size
constexpr int kMaxRGb = 128;              // row groups per band
constexpr int kLutRegion = 2 * kLutBytes; // 128 KB: slots 0-3
constexpr int kXStage = kMaxSc * kTileK * 2;                      // 2 KB
constexpr int kPart = kMaxSc * kMaxRGb * kTileRows * 4;           // 32 KB
constexpr int kRecv = (kMaxRGb * kTileRows + kMaxC) * 4;          // 8 KB + 32 B
constexpr int kDynSmemCl = kLutRegion + kXStage + kPart + kRecv;  // 170 KB

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Shared address of the dynamic region including the cluster-rank bits.
__device__ __forceinline__ uint32_t dyn_smem_base_cluster() {
  asm volatile("" ::"l"(shiftadd_dyn_smem));
  uint32_t b;
  asm("mov.u32 %0, shiftadd_dyn_smem;" : "=r"(b));
  return b;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t local_addr, uint32_t rank, float v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
}

// a2 from staged x: LUT slot at `slot_base` (slab base + 0 / 128 B half) from the 256
// activations at shared address xaddr; warp = hi nibble, lane = 8-k group (column).
__device__ __forceinline__ void build_lut_slot(uint32_t slot_base, uint32_t xaddr, int warp, int lane) {
  uint4 xv;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xv.x), "=r"(xv.y), "=r"(xv.z), "=r"(xv.w)
               : "r"(xaddr + 16 * lane));
  const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
  const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
  const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
  const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
  const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
  const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
  const int hi = warp;
  const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                  ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
  const uint32_t col = slot_base + 4 * lane;
#pragma unroll
  for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), (A[lo & 3] + B[lo >> 2]) + H);
}

// Lookup address of step j: byte 0 = column byte (cst byte j&1), byte 1 = key byte (word
// byte j&3), byte 2 = 0 (cst byte 3), byte 3 = cluster rank (cst byte 2).
__host__ __device__ constexpr uint32_t step_sel_c(int j) {
  return (6u << 12) | (7u << 8) | ((uint32_t)(j & 3) << 4) | (4u + (j & 1));
}

template <int Q, uint32_t IMM>
__device__ __forceinline__ float unit_dot_c(const uint4 (&w)[Q], const int (&e)[Q], const uint32_t (&cst)[8]) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float p0 = 0.f, p1 = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float v = lds_f32(IMM + prmt(word, cst[j >> 1], step_sel_c(j)));
      if (j & 1) p1 += v; else p0 += v;
    }
    acc += shift_pow2(p0 + p1, e[i]);
  }
  return acc;
}

__host__ __device__ constexpr int cl_ring(int Q, int REGS) {
  return (REGS - 56) / (5 * Q) < 1 ? 1 : ((REGS - 56) / (5 * Q) > 8 ? 8 : (REGS - 56) / (5 * Q));
}

// Items of a CTA: i = t * RGb + rgl (slice t of its Sc, row group rgl of the band), warp w
// takes i = w, w + NW, ...; item i is tiled-layout unit (s0 + t) * RG + rg0 + rgl.  The
// warp walks its items with (t, rgl) cursors (no division per item).
struct Cursor {
  int t, rgl;
  __device__ __forceinline__ void advance(int RGb) {
    rgl += kNW;
    while (rgl >= RGb) { rgl -= RGb; ++t; }
  }
};

constexpr int kFlagPdl = 1, kFlagXFirst = 2;

template <int Q, int SCM, int REGS>
__global__ void __launch_bounds__(kNW * 32) __maxnreg__(REGS)
gemv_cluster_kernel(const __half* __restrict__ x, const uint4* __restrict__ planes,
                    const int8_t* __restrict__ exps, int N, int S, int RG, int C, __half* __restrict__ y,
                    int flags, unsigned long long* __restrict__ trace) {
  constexpr int D = cl_ring(Q, REGS);
  const bool pdl = flags & kFlagPdl;
  if (threadIdx.x == 0) check_dyn_base();
  unsigned long long* tr = trace ? trace + 32 * blockIdx.x : nullptr;   // dev trace
  if (tr && threadIdx.x == 0) tr[0] = gtimer_ns();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 1, h = lane & 1;
  const uint32_t rank = cluster_rank();
  // band and slice range in 32-bit arithmetic (cl * RG < 148 * 65536)
  const unsigned Cu = (unsigned)C, ncl = gridDim.x / Cu, cl = blockIdx.x / Cu;
  const int rg0 = (int)((cl * (unsigned)RG) / ncl);
  const int RGb = (int)(((cl + 1) * (unsigned)RG) / ncl) - rg0;
  const int s0 = (int)((rank * (unsigned)S) / Cu);
  const int Sc = (int)(((rank + 1) * (unsigned)S) / Cu) - s0;
  const int Mc = Sc * RGb;
  const int Mw = Mc > warp ? (Mc - warp + kNW - 1) / kNW : 0;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  if (pdl) pdl_launch_dependents();

  const uint32_t base = dyn_smem_base_cluster();   // kDynBase | rank << 24
  const uint32_t xs = base + kLutRegion;
  const uint32_t part = xs + kXStage;
  const bool xthread = tid < Sc * (kTileK / 8);    // one 16-B chunk of x per thread
  const uint4* xsrc = reinterpret_cast<const uint4*>(x + (size_t)s0 * kTileK) + tid;
  Cursor ld{warp / RGb, warp % RGb};
  Cursor pc = ld;
  uint4 w[D][Q];
  int e[D][Q];
  auto stage_x = [&]() {
    if (xthread) {
      const uint4 xv = ldg_keep(xsrc, pol_keep);
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(xs + 16 * tid), "r"(xv.x), "r"(xv.y), "r"(xv.z),
                   "r"(xv.w) : "memory");
      if (tr && threadIdx.x == 0) tr[9] = gtimer_ns();
    }
  };
  auto prefill = [&]() {
#pragma unroll
    for (int k = 0; k < D; ++k)
      if (k < Mw) {
        load_unit<Q>(planes, exps, (long long)(s0 + ld.t) * RG + rg0 + ld.rgl, lane, pol_stream, w[k], e[k]);
        ld.advance(RGb);
      }
  };
  // Weights do not depend on the upstream kernel: under PDL they are requested before
  // griddepcontrol.wait.  Without PDL the order is a measured choice (kFlagXFirst).
  if (pdl || !(flags & kFlagXFirst)) prefill();
  if (pdl) pdl_wait();
  if (tr && threadIdx.x == 0) tr[8] = gtimer_ns();
  stage_x();
  if (!pdl && (flags & kFlagXFirst)) prefill();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[1] = gtimer_ns();
#pragma unroll
  for (int t = 0; t < SCM; ++t)
    if (t < Sc)
      build_lut_slot(base + (uint32_t)(t >> 1) * kLutBytes + (uint32_t)(t & 1) * 128u, xs + t * (kTileK * 2), warp,
                     lane);
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[2] = gtimer_ns();

  // column bytes of steps 2c, 2c+1 for even slots (cstE) and odd slots (+128 B, cstO)
  uint32_t cstE[8], cstO[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t c0 = 4u * (uint32_t)(16 * h + ((2 * c + r) & 15));
    const uint32_t c1 = 4u * (uint32_t)(16 * h + ((2 * c + 1 + r) & 15));
    cstE[c] = c0 | (c1 << 8) | (rank << 16);
    cstO[c] = cstE[c] + 0x8080u;
  }
  for (int b = 0; b < Mw; b += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int m = b + k;
      if (m >= Mw) break;
      float v;
      if (SCM <= 2) {
        v = (pc.t & 1) ? unit_dot_c<Q, kDynBase>(w[k], e[k], cstO) : unit_dot_c<Q, kDynBase>(w[k], e[k], cstE);
      } else {
        switch (pc.t) {   // slot t: slab t >> 1 (LDS immediate), half t & 1 (constant set)
          case 0: v = unit_dot_c<Q, kDynBase>(w[k], e[k], cstE); break;
          case 1: v = unit_dot_c<Q, kDynBase>(w[k], e[k], cstO); break;
          case 2: v = unit_dot_c<Q, kDynBase + kLutBytes>(w[k], e[k], cstE); break;
          default: v = unit_dot_c<Q, kDynBase + kLutBytes>(w[k], e[k], cstO); break;
        }
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (h == 0) sts_f32(part + 4u * (uint32_t)((pc.t * RGb + pc.rgl) * kTileRows + r), v);
      pc.advance(RGb);
      if (m + D < Mw) {
        load_unit<Q>(planes, exps, (long long)(s0 + ld.t) * RG + rg0 + ld.rgl, lane, pol_stream, w[k], e[k]);
        ld.advance(RGb);
      }
    }
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[3] = gtimer_ns();

  // a5: each CTA sums its slices (t in order) per row and pushes the sum into the owner
  // rank's receive buffer, recv[rank][row - owner*chunk], with a DSMEM store; one cluster
  // barrier (release/acquire) publishes them; the owner sums over ranks 0..C-1 in order.
  const int rows = RGb * kTileRows;
  const int chunk = (rows + C - 1) / C;
  const uint32_t recv = part + kPart;
  for (int i = tid; i < rows; i += kNW * 32) {
    float v = 0.f;
    for (int t = 0; t < Sc; ++t) v += lds_f32(part + 4u * (uint32_t)(t * rows + i));
    const int o = i / chunk;
    st_dsmem_f32(recv + 4u * (uint32_t)(rank * chunk + (i - o * chunk)), (uint32_t)o, v);
  }
  cluster_sync();
  if (tr && threadIdx.x == 0) tr[4] = gtimer_ns();
  const int lo = (int)rank * chunk;
  const int cnt = rows - lo < chunk ? rows - lo : chunk;
  for (int j = tid; j < cnt; j += kNW * 32) {
    float v = lds_f32(recv + 4u * (uint32_t)j);
    for (int c = 1; c < C; ++c) v += lds_f32(recv + 4u * (uint32_t)(c * chunk + j));
    const int n = rg0 * kTileRows + lo + j;
    if (n < N) y[n] = __float2half_rn(v);
  }
  if (tr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[5] = gtimer_ns();
    tr[6] = smid;
    tr[7] = (unsigned long long)Mw;
  }
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
int cluster_enabled() {
  static int v = env_int("SHIFTADD_CLUSTER", 1);
  return v;
}
int cluster_trace() {
  static int v = env_int("SHIFTADD_CLUSTER_TRACE", 0);
  return v;
}

// Slices per CTA (LUT slots).  Fewer slots mean fewer serial LUT builds per CTA and a larger
// cluster (more ranks to combine, and clusters of > 4 pack fewer SMs).  Measured on B200
// (tools/sweep_r1t.sh, 4096x4096): 2 slots win below ~5 MB of planes (4096^2 q=2: 4.93 vs
// 5.2 us), 4 above; SHIFTADD_CLUSTER_SC overrides.
struct ClusterShape {
  int sc;   // max slices per CTA (2 or 4)
  int C;    // cluster size
};
constexpr double kSmallLayer = 5.0 * (1 << 20);

ClusterShape cluster_shape(int N, int K, int q) {
  static const int forced = env_int("SHIFTADD_CLUSTER_SC", 0);
  const int S = K / kTileK;
  int sc = forced > 0 ? (forced > kMaxSc ? kMaxSc : forced)
                      : (((double)q * N * K / 8 <= kSmallLayer && (S + 1) / 2 <= kMaxC) ? 2 : kMaxSc);
  return ClusterShape{sc, (S + sc - 1) / sc};
}

template <int Q, int SCM, int REGS>
cudaError_t set_attrs() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(gemv_cluster_kernel<Q, SCM, REGS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kDynSmemCl);
  });
  return err;
}

// Max co-resident clusters of size C (cached per C; the kernels share one resource shape).
int max_clusters(int C) {
  static int cache[kMaxC + 1] = {0};
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (cache[C]) return cache[C];
  if (set_attrs<2, 4, 128>() != cudaSuccess) return 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(C * 64);
  c.blockDim = dim3(kNW * 32);
  c.dynamicSmemBytes = kDynSmemCl;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  c.attrs = &attr;
  c.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemv_cluster_kernel<2, 4, 128>, &c) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[C] = n > 0 ? n : -1;
  return cache[C];
}

int x_first() {
  static int v = env_int("SHIFTADD_CLUSTER_XFIRST", 0);
  return v;
}

template <int Q, int SCM, int REGS>
cudaError_t launch_cluster_q(const GemmArgs& a, const LaunchPlan& p, int C) {
  const cudaError_t ae = set_attrs<Q, SCM, REGS>();
  if (ae != cudaSuccess) return ae;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(p.grid);
  c.blockDim = dim3(p.threads);
  c.dynamicSmemBytes = p.smem;
  c.stream = a.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = attr;
  c.numAttrs = pdl ? 2 : 1;
  unsigned long long* trace = nullptr;
  if (cluster_trace() && a.workspace && a.workspace_bytes >= kCounterBytes + (size_t)p.grid * 256)
    trace = reinterpret_cast<unsigned long long*>(static_cast<char*>(a.workspace) + kCounterBytes);
  const int flags = (pdl ? kFlagPdl : 0) | (x_first() ? kFlagXFirst : 0);
  return cudaLaunchKernelEx(&c, gemv_cluster_kernel<Q, SCM, REGS>, a.x, reinterpret_cast<const uint4*>(a.planes),
                            a.exps, a.N, S, RG, C, a.y, flags, trace);
}

template <int SCM>
cudaError_t launch_cluster_sc(const GemmArgs& a, const LaunchPlan& p, int C) {
  switch (a.q) {
    case 1: return launch_cluster_q<1, SCM, 128>(a, p, C);
    case 2: return launch_cluster_q<2, SCM, 128>(a, p, C);
    case 3: return launch_cluster_q<3, SCM, 128>(a, p, C);
    case 4: return launch_cluster_q<4, SCM, 128>(a, p, C);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// Clusters of <= 4 pack 132 of the 148 SMs; of 5-8 fewer (120 at C = 8, measured), which
// costs more than the grid split-K's hand-off once the layer streams long enough: C > 4 only
// for layers up to kBigC bytes of planes (measured: 2048x8192 q=3 6.2 vs 8.4 us, 8192^2 q=2
// a tie, 28672x8192 q=3 27.7 vs 24.3 us).
constexpr double kBigC = 12.0 * (1 << 20);

bool cluster_applicable(int N, int K, int q, int sms) {
  (void)sms;
  if (!cluster_enabled()) return false;
  const int S = K / kTileK;
  if (S < 1) return false;
  const ClusterShape cs = cluster_shape(N, K, q);
  if (cs.C > kMaxC) return false;
  if (cs.C > 4 && (double)q * N * K / 8 > kBigC) return false;
  const int ncl = max_clusters(cs.C);
  if (ncl <= 0) return false;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int bands = ncl < RG ? ncl : RG;
  return (RG + bands - 1) / bands <= kMaxRGb;
}

LaunchPlan plan_gemv_cluster(int N, int K, int q, int sms) {
  (void)sms;
  const ClusterShape cs = cluster_shape(N, K, q);
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int ncl = max_clusters(cs.C);
  const int bands = ncl < RG ? ncl : RG;
  return LaunchPlan{bands * cs.C, kNW * 32, kDynSmemCl, 3};
}

cudaError_t launch_gemv_cluster(const GemmArgs& a, const LaunchPlan& p) {
  const ClusterShape cs = cluster_shape(a.N, a.K, a.q);
  return cs.sc <= 2 ? launch_cluster_sc<2>(a, p, cs.C) : launch_cluster_sc<4>(a, p, cs.C);
}

}  // namespace shiftadd
