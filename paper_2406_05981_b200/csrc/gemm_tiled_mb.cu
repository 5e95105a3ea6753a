// gemm_tiled_mb.cu -- §8 a7: small-batch (2 <= M <= 16) LUT-GEMM on the tiled layout.
//
// Same work decomposition, lane mapping and split-K reduction as gemv_tiled.cu, but each
// LUT entry carries the partial sums of MC batch rows -- MC = 4 (one float4, LDS.128) or, for
// M = 2, MC = 2 (one float2, LDS.64) -- so one key byte loaded from HBM and one LDS serve MC
// rows (App. D :804-817 evaluates batch 1/2/4/8).  Rows are processed in
// ceil(M/MC) chunks; the CTA re-walks its own units for each chunk, which it just read, so
// chunks after the first stream from L2.  Each warp keeps D units in flight in a register
// ring (D from the register budget; a 2-deep double buffer measured latency-bound).
//
// MC = 4 LUT slab for one 256-k slice and one row chunk: 2 regions (h = chunk half of the
// tile) x 256 keys x 16 columns x 16 B = 128 KB.  Entry (key, group t) lives at byte offset
//     (t >> 4) * 64 KB + key * 256 + ((t & 15) ^ (4 * (t >> 4))) * 16
// -- one PRMT builds it from the key byte; the LDS adds the (uniform) region base.  The XOR
// swizzle makes the 8 lanes of every LDS.128 phase (rows r..r+3, halves 0/1) hit 8 distinct
// 16-B bank quads: conflict free.
// MC = 2 slab: 256 keys x 32 columns x 8 B = 64 KB, entry (key, t) at
//     key * 256 + ((t & 15) ^ (8 * (t >> 4)) + 16 * (t >> 4)) * 8
// -- an LDS.64 phase is 16 lanes (rows r..r+7, halves 0/1); lanes of half 0 read 8
// consecutive columns mod 16, and the XOR 8 sends half 1's to the complementary 8, so the 16
// lanes cover 32 distinct banks.
// With M rows the smem traffic per weight byte is 4*M bytes, so for M >= 2 the shared-
// memory bandwidth (128 B/clk/SM), not HBM, is the roof.
#include <mutex>

#include "common.cuh"

namespace shiftadd {
namespace {

constexpr int kMC = 4;                       // batch rows per LUT entry (the float4 variant)
constexpr int kLutMbBytes = 2 * 256 * 256;   // 128 KB
constexpr int kDynSmemMb = kLutMbBytes;

// MC = 2: column position of group t (see the header).
__host__ __device__ constexpr int swz2(int t) { return ((t & 15) ^ (8 * (t >> 4))) + 16 * (t >> 4); }

template <int NW>
__device__ __forceinline__ void build_lut2(const __half* __restrict__ x, int ldx, int m0, int M, int s,
                                           uint32_t lut, int warp, int lane) {
  float L[2][16];
  float X4[2][4];
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    float xv[8];
    if (m0 + mm < M) {
      const uint4 raw = *reinterpret_cast<const uint4*>(x + (size_t)(m0 + mm) * ldx + s * kTileK + 8 * lane);
      const __half2* hp = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float2 f = __half22float2(hp[b]);
        xv[2 * b] = f.x;
        xv[2 * b + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) xv[b] = 0.f;
    }
    const float A[4] = {-xv[0] - xv[1], xv[0] - xv[1], xv[1] - xv[0], xv[0] + xv[1]};
    const float B[4] = {-xv[2] - xv[3], xv[2] - xv[3], xv[3] - xv[2], xv[2] + xv[3]};
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) L[mm][lo] = A[lo & 3] + B[lo >> 2];
#pragma unroll
    for (int b = 0; b < 4; ++b) X4[mm][b] = xv[4 + b];
  }
  const uint32_t col = lut + (uint32_t)swz2(lane) * 8u;
#pragma unroll
  for (int hh = 0; hh < 16 / NW; ++hh) {
    const int hi = warp + NW * hh;
    float H[2];
#pragma unroll
    for (int mm = 0; mm < 2; ++mm)
      H[mm] = ((hi & 1 ? X4[mm][0] : -X4[mm][0]) + (hi & 2 ? X4[mm][1] : -X4[mm][1])) +
              ((hi & 4 ? X4[mm][2] : -X4[mm][2]) + (hi & 8 ? X4[mm][3] : -X4[mm][3]));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) {
      const float a = L[0][lo] + H[0], b = L[1][lo] + H[1];
      asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(col + ((hi * 16 + lo) << 8)), "f"(a), "f"(b) : "memory");
    }
  }
}

template <int Q>
__device__ __forceinline__ void unit_dot2(const uint4 (&w)[Q], const int (&e)[Q], uint32_t lut,
                                          const uint32_t (&cst)[16], float (&acc)[4]) {
  acc[0] = acc[1] = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float2 p0 = make_float2(0.f, 0.f), p1 = p0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      // byte0 <- swizzled col*8, byte1 <- key, bytes 2-3 <- 0
      const uint32_t off = __byte_perm(word, cst[j], 0x5504u | ((uint32_t)(j & 3) << 4));
      float2 v;
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(lut + off));
      if (j & 1) { p1.x += v.x; p1.y += v.y; }
      else { p0.x += v.x; p0.y += v.y; }
    }
    acc[0] += shift_pow2(p0.x + p1.x, e[i]);
    acc[1] += shift_pow2(p0.y + p1.y, e[i]);
  }
}

template <int NW>
__device__ __forceinline__ void build_lut4(const __half* __restrict__ x, int ldx, int m0, int M, int s,
                                           uint32_t lut, int warp, int lane) {
  // thread (warp w, lane t): group t of the slice, every hi nibble assigned to the warp.
  float L[kMC][16];
  float X4[kMC][4];  // x4..x7 of each row, for the hi-nibble half sums
#pragma unroll
  for (int mm = 0; mm < kMC; ++mm) {
    float xv[8];
    if (m0 + mm < M) {
      const uint4 raw = *reinterpret_cast<const uint4*>(x + (size_t)(m0 + mm) * ldx + s * kTileK + 8 * lane);
      const __half2* hp = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float2 f = __half22float2(hp[b]);
        xv[2 * b] = f.x;
        xv[2 * b + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) xv[b] = 0.f;
    }
    const float A[4] = {-xv[0] - xv[1], xv[0] - xv[1], xv[1] - xv[0], xv[0] + xv[1]};
    const float B[4] = {-xv[2] - xv[3], xv[2] - xv[3], xv[3] - xv[2], xv[2] + xv[3]};
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) L[mm][lo] = A[lo & 3] + B[lo >> 2];
#pragma unroll
    for (int b = 0; b < 4; ++b) X4[mm][b] = xv[4 + b];
  }
  const int t = lane;
  const uint32_t col = lut + (t >> 4) * 65536 + (((t & 15) ^ (4 * (t >> 4))) << 4);
#pragma unroll
  for (int hh = 0; hh < 16 / NW; ++hh) {
    const int hi = warp + NW * hh;
    float H[kMC];
#pragma unroll
    for (int mm = 0; mm < kMC; ++mm)
      H[mm] = ((hi & 1 ? X4[mm][0] : -X4[mm][0]) + (hi & 2 ? X4[mm][1] : -X4[mm][1])) +
              ((hi & 4 ? X4[mm][2] : -X4[mm][2]) + (hi & 8 ? X4[mm][3] : -X4[mm][3]));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) {
      float4 v;
      v.x = L[0][lo] + H[0];
      v.y = L[1][lo] + H[1];
      v.z = L[2][lo] + H[2];
      v.w = L[3][lo] + H[3];
      sts_f32x4(col + ((hi * 16 + lo) << 8), v);
    }
  }
}

template <int Q>
__device__ __forceinline__ void unit_dot4(const uint4 (&w)[Q], const int (&e)[Q], uint32_t lut,
                                          const uint32_t (&cst)[16], float (&acc)[4]) {
#pragma unroll
  for (int mm = 0; mm < kMC; ++mm) acc[mm] = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      // byte0 <- swizzled col*16, byte1 <- key, byte2 <- region h, byte3 <- 0
      const uint32_t off = __byte_perm(word, cst[j], 0x7604u | ((uint32_t)(j & 3) << 4));
      const float4 v = lds_f32x4(lut + off);
      if (j & 1) { p1.x += v.x; p1.y += v.y; p1.z += v.z; p1.w += v.w; }
      else { p0.x += v.x; p0.y += v.y; p0.z += v.z; p0.w += v.w; }
    }
    acc[0] += shift_pow2(p0.x + p1.x, e[i]);
    acc[1] += shift_pow2(p0.y + p1.y, e[i]);
    acc[2] += shift_pow2(p0.z + p1.z, e[i]);
    acc[3] += shift_pow2(p0.w + p1.w, e[i]);
  }
}

// units in flight per warp within 128 registers (the float4 variant keeps more live state)
__host__ __device__ constexpr int mb_ring(int Q, int MC) {
  return (128 - (MC == 4 ? 90 : 80)) / (5 * Q) < 2 ? 2
         : ((128 - (MC == 4 ? 90 : 80)) / (5 * Q) > 4 ? 4 : (128 - (MC == 4 ? 90 : 80)) / (5 * Q));
}

template <int Q, int NW, int MC>
__global__ void __launch_bounds__(NW * 32, 1)
gemm_tiled_mb_kernel(const __half* __restrict__ x, int ldx, const uint4* __restrict__ planes,
                     const int8_t* __restrict__ exps, int M, int N, int S, int RG, long long U,
                     __half* __restrict__ y, int ldy, float* __restrict__ partial, unsigned* __restrict__ cnt,
                     int pdl) {
  constexpr int D = mb_ring(Q, MC);
  if (threadIdx.x == 0) check_dyn_base();
  const uint32_t lut = kDynBase;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 1, h = lane & 1;
  const long long G = gridDim.x;
  const long long u0 = ((long long)blockIdx.x * U) / G;
  const long long u1 = ((long long)(blockIdx.x + 1) * U) / G;
  const size_t Npad = (size_t)RG * kTileRows;

  uint32_t cst[16];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    cst[j] = MC == 4 ? (((uint32_t)((((j + r) & 15) ^ (4 * h)) << 4)) | ((uint32_t)h << 16))
                     : (uint32_t)(swz2(16 * h + ((j + r) & 15)) * 8);

  if (pdl) pdl_launch_dependents();
  const uint64_t pol = policy_evict_first();
  uint4 w[D][Q];
  int e[D][Q];
  bool waited = false;
  for (int m0 = 0; m0 < M; m0 += MC) {
    long long u = u0;
    while (u < u1) {
      const int s = (int)(u / RG);
      const long long seg_end = min(u1, (long long)(s + 1) * RG);
      const long long first = u + warp;
      // ring prefill: units first + k*NW, k < D
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (first + (long long)k * NW < seg_end) load_unit<Q>(planes, exps, first + (long long)k * NW, lane, pol, w[k], e[k]);
      if (!waited) {
        if (pdl) pdl_wait();
        waited = true;
      }
      __syncthreads();  // previous LUT fully consumed
      if (MC == 4) build_lut4<NW>(x, ldx, m0, M, s, lut, warp, lane);
      else build_lut2<NW>(x, ldx, m0, M, s, lut, warp, lane);
      __syncthreads();
      const long long rg_base = (long long)s * RG;
      for (long long base = first; base < seg_end; base += (long long)D * NW) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const long long uu = base + (long long)k * NW;
          if (uu >= seg_end) break;
          float acc[4];
          if (MC == 4) unit_dot4<Q>(w[k], e[k], lut, cst, acc);
          else unit_dot2<Q>(w[k], e[k], lut, cst, acc);
          const long long un = uu + (long long)D * NW;
          if (un < seg_end) load_unit<Q>(planes, exps, un, lane, pol, w[k], e[k]);
#pragma unroll
          for (int mm = 0; mm < MC; ++mm) acc[mm] += __shfl_xor_sync(0xffffffffu, acc[mm], 1);
          const int n = (int)(uu - rg_base) * kTileRows + r;
          if (h == 0) {
#pragma unroll
            for (int mm = 0; mm < MC; ++mm) {
              const int m = m0 + mm;
              if (m < M) {
                if (S == 1) { if (n < N) y[(size_t)m * ldy + n] = __float2half_rn(acc[mm]); }
                else partial[((size_t)m * S + s) * Npad + n] = acc[mm];
              }
            }
          }
        }
      }
      u = seg_end;
    }
  }
  if (S == 1) return;

  // Deterministic split-K reduction, balanced over the grid, with per-row-group arrival
  // counters exactly as in gemv_tiled.cu (each counter counts the (slice, rg) units of all
  // row chunks, so the owner waits for S * ceil(M/4) arrivals).
  const long long own0 = ((long long)blockIdx.x * RG) / G;
  const long long own1 = ((long long)(blockIdx.x + 1) * RG) / G;
  const long long n0 = own0 * kTileRows;
  const long long rows = (own1 - own0) * kTileRows;
  const unsigned expect = (unsigned)S * (unsigned)((M + MC - 1) / MC);
  __syncthreads();
  if (tid == 0) __threadfence();
  __syncthreads();
  for (int m0 = 0; m0 < M; m0 += MC)
    for (long long uq = u0 + tid; uq < u1; uq += NW * 32)
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + (uq % RG)) : "memory");
  for (long long rg = own0 + tid; rg < own1; rg += NW * 32)
    while (ld_acquire_gpu(cnt + rg) < expect) {
    }
  __syncthreads();
  for (long long it = tid; it < rows * M; it += NW * 32) {
    const int m = (int)(it / rows);
    const long long n = n0 + (it - (long long)m * rows);
    const float* p = partial + (size_t)m * S * Npad + n;
    float sum = 0.f;
    for (int s = 0; s < S; s += 16) {
      float v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = (s + k < S) ? __ldcg(p + (size_t)(s + k) * Npad) : 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) sum += v[k];
    }
    if (n < N) y[(size_t)m * ldy + n] = __float2half_rn(sum);
  }
  for (long long rg = own0 + tid; rg < own1; rg += NW * 32) cnt[rg] = 0u;   // for the next call
}

constexpr int kNW = 16;

template <int Q, int MC>
cudaError_t launch_q(const GemmArgs& a, const LaunchPlan& p) {
  const cudaError_t attr_err = once_per_device([] {
    cudaError_t attr_err = cudaSuccess;
    attr_err = cudaFuncSetAttribute(gemm_tiled_mb_kernel<Q, kNW, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kDynSmemMb);
    return attr_err;
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const long long U = (long long)S * RG;
  const size_t Npad = (size_t)RG * kTileRows;
  unsigned* sync = S > 1 ? reinterpret_cast<unsigned*>(a.workspace) : nullptr;
  float* partial = S > 1 ? reinterpret_cast<float*>(reinterpret_cast<char*>(a.workspace) + kPartOff) : nullptr;
  (void)Npad;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gemm_tiled_mb_kernel<Q, kNW, MC>, a.x, a.ldx,
                            reinterpret_cast<const uint4*>(a.planes), a.exps, a.M, a.N, S, RG, U, a.y, a.ldy,
                            partial, sync, pdl);
}

}  // namespace

LaunchPlan plan_gemm_tiled_mb(int M, int N, int K, int q, int sms) {
  (void)M; (void)q;
  const long long S = K / kTileK;
  const long long RG = (N + kTileRows - 1) / kTileRows;
  const long long U = S * RG;
  const long long grid = U < sms ? U : sms;
  return LaunchPlan{(int)grid, kNW * 32, kDynSmemMb, 2};
}

size_t workspace_gemm_tiled_mb(int M, int N, int K) {
  const size_t S = K / kTileK;
  if (S <= 1) return 0;
  const size_t RG = (N + kTileRows - 1) / kTileRows;
  return kPartOff + (size_t)M * S * RG * kTileRows * sizeof(float);
}

cudaError_t launch_gemm_tiled_mb(const GemmArgs& a, const LaunchPlan& p) {
  if (a.M == 2) {   // float2 entries: half the LDS traffic of the float4 variant
    switch (a.q) {
      case 1: return launch_q<1, 2>(a, p);
      case 2: return launch_q<2, 2>(a, p);
      case 3: return launch_q<3, 2>(a, p);
      case 4: return launch_q<4, 2>(a, p);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.q) {
    case 1: return launch_q<1, 4>(a, p);
    case 2: return launch_q<2, 4>(a, p);
    case 3: return launch_q<3, 4>(a, p);
    case 4: return launch_q<4, 4>(a, p);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace shiftadd
