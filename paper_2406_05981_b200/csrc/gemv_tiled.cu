// gemv_tiled.cu -- the batch-1 hot path on sm_100a (§8 a2-a6), device-tiled layout.
//
// y = sum_i alpha_i (.) (B_i x) with LUT queries.  Memory-bound: every
// packed key byte is read once from HBM (coalesced LDG.128, straight to registers) and
// becomes exactly one shared-memory LUT lookup and one fp32 add.
//
// Work decomposition.  A unit is one (256-k slice s, 16-row group rg) pair; units are
// numbered slice-major (u = s*RG + rg, the order of the tiled layout) and split into
// gridDim.x equal contiguous chunks (one chunk per CTA, ~1 CTA per SM).  A CTA builds the
// LUT of each slice its chunk touches -- usually one, so the chip builds each slice's LUT
// only ~gridDim.x/S times -- and warps stride over the chunk's units.
//
// a2 LUT build: 32 groups x 256 keys fp32 per slice, built from two
//    4-activation half sums per key: T[key] = (A[lo&3] + B[lo>>2]) + (C[hi&3] + D[hi>>2]).
//    Word (key, col) sits at byte key*256 + col*4; cols 0..31 / 32..63 alternate between
//    consecutive slice segments, so building the next LUT needs no barrier before it.
// a3 query: lane (r = lane/2, h = lane&1) holds the 16 key bytes of row r, chunk h of a
//    plane tile.  The tiled layout stores them rotated by r, so at unrolled step j every
//    lane reads its byte j and the 32 lanes look up 32 different LUTs (cols 16h+(j+r)&15):
//    bank-conflict free for any keys.  One PRMT assembles key*256 + col*4, one LDS, one FADD.
// a4 shift: the chunk sum (16 lookups, inside one scale group since 128 | g) is scaled by
//    2^e with an exponent-field integer add.
// a5 reduce: lanes h=0,1 combine with one shuffle; split-K partials (one fp32 per slice and
//    row) go to the workspace; the last CTA to finish a row group (per-group arrival
//    counter) sums its S partials in fixed slice order and stores fp16 (RNE).  The counters
//    are reset by that CTA, leaving the workspace zeroed for the next call.
#include <mutex>

#include "common.cuh"

namespace shiftadd {
namespace {

// a2: build the 32 LUTs of one 256-k slice into column half `hoff` (0 or 128 bytes).
template <int NW>
__device__ __forceinline__ void build_lut(const __half* __restrict__ xs, uint32_t hoff,
                                          int warp, int lane) {
  const uint4 xv = *reinterpret_cast<const uint4*>(xs + 8 * lane);  // activations 8*lane .. +7
  const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
  const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
  const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
  const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
  // key bit b <-> activation b: +x_b if set, -x_b if clear.
  const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
  const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
  float L[16];
#pragma unroll
  for (int lo = 0; lo < 16; ++lo) L[lo] = A[lo & 3] + B[lo >> 2];
  const uint32_t col = kLutBase + hoff + 4 * lane;
#pragma unroll
  for (int hh = 0; hh < 16 / NW; ++hh) {
    const int hi = warp + NW * hh;
    // hi is warp-dependent: select the signs instead of indexing (keeps it in registers)
    const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                    ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), L[lo] + H);
  }
}

// a3 + a4 for one unit: sum over planes of 2^e * (16 LUT lookups).
template <int Q>
__device__ __forceinline__ float unit_dot(const uint4 (&w)[Q], const int (&e)[Q], const uint32_t (&cst)[16]) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float p0 = 0.f, p1 = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      // byte0 <- cst (col*4 + half), byte1 <- key byte (j&3) of word, bytes 2,3 <- cst (0x0001)
      const uint32_t addr = __byte_perm(word, cst[j], 0x7604u | ((uint32_t)(j & 3) << 4));
      const float v = lds_f32(addr);
      if (j & 1) p1 += v; else p0 += v;
    }
    acc += shift_pow2(p0 + p1, e[i]);
  }
  return acc;
}

template <int Q, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
gemv_tiled_kernel(const __half* __restrict__ x, const uint4* __restrict__ planes,
                  const int8_t* __restrict__ exps, int N, int S, int RG, long long U,
                  __half* __restrict__ y, float* __restrict__ partial, int* __restrict__ counters,
                  int pdl) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ int fin_list[NW * 32];
  __shared__ int fin_count;
  check_lut_window(dyn_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 1, h = lane & 1;
  const long long G = gridDim.x;
  const long long u0 = ((long long)blockIdx.x * U) / G;
  const long long u1 = ((long long)(blockIdx.x + 1) * U) / G;
  const int Npad = RG * kTileRows;

  uint4 wa[Q], wb[Q];
  int ea[Q], eb[Q];
  long long u = u0;
  int seg = 0;
  bool waited = false;
  while (u < u1) {
    const int s = (int)(u / RG);
    const long long seg_end = min(u1, (long long)(s + 1) * RG);
    long long uu = u + warp;
    if (uu < seg_end) load_unit<Q>(planes, exps, uu, lane, wa, ea);  // weights never depend on
    if (!waited) {                                                    // the upstream kernel
      if (pdl) pdl_wait();
      waited = true;
    }
    const uint32_t hoff = (seg & 1) ? 128u : 0u;
    build_lut<NW>(x + (size_t)s * kTileK, hoff, warp, lane);
    __syncthreads();
    uint32_t cst[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cst[j] = kLutBase + 4u * (uint32_t)(16 * h + ((j + r) & 15)) + hoff;
    const long long rg_base = (long long)s * RG;
    for (; uu < seg_end; uu += 2 * NW) {
      const long long un = uu + NW;
      if (un < seg_end) load_unit<Q>(planes, exps, un, lane, wb, eb);
      {
        float acc = unit_dot<Q>(wa, ea, cst);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        const int n = (int)(uu - rg_base) * kTileRows + r;
        if (h == 0) {
          if (S == 1) { if (n < N) y[n] = __float2half_rn(acc); }
          else partial[(size_t)s * Npad + n] = acc;
        }
      }
      if (un >= seg_end) break;
      const long long unn = un + NW;
      if (unn < seg_end) load_unit<Q>(planes, exps, unn, lane, wa, ea);
      {
        float acc = unit_dot<Q>(wb, eb, cst);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        const int n = (int)(un - rg_base) * kTileRows + r;
        if (h == 0) {
          if (S == 1) { if (n < N) y[n] = __float2half_rn(acc); }
          else partial[(size_t)s * Npad + n] = acc;
        }
      }
    }
    u = seg_end;
    ++seg;
  }
  if (pdl) pdl_launch_dependents();
  if (S == 1) return;

  // a5: deterministic split-K reduction by the last-arriving CTA of each row group.
  __threadfence();
  __syncthreads();
  for (long long ub = u0; ub < u1; ub += NW * 32) {
    if (tid == 0) fin_count = 0;
    __syncthreads();
    const long long uq = ub + tid;
    if (uq < u1) {
      const int rg = (int)(uq % RG);
      if (atomicAdd(&counters[rg], 1) == S - 1) fin_list[atomicAdd(&fin_count, 1)] = rg;
    }
    __syncthreads();
    const int nf = fin_count;
    if (nf > 0) {
      __threadfence();
      for (int f = warp; f < nf; f += NW) {
        const int rg = fin_list[f];
        const int rr = lane & 15, part = lane >> 4;
        const int n = rg * kTileRows + rr;
        float sum = 0.f;
        for (int s = part; s < S; s += 2) sum += __ldcg(partial + (size_t)s * Npad + n);
        sum += __shfl_xor_sync(0xffffffffu, sum, 16);
        if (part == 0 && n < N) y[n] = __float2half_rn(sum);
        if (lane == 0) counters[rg] = 0;
      }
    }
    __syncthreads();
  }
}

constexpr int kNW = 16;
constexpr int kDynSmem = (int)kLutBase + kLutBytes;  // covers [kLutBase, kLutBase + 64 KB)

template <int Q>
cudaError_t launch_q(const GemmArgs& a, const LaunchPlan& p) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemv_tiled_kernel<Q, kNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kDynSmem);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const long long U = (long long)S * RG;
  const size_t Npad = (size_t)RG * kTileRows;
  int* counters = S > 1 ? reinterpret_cast<int*>(a.workspace) : nullptr;
  float* partial = S > 1 ? reinterpret_cast<float*>(reinterpret_cast<char*>(a.workspace) + kCounterBytes) : nullptr;
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
  return cudaLaunchKernelEx(&cfg, gemv_tiled_kernel<Q, kNW>, a.x, reinterpret_cast<const uint4*>(a.planes),
                            a.exps, a.N, S, RG, U, a.y, partial, counters, pdl);
}

}  // namespace

LaunchPlan plan_gemv_tiled(int N, int K, int q, int sms) {
  (void)q;
  const long long S = K / kTileK;
  const long long RG = (N + kTileRows - 1) / kTileRows;
  const long long U = S * RG;
  const long long grid = U < sms ? U : sms;
  return LaunchPlan{(int)grid, kNW * 32, kDynSmem, 1};
}

size_t workspace_gemv_tiled(int N, int K) {
  const size_t S = K / kTileK;
  if (S <= 1) return 0;
  const size_t RG = (N + kTileRows - 1) / kTileRows;
  return kCounterBytes + S * RG * kTileRows * sizeof(float);
}

cudaError_t launch_gemv_tiled(const GemmArgs& a, const LaunchPlan& p) {
  switch (a.q) {
    case 1: return launch_q<1>(a, p);
    case 2: return launch_q<2>(a, p);
    case 3: return launch_q<3>(a, p);
    case 4: return launch_q<4>(a, p);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace shiftadd
