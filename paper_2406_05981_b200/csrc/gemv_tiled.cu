// gemv_tiled.cu -- the batch-1 hot path on sm_100a (§8 a2-a6), device-tiled layout.
//
// y = sum_i alpha_i (.) (B_i x) with LUT queries.  Memory-bound: every
// packed key byte is read once from HBM (coalesced LDG.128, straight to registers) and
// becomes exactly one shared-memory LUT lookup and one fp32 add.
//
// Work decomposition.  A unit is one (256-k slice s, 16-row group rg) pair; units are
// numbered slice-major (u = s*RG + rg, the order of the tiled layout) and split into
// gridDim.x equal contiguous chunks (one chunk per CTA).  A CTA builds the LUT of each slice
// its chunk touches -- usually one, so the chip builds each slice's LUT only ~gridDim.x/S
// times -- and warps stride over the chunk's units.
//
// a2 LUT build: 32 groups x 256 keys fp32 per slice, built from two
//    4-activation half sums per key: T[key] = (A[lo&3] + B[lo>>2]) + (C[hi&3] + D[hi>>2]).
//    Word (key, col) sits at byte key*256 + col*4 of the LUT region; cols 0..31 / 32..63
//    alternate between consecutive slice segments, so building the next LUT needs no barrier
//    before it.
// a3 query: lane (r = lane/2, h = lane&1) holds the 16 key bytes of row r, chunk h of a
//    plane tile.  The tiled layout stores them rotated by r, so at unrolled step j every
//    lane reads its byte j and the 32 lanes look up 32 different LUTs (cols 16h+(j+r)&15):
//    bank-conflict free for any keys.  One PRMT forms key*256 + col*4, one LDS [R + UR_base],
//    one FADD per key byte.
// a4 shift: the chunk sum (16 lookups, inside one scale group since 128 | g) is scaled by
//    2^e with an exponent-field integer add.
// a5 reduce: lanes h=0,1 combine with one shuffle; split-K partials (one fp32 per slice and
//    row) go to the workspace; the last CTA to finish a row group (per-group arrival
//    counter) sums its S partials in fixed slice order and stores fp16 (RNE).  The final
//    sums are spread over all threads of that CTA with independent (unrolled) loads.  The
//    counters are reset by that CTA, leaving the counter region zeroed for the next call.
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace shiftadd {
namespace {

// a2: build the 32 LUTs of one 256-k slice into column half `hoff` (0 or 128 bytes).
template <int NW>
__device__ __forceinline__ void build_lut(const __half* __restrict__ xs, uint32_t lut, uint32_t hoff,
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
  const uint32_t col = lut + hoff + 4 * lane;
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
template <int Q, int MODE>
__device__ __forceinline__ float unit_dot(const uint4 (&w)[Q], const int (&e)[Q], uint32_t lut,
                                          const uint32_t (&cst)[16]) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float p0 = 0.f, p1 = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      // byte0 <- cst (col*4 + half), byte1 <- key byte (j&3) of word, bytes 2,3 <- 0
      const uint32_t off = __byte_perm(word, cst[j], 0x7604u | ((uint32_t)(j & 3) << 4));
      float v;
      if (MODE == 2) v = __uint_as_float(off);   // experiment: no LUT lookup
      else v = lds_f32(lut + off);
      if (j & 1) p1 += v; else p0 += v;
    }
    acc += shift_pow2(p0 + p1, e[i]);
  }
  return acc;
}

template <int Q>
__device__ __forceinline__ float unit_xor(const uint4 (&w)[Q], const int (&e)[Q]) {
  uint32_t a = 0;
#pragma unroll
  for (int i = 0; i < Q; ++i) a ^= w[i].x ^ w[i].y ^ w[i].z ^ w[i].w ^ (uint32_t)e[i];
  return __uint_as_float(a & 0x3fffffffu);
}

// MODE: 0 = product; 1 = no split-K finalize; 2 = no LUT lookups; 3 = loads only.
// Modes 1-3 are internal bottleneck experiments (SHIFTADD_EXP), never the product path.
template <int Q, int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 1)
gemv_tiled_kernel(const __half* __restrict__ x, const uint4* __restrict__ planes,
                  const int8_t* __restrict__ exps, int N, int S, int RG, long long U,
                  __half* __restrict__ y, float* __restrict__ partial, int* __restrict__ counters,
                  int pdl) {
  // dynamic smem: [LUT][fin_count][fin_list[NW*32]]; no static shared memory (kDynBase)
  int& fin_count = *reinterpret_cast<int*>(shiftadd_dyn_smem + kLutBytes);
  int* fin_list = reinterpret_cast<int*>(shiftadd_dyn_smem + kLutBytes + 16);
  if (threadIdx.x == 0) check_dyn_base();
  const uint32_t lut = kDynBase;
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
    if (MODE != 3) build_lut<NW>(x + (size_t)s * kTileK, lut, hoff, warp, lane);
    __syncthreads();
    uint32_t cst[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cst[j] = 4u * (uint32_t)(16 * h + ((j + r) & 15)) + hoff;
    const long long rg_base = (long long)s * RG;
    for (; uu < seg_end; uu += 2 * NW) {
      const long long un = uu + NW;
      if (un < seg_end) load_unit<Q>(planes, exps, un, lane, wb, eb);
      {
        float acc = (MODE == 3) ? unit_xor<Q>(wa, ea) : unit_dot<Q, MODE>(wa, ea, lut, cst);
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
        float acc = (MODE == 3) ? unit_xor<Q>(wb, eb) : unit_dot<Q, MODE>(wb, eb, lut, cst);
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
  if (S == 1 || MODE != 0) return;

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
      // (row group, row) items spread over all threads; 16 consecutive threads read the 16
      // consecutive rows of one group (64 B per slice).  Loads are issued 8 at a time,
      // independent of each other; the sum order is always s = 0, 1, ..., S-1.
      for (int item = tid; item < nf * kTileRows; item += NW * 32) {
        const int rg = fin_list[item >> 4];
        const int n = rg * kTileRows + (item & 15);
        const float* p = partial + n;
        float sum = 0.f;
        int s = 0;
        for (; s + 8 <= S; s += 8) {
          float v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = __ldcg(p + (size_t)(s + k) * Npad);
#pragma unroll
          for (int k = 0; k < 8; ++k) sum += v[k];
        }
        for (; s < S; ++s) sum += __ldcg(p + (size_t)s * Npad);
        if (n < N) y[n] = __float2half_rn(sum);
        if ((item & 15) == 0) counters[rg] = 0;
      }
    }
    __syncthreads();
  }
}

struct Cfg {
  int nw;          // warps per CTA
  int per_sm;      // CTAs per SM
  int mode;        // experiment mode (0 = product)
};

Cfg config_from_env() {
  Cfg c{8, 1, 0};
  if (const char* e = std::getenv("SHIFTADD_EXP")) c.mode = std::atoi(e);
  if (const char* e = std::getenv("SHIFTADD_NW")) c.nw = std::atoi(e) == 16 ? 16 : 8;
  if (const char* e = std::getenv("SHIFTADD_PER_SM")) c.per_sm = std::atoi(e) < 1 ? 1 : std::atoi(e);
  if (c.mode < 0 || c.mode > 3) c.mode = 0;
  return c;
}

const Cfg& cfg() {
  static Cfg c = config_from_env();
  return c;
}

constexpr int kDynSmem = kLutBytes + 16 + 16 * 32 * 4;  // 64 KB LUT + finalize list

template <int Q, int NW, int MODE>
cudaError_t launch_qnm(const GemmArgs& a, const LaunchPlan& p) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemv_tiled_kernel<Q, NW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kDynSmem);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const long long U = (long long)S * RG;
  int* counters = S > 1 ? reinterpret_cast<int*>(a.workspace) : nullptr;
  float* partial = S > 1 ? reinterpret_cast<float*>(reinterpret_cast<char*>(a.workspace) + kCounterBytes) : nullptr;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;

  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(p.grid);
  c.blockDim = dim3(p.threads);
  c.dynamicSmemBytes = p.smem;
  c.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = attr;
  c.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&c, gemv_tiled_kernel<Q, NW, MODE>, a.x, reinterpret_cast<const uint4*>(a.planes),
                            a.exps, a.N, S, RG, U, a.y, partial, counters, pdl);
}

template <int Q, int NW>
cudaError_t launch_qn(const GemmArgs& a, const LaunchPlan& p) {
  switch (cfg().mode) {
    case 1: return launch_qnm<Q, NW, 1>(a, p);
    case 2: return launch_qnm<Q, NW, 2>(a, p);
    case 3: return launch_qnm<Q, NW, 3>(a, p);
    default: return launch_qnm<Q, NW, 0>(a, p);
  }
}

template <int Q>
cudaError_t launch_q(const GemmArgs& a, const LaunchPlan& p) {
  return p.threads == 512 ? launch_qn<Q, 16>(a, p) : launch_qn<Q, 8>(a, p);
}

}  // namespace

LaunchPlan plan_gemv_tiled(int N, int K, int q, int sms) {
  (void)q;
  const long long S = K / kTileK;
  const long long RG = (N + kTileRows - 1) / kTileRows;
  const long long U = S * RG;
  const long long want = (long long)sms * cfg().per_sm;
  const long long grid = U < want ? U : want;
  return LaunchPlan{(int)grid, cfg().nw * 32, kDynSmem, 1};
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
