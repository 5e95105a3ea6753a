// pack.cu -- §8 a1: bit-plane packing and PoT exponent encoding on the device.
//
// PAPER.md:120 (BCQ planes b_i in {-1,+1}), Eq. 2 PAPER.md:174-177 (alpha -> sign * 2^P,
// P = round(log2|alpha|)), PAPER.md:185 (8 grouped binary weights form an 8-bit key).
// Integer/bit work, bit-exact against the oracle.  One-time per layer, HBM-bound.
#include "common.cuh"

namespace shiftadd {
namespace {

// P = round(log2 a) for a = |alpha| as an exact integer rule on the fp32 bits: log2 a lies in
// [E, E+1) for biased exponent field E+127, and rounds up iff the mantissa m (as 1.m) has
// (1.m)^2 >= 2, i.e. 1.m >= sqrt(2).  0x3504F4 is the first 23-bit mantissa with
// 1.m > sqrt(2) (1.m for 0x3504F3 is 1.41421354 < sqrt(2) < 1.41421366 for 0x3504F4);
// sqrt(2) itself is irrational, so there are no ties.  Subnormal a -> below 2^-126, clamps.
__device__ __forceinline__ int pot_exponent(float alpha, int* clamped, int* invalid) {
  const uint32_t u = __float_as_uint(alpha) & 0x7fffffffu;
  *clamped = 0;
  *invalid = 0;
  if (u >= 0x7f800000u) {  // Inf / NaN
    *invalid = 1;
    return SHIFTADD_EXP_ZERO;
  }
  if (u == 0u) return SHIFTADD_EXP_ZERO;  // alpha == +-0
  const int ef = (int)(u >> 23);
  int e = (ef == 0) ? -127 : ef - 127 + ((u & 0x7fffffu) >= 0x3504F4u ? 1 : 0);
  if (e < SHIFTADD_EXP_MIN) {
    e = SHIFTADD_EXP_MIN;
    *clamped = 1;
  } else if (e > SHIFTADD_EXP_MAX) {
    e = SHIFTADD_EXP_MAX;
    *clamped = 1;
  }
  return e;
}

__device__ __forceinline__ void warp_count(int v, int32_t* dst) {
  const unsigned lanes = __ballot_sync(0xffffffffu, v != 0);
  if (dst != nullptr && lanes != 0u && (threadIdx.x & 31) == (__ffs(lanes) - 1))
    atomicAdd(dst, __popc(lanes));
}

// Exponents of every canonical scale group (i, n, G); counts clamps / invalid scales once
// per group; writes the canonical exps array when `exps` is non-null.
__global__ void pack_exps_kernel(const float* __restrict__ alpha, long long groups,
                                 int8_t* __restrict__ exps, int32_t* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < groups; base += stride) {
    const long long idx = base + threadIdx.x;
    int clamped = 0, invalid = 0, e = 0;
    if (idx < groups) {
      e = pot_exponent(__ldg(alpha + idx), &clamped, &invalid);
      if (exps) exps[idx] = (int8_t)e;
    }
    if (counts) {
      warp_count(clamped, counts);
      warp_count(invalid, counts + 1);
    }
  }
}

// Canonical (i, n, key byte kb) of an output byte in either layout; false for a padded row.
__device__ __forceinline__ bool byte_source(int layout, long long o, int q, int N, int KB, int RG,
                                            int* i, int* n, int* kb) {
  if (layout == SHIFTADD_LAYOUT_CANONICAL) {
    *kb = (int)(o % KB);
    const long long rest = o / KB;
    *n = (int)(rest % N);
    *i = (int)(rest / N);
    return true;
  }
  const int j = (int)(o & 15);
  const int h = (int)((o >> 4) & 1);
  const int r = (int)((o >> 5) & 15);
  const long long t = o >> 9;  // tile index ((s*RG + rg)*q + i)
  *i = (int)(t % q);
  const long long sr = t / q;
  const int rg = (int)(sr % RG);
  const int s = (int)(sr / RG);
  *n = rg * kTileRows + r;
  *kb = s * (kTileK / 8) + h * 16 + ((j + r) & 15);
  return *n < N;
}

// One thread per output key byte: 8 consecutive signs -> 8 bits (bit b <-> k = 8kb + b,
// 1 <-> +1 after the sign fold of the byte's scale group).
// colwise (NEXT-f1): alpha is alpha_col [q][K] and each bit b flips with the sign of its own
// column's scale alpha_col[i][8kb + b] (the column-wise sign fold, R17).
__global__ void pack_planes_kernel(const int8_t* __restrict__ signs, const float* __restrict__ alpha,
                                   int q, int N, int K, int g, int layout, long long nbytes, int RG,
                                   uint8_t* __restrict__ planes, int32_t* counts, int colwise) {
  const int KB = K >> 3;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < nbytes; base += stride) {
    const long long o = base + threadIdx.x;
    int bad = 0;
    if (o < nbytes) {
      int i, n, kb;
      uint8_t out = 0;
      if (byte_source(layout, o, q, N, KB, RG, &i, &n, &kb)) {
        const long long row = (long long)i * N + n;
        const uint2 sv = __ldg(reinterpret_cast<const uint2*>(signs + row * K) + kb);
        uint32_t flip;
        if (colwise == 2) {   // NEXT-f1 block-wise: alpha_bw [q][8][K/8], block b = n / (N/8)
          const float a = __ldg(alpha + ((long long)i * 8 + n / (N / 8)) * KB + kb);
          flip = (a < 0.f) ? 0xffu : 0u;
        } else if (colwise) {
          const float* ac = alpha + (long long)i * K + kb * 8;
          flip = 0u;
#pragma unroll
          for (int b = 0; b < 8; ++b) flip |= (__ldg(ac + b) < 0.f ? 1u : 0u) << b;
        } else {
          const float a = __ldg(alpha + row * (K / g) + (kb * 8) / g);
          flip = (a < 0.f) ? 0xffu : 0u;
        }
        uint32_t bits = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const uint32_t w = (b < 4) ? sv.x : sv.y;
          const int s = (int)(int8_t)((w >> (8 * (b & 3))) & 0xffu);
          bad |= (s != 1 && s != -1);
          bits |= (s == 1 ? 1u : 0u) << b;
        }
        out = (uint8_t)(bits ^ flip);
      }
      planes[o] = out;
    }
    warp_count(bad, counts ? counts + 1 : nullptr);
  }
}

// Tiled exponents: one per (tile, r, h) = the exponent of the scale group holding the
// 128-k chunk h of row r (the chunk lies inside one group because 128 | g).
__global__ void pack_exps_tiled_kernel(const float* __restrict__ alpha, int q, int N, int K, int g,
                                       int RG, long long count, int8_t* __restrict__ exps) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < count; o += stride) {
    const int h = (int)(o & 1);
    const int r = (int)((o >> 1) & 15);
    const long long t = o >> 5;
    const int i = (int)(t % q);
    const long long sr = t / q;
    const int rg = (int)(sr % RG);
    const int s = (int)(sr / RG);
    const int n = rg * kTileRows + r;
    int e = SHIFTADD_EXP_ZERO;
    if (n < N) {
      int c, v;
      e = pot_exponent(__ldg(alpha + ((long long)i * N + n) * (K / g) + (s * kTileK + h * 128) / g), &c, &v);
    }
    exps[o] = (int8_t)e;
  }
}

// NEXT-f2: the second additive-PoT term code of one scale (R19): term 1 is the
// pot_exponent above (sign folded into the bits); r1 = alpha - s1 2^P1 is exact in fp32
// (Sterbenz: |alpha| / 2^P1 in [2^-0.5, 2^0.5)); c2 = s1 s2 (P1 - P2) with P2 the unclamped
// round(log2|r1|); 0 if alpha is 0/Inf/NaN, P1 was clamped, r1 == 0, P2 < EXP_MIN or
// P1 - P2 > 127.
__device__ __forceinline__ int apot2_code(float alpha) {
  int clamped, invalid;
  const int e1 = pot_exponent(alpha, &clamped, &invalid);
  if (invalid || clamped || e1 == SHIFTADD_EXP_ZERO) return 0;
  const float t1 = __int_as_float((e1 + 127) << 23);
  const float r1 = alpha < 0.f ? alpha + t1 : alpha - t1;
  const uint32_t u = __float_as_uint(r1) & 0x7fffffffu;
  if (u == 0u) return 0;
  const int ef = (int)(u >> 23);
  if (ef == 0) return 0;                                    // subnormal: P2 < -126
  const int e2 = ef - 127 + ((u & 0x7fffffu) >= 0x3504F4u ? 1 : 0);
  const int d = e1 - e2;
  if (e2 < SHIFTADD_EXP_MIN || d > 127) return 0;
  const bool neg = (alpha < 0.f) != (r1 < 0.f);
  return neg ? -d : d;
}

__global__ void pack_apot2_kernel(const float* __restrict__ alpha, int q, int N, int K, int g, int layout, int RG,
                                  long long count, int8_t* __restrict__ exps2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < count; o += stride) {
    long long src;
    if (layout == SHIFTADD_LAYOUT_CANONICAL) {
      src = o;
    } else {   // tiled: same permutation as pack_exps_tiled_kernel
      const int h = (int)(o & 1);
      const int r = (int)((o >> 1) & 15);
      const long long t = o >> 5;
      const int i = (int)(t % q);
      const long long sr = t / q;
      const int rg = (int)(sr % RG);
      const int s = (int)(sr / RG);
      const int n = rg * kTileRows + r;
      src = n < N ? ((long long)i * N + n) * (K / g) + (s * kTileK + h * 128) / g : -1;
    }
    exps2[o] = (int8_t)(src < 0 ? 0 : apot2_code(__ldg(alpha + src)));
  }
}

int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  if (b > 148LL * 32) b = 148LL * 32;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_pack(const int8_t* signs, const float* alpha, int q, int N, int K, int g,
                        int layout, uint8_t* planes, int8_t* exps, int32_t* counts,
                        cudaStream_t stream) {
  const int threads = 256;
  const long long groups = (long long)q * N * (K / g);
  const bool canon = layout == SHIFTADD_LAYOUT_CANONICAL;
  const int RG = (N + kTileRows - 1) / kTileRows;
  pack_exps_kernel<<<grid_for(groups, threads), threads, 0, stream>>>(alpha, groups,
                                                                       canon ? exps : nullptr, counts);
  const long long nbytes = canon ? (long long)q * N * (K / 8)
                                 : (long long)(K / kTileK) * RG * q * kTileBytes;
  pack_planes_kernel<<<grid_for(nbytes, threads), threads, 0, stream>>>(signs, alpha, q, N, K, g, layout,
                                                                         nbytes, RG, planes, counts, 0);
  if (!canon) {
    const long long ne = (long long)(K / kTileK) * RG * q * kTileExps;
    pack_exps_tiled_kernel<<<grid_for(ne, threads), threads, 0, stream>>>(alpha, q, N, K, g, RG, ne, exps);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_apot2(const float* alpha, int q, int N, int K, int g, int layout, int8_t* exps2,
                              cudaStream_t stream) {
  const int threads = 256;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const long long count = layout == SHIFTADD_LAYOUT_CANONICAL ? (long long)q * N * (K / g)
                                                              : (long long)(K / kTileK) * RG * q * kTileExps;
  pack_apot2_kernel<<<grid_for(count, threads), threads, 0, stream>>>(alpha, q, N, K, g, layout, RG, count, exps2);
  return cudaGetLastError();
}

// NEXT-f1 column-wise pack: exps_col [q][K] (no layout permutation: the kernels read it by
// column when they pre-shift x) and planes in either layout with the per-column sign fold.
cudaError_t launch_pack_colwise(const int8_t* signs, const float* alpha_col, int q, int N, int K,
                                int layout, uint8_t* planes, int8_t* exps_col, int32_t* counts,
                                cudaStream_t stream) {
  const int threads = 256;
  const long long groups = (long long)q * K;
  const bool canon = layout == SHIFTADD_LAYOUT_CANONICAL;
  const int RG = (N + kTileRows - 1) / kTileRows;
  pack_exps_kernel<<<grid_for(groups, threads), threads, 0, stream>>>(alpha_col, groups, exps_col, counts);
  const long long nbytes = canon ? (long long)q * N * (K / 8)
                                 : (long long)(K / kTileK) * RG * q * kTileBytes;
  pack_planes_kernel<<<grid_for(nbytes, threads), threads, 0, stream>>>(signs, alpha_col, q, N, K, 8, layout,
                                                                         nbytes, RG, planes, counts, 1);
  return cudaGetLastError();
}

cudaError_t launch_pack_blockwise(const int8_t* signs, const float* alpha_bw, int q, int N, int K, int layout,
                                  uint8_t* planes, int8_t* exps_bw, int32_t* counts, cudaStream_t stream) {
  const int threads = 256;
  const long long groups = (long long)q * 8 * (K / 8);
  const bool canon = layout == SHIFTADD_LAYOUT_CANONICAL;
  const int RG = (N + kTileRows - 1) / kTileRows;
  pack_exps_kernel<<<grid_for(groups, threads), threads, 0, stream>>>(alpha_bw, groups, exps_bw, counts);
  const long long nbytes = canon ? (long long)q * N * (K / 8)
                                 : (long long)(K / kTileK) * RG * q * kTileBytes;
  pack_planes_kernel<<<grid_for(nbytes, threads), threads, 0, stream>>>(signs, alpha_bw, q, N, K, 8, layout,
                                                                         nbytes, RG, planes, counts, 2);
  return cudaGetLastError();
}

}  // namespace shiftadd
