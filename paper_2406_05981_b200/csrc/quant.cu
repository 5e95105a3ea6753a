// quant.cu -- NEXT-f4: Alg. 1 alternating multi-bit BCQ on the device (the step before a1).
//
// greedy initialisation (Eq. 1, Line 4), then T cycles of least-squares
// scale refit alpha = (B^T B)^-1 B^T w (Line 6) and binary-search code refit (Line 7); with
// SHIFTADD_BCQ_POT every alpha is projected to sign * 2^round(log2|alpha|) after each LS
// refit ("during the alternating optimization cycles, we further quantize all scaling
// factors to powers of two").  One CTA per scale group (g consecutive k
// of one output row), all arithmetic in fp64: an offline, one-time step, and fp64 makes the
// integer decisions (signs, codes) those of the fp64 oracle except at ties within ~1e-16.
//
// Codes are never stored: at any point they are a pure function of w_j and the alphas that
// produced them -- greedy: b_i = sign(r_{i-1}) with r_i = r_{i-1} - alpha_i b_i; BS: the
// level sum_i c_i alpha_i nearest to w_j (ties: smaller |level|, then the negative level,
// DESIGN.md R23) -- so every pass re-derives them from w in registers.
#include "common.cuh"

namespace shiftadd {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Block-wide sums of NV doubles (fixed order: warp butterflies, then warp 0 over warps).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) red[k * 32 + warp] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[k * 32 + i];
    v[k] = s;
  }
  __syncthreads();
}

// sign(a) 2^round(log2|a|) in fp64 by the exact mantissa rule (0x6A09E667F3BCD is the first
// 52-bit mantissa with (1.m)^2 >= 2; sqrt(2) is irrational, so there are no ties).
__device__ __forceinline__ double pot_round64(double a) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(a);
  const unsigned long long mag = u & 0x7fffffffffffffffull;
  if (mag == 0ull) return 0.0;
  int e = (int)(mag >> 52) - 1023;
  if ((mag & 0xfffffffffffffull) >= 0x6A09E667F3BCDull) ++e;
  const double p = ldexp(1.0, e);
  return (u >> 63) ? -p : p;
}

template <int Q>
__device__ __forceinline__ void greedy_codes(double w, const double (&al)[Q], int upto, double (&b)[Q]) {
  double r = w;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    if (i < upto) {
      b[i] = r >= 0.0 ? 1.0 : -1.0;
      r -= al[i] * b[i];
    }
  }
}

template <int Q>
__device__ __forceinline__ void bs_codes(double w, const double (&al)[Q], double (&b)[Q]) {
  double best_d = 0.0, best_m = 0.0, best_l = 0.0;
  int best = -1;
#pragma unroll
  for (int c = 0; c < (1 << Q); ++c) {
    double lv = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) lv += ((c >> i) & 1) ? al[i] : -al[i];
    const double d = fabs(w - lv), m = fabs(lv);
    const bool better = best < 0 || d < best_d || (d == best_d && (m < best_m || (m == best_m && lv < best_l)));
    if (better) {
      best = c;
      best_d = d;
      best_m = m;
      best_l = lv;
    }
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) b[i] = ((best >> i) & 1) ? 1.0 : -1.0;
}

// (G + reg I) x = rhs, Q <= 4, Gaussian elimination with partial pivoting (one thread).
template <int Q>
__device__ void solve_small(double (&G)[Q][Q], double (&rhs)[Q], double (&x)[Q]) {
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    int piv = c;
    for (int r = c + 1; r < Q; ++r)
      if (fabs(G[r][c]) > fabs(G[piv][c])) piv = r;
    if (piv != c) {
      for (int k = 0; k < Q; ++k) {
        const double t = G[c][k];
        G[c][k] = G[piv][k];
        G[piv][k] = t;
      }
      const double t = rhs[c];
      rhs[c] = rhs[piv];
      rhs[piv] = t;
    }
    for (int r = c + 1; r < Q; ++r) {
      const double f = G[r][c] / G[c][c];
      for (int k = c; k < Q; ++k) G[r][k] -= f * G[c][k];
      rhs[r] -= f * rhs[c];
    }
  }
  for (int r = Q - 1; r >= 0; --r) {
    double s = rhs[r];
    for (int k = r + 1; k < Q; ++k) s -= G[r][k] * x[k];
    x[r] = s / G[r][r];
  }
}

template <int Q>
__global__ void __launch_bounds__(256) bcq_quantize_kernel(const float* __restrict__ w, int N, int K, int g, int T,
                                                           int pot, int8_t* __restrict__ signs,
                                                           float* __restrict__ alpha) {
  __shared__ double red[(Q + Q * (Q + 1) / 2) * 32];
  __shared__ double al_s[Q];
  const int G = K / g;
  const long long grp = blockIdx.x;
  const int n = (int)(grp / G), gi = (int)(grp - (long long)n * G);
  const float* wg = w + (size_t)n * K + (size_t)gi * g;
  double al[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) al[i] = 0.0;

  // Line 4 / Eq. 1: alpha_i = r_{i-1}^T sign(r_{i-1}) / g = mean |r_{i-1}|
  for (int i = 0; i < Q; ++i) {
    double v[1] = {0.0};
    for (int j = threadIdx.x; j < g; j += blockDim.x) {
      double r = (double)__ldg(wg + j);
      for (int k = 0; k < i; ++k) r -= al[k] * (r >= 0.0 ? 1.0 : -1.0);
      v[0] += fabs(r);
    }
    block_sum<1>(v, red);
    al[i] = v[0] / (double)g;
  }
  bool greedy = true;

  // Lines 5-7: T x (LS, [PoT], BS).  The codes used by LS are those of the previous stage.
  for (int t = 0; t < T; ++t) {
    constexpr int NG = Q * (Q + 1) / 2;
    double v[Q + NG];
#pragma unroll
    for (int k = 0; k < Q + NG; ++k) v[k] = 0.0;
    for (int j = threadIdx.x; j < g; j += blockDim.x) {
      const double wj = (double)__ldg(wg + j);
      double b[Q];
      if (greedy) greedy_codes<Q>(wj, al, Q, b);
      else bs_codes<Q>(wj, al, b);
      int idx = Q;
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        v[i] += b[i] * wj;
#pragma unroll
        for (int k = i; k < Q; ++k) v[idx++] += b[i] * b[k];
      }
    }
    block_sum<Q + NG>(v, red);
    if (threadIdx.x == 0) {
      double Gm[Q][Q], rhs[Q], x[Q];
      int idx = Q;
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        rhs[i] = v[i];
#pragma unroll
        for (int k = i; k < Q; ++k) {
          Gm[i][k] = v[idx];
          Gm[k][i] = v[idx];
          ++idx;
        }
        Gm[i][i] += 1e-8 * (double)g;   // DESIGN.md R22
      }
      solve_small<Q>(Gm, rhs, x);
#pragma unroll
      for (int i = 0; i < Q; ++i) al_s[i] = pot ? pot_round64(x[i]) : x[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Q; ++i) al[i] = al_s[i];
    __syncthreads();
    greedy = false;
  }

  // outputs: the final codes (greedy or BS of the final alphas) and the alphas
  for (int j = threadIdx.x; j < g; j += blockDim.x) {
    const double wj = (double)__ldg(wg + j);
    double b[Q];
    if (greedy) greedy_codes<Q>(wj, al, Q, b);
    else bs_codes<Q>(wj, al, b);
#pragma unroll
    for (int i = 0; i < Q; ++i) signs[((size_t)i * N + n) * K + (size_t)gi * g + j] = (int8_t)(b[i] > 0.0 ? 1 : -1);
  }
  if (threadIdx.x < Q) alpha[((size_t)threadIdx.x * N + n) * G + gi] = (float)al[threadIdx.x];
}

}  // namespace

cudaError_t launch_bcq_quantize(const float* w, int N, int K, int q, int g, int T, int pot, int8_t* signs,
                                float* alpha, cudaStream_t stream) {
  const long long groups = (long long)N * (K / g);
  if (groups > 0x7fffffffLL) return cudaErrorInvalidValue;
  int threads = g < 256 ? ((g + 31) / 32) * 32 : 256;
  const dim3 grid((unsigned)groups);
  switch (q) {
    case 1: bcq_quantize_kernel<1><<<grid, threads, 0, stream>>>(w, N, K, g, T, pot, signs, alpha); break;
    case 2: bcq_quantize_kernel<2><<<grid, threads, 0, stream>>>(w, N, K, g, T, pot, signs, alpha); break;
    case 3: bcq_quantize_kernel<3><<<grid, threads, 0, stream>>>(w, N, K, g, T, pot, signs, alpha); break;
    case 4: bcq_quantize_kernel<4><<<grid, threads, 0, stream>>>(w, N, K, g, T, pot, signs, alpha); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace shiftadd
