// gemm_generic.cu -- canonical-layout LUT-GEMM for any supported shape (§8 a2-a5, a7).
//
// Plain and correct rather than fast: it accepts the north_star layout
// planes[q][N][K/8] / exps[q][N][K/g] for every K % 8 == 0, g % 8 == 0, M <= 16.
// One CTA owns 64 output rows and walks all of K in 256-k slices.  Per slice and batch
// row it builds the 32 LUTs of the slice in shared memory (a2), then
// each warp takes rows; lane t queries LUT t with key byte planes[i][n][32s + t] (a3,
// "every eight grouped binary weights form an 8-bit key") -- 32 lanes read
// 32 different LUT columns, so the lookups are bank-conflict free by construction --
// shifts the queried partial sum by its group exponent (a4), and reduces
// the warp with a fixed shuffle tree (a5).  Results accumulate in shared memory and are
// stored as fp16 (RNE) at the end: deterministic, no workspace.  With exps2 (NEXT-f2) each
// shifted partial sum also adds its second additive-PoT term (shift_apot2).
#include "common.cuh"

namespace shiftadd {
namespace {

constexpr int kRows = 64;     // output rows per CTA
constexpr int kWarps = 8;     // 256 threads
constexpr int kMaxM = 16;

__global__ void __launch_bounds__(kWarps * 32)
gemm_generic_kernel(const __half* __restrict__ x, int ldx, const uint8_t* __restrict__ planes,
                    const int8_t* __restrict__ exps, const int8_t* __restrict__ exps2, int M, int N,
                    int K, int q, int g, __half* __restrict__ y, int ldy) {
  __shared__ float lut[256 * 32];          // word (key, t) = key*32 + t
  __shared__ float acc[kMaxM * kRows];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * kRows;
  const int rows = min(kRows, N - n0);
  const int KB = K >> 3;
  const int KG = K / g;
  for (int idx = tid; idx < kMaxM * kRows; idx += blockDim.x) acc[idx] = 0.f;

  for (int s0 = 0; s0 < KB; s0 += 32) {           // slice of 32 key bytes = 256 k
    const int ng = min(32, KB - s0);
    for (int m = 0; m < M; ++m) {
      __syncthreads();                            // previous LUT fully consumed
      // a2: thread (warp w, lane t) builds T_t[key] for hi nibbles {w, w+8}, all lo.
      if (lane < ng) {
        const __half* xs = x + (size_t)m * ldx + 8 * (s0 + lane);
        float xv[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) xv[b] = __half2float(xs[b]);
        float L[16];
#pragma unroll
        for (int lo = 0; lo < 16; ++lo)
          L[lo] = ((lo & 1 ? xv[0] : -xv[0]) + (lo & 2 ? xv[1] : -xv[1])) +
                  ((lo & 4 ? xv[2] : -xv[2]) + (lo & 8 ? xv[3] : -xv[3]));
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int hi = warp + 8 * hh;
          const float H = ((hi & 1 ? xv[4] : -xv[4]) + (hi & 2 ? xv[5] : -xv[5])) +
                          ((hi & 4 ? xv[6] : -xv[6]) + (hi & 8 ? xv[7] : -xv[7]));
#pragma unroll
          for (int lo = 0; lo < 16; ++lo) lut[(hi * 16 + lo) * 32 + lane] = L[lo] + H;
        }
      }
      __syncthreads();
      // a3 + a4: lane = LUT column; warp-stride over the CTA's rows.
      for (int rr = warp; rr < rows; rr += kWarps) {
        const int n = n0 + rr;
        float v = 0.f;
        if (lane < ng) {
          const int k0 = 8 * (s0 + lane);
#pragma unroll 1
          for (int i = 0; i < q; ++i) {
            const size_t row = (size_t)i * N + n;
            const uint32_t key = __ldg(planes + row * KB + s0 + lane);
            const int e = __ldg(exps + row * KG + k0 / g);
            const float v1 = shift_pow2(lut[key * 32 + lane], e);
            v += v1;
            if (exps2) v += shift_apot2(v1, __ldg(exps2 + row * KG + k0 / g));   // NEXT-f2
          }
        }
        // a5: fixed-order butterfly over the 32 columns.
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) acc[m * kRows + rr] += v;
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < M * rows; idx += blockDim.x) {
    const int m = idx / rows, rr = idx - m * rows;
    y[(size_t)m * ldy + n0 + rr] = __float2half_rn(acc[m * kRows + rr]);
  }
}

}  // namespace

LaunchPlan plan_generic(int M, int N, int K, int q, int g, int sms) {
  (void)M; (void)K; (void)q; (void)g; (void)sms;
  return LaunchPlan{(N + kRows - 1) / kRows, kWarps * 32, 0, 0};
}

cudaError_t launch_gemm_generic(const GemmArgs& a, const LaunchPlan& p) {
  gemm_generic_kernel<<<p.grid, p.threads, 0, a.stream>>>(a.x, a.ldx, a.planes, a.exps, a.exps2, a.M,
                                                           a.N, a.K, a.q, a.g, a.y, a.ldy);
  return cudaGetLastError();
}

}  // namespace shiftadd
