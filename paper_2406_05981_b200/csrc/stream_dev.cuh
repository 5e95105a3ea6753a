// stream_dev.cuh -- device helpers shared by the TMA-ring streaming kernels (lut_stream.cu,
// kernel 8; lut_program.cu, kernel 9): mbarrier / bulk-copy wrappers, the a2 LUT build into
// the 64 KB slab, and the a3 + a4 unit dot products over a ring stage.
#pragma once

#include "common.cuh"

namespace shiftadd {
namespace stream_dev {

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  smem_check(bar, 8);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  smem_check(bar, 8);
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  smem_check(bar, 8);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  smem_check(dst, bytes);
  smem_check(bar, 8);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
  smem_check(addr, 16);
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ int lds_s8(uint32_t addr) {
  smem_check(addr, 1);
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// a2: the 32 LUTs of one 256-k slice into column half `hoff` (0 or 128 B) of the slab at
// kDynBase, from the 8 activations of group `lane` (xv).  T[key] = (A[lo&3] + B[lo>>2]) +
// (C[hi&3] + D[hi>>2]): key bit b <-> +x_b if set, -x_b if clear;
// warp w writes the keys with hi nibble w, 32 consecutive words per store (conflict-free).
template <int NWC>
__device__ __forceinline__ void build_lut(const uint4 xv, uint32_t hoff, int warp, int lane) {
  const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
  const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
  const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
  const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
  const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
  const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
  const uint32_t col = kDynBase + hoff + 4 * lane;
#pragma unroll
  for (int hh = 0; hh < 16 / NWC; ++hh) {
    const int hi = warp + hh * NWC;
    const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                    ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), (A[lo & 3] + B[lo >> 2]) + H);
  }
}

// PRMT selector for step j: byte0 <- column byte (j&3) of cst[j>>2], byte1 <- key byte (j&3)
// of the weight word, bytes 2,3 <- sign of the column byte (< 0x80, so 0x00).
__host__ __device__ constexpr uint32_t step_sel(int j) {
  return ((8u | (4u + (j & 3))) << 12) | ((8u | (4u + (j & 3))) << 8) | ((uint32_t)(j & 3) << 4) | (4u + (j & 3));
}

// a4 -- the shift: 2^e as the float whose exponent field is e plus the
// bias, formed with one integer multiply-add on the bits of 1.0 (e << 23 + 0x3f800000); the
// chunk sum is then scaled in the accumulating FFMA.  p * 2^e is exact here (|p| in
// [2^-24, 2^24] or 0, e in [EXP_MIN, EXP_MAX]), so fma(p, 2^e, acc) rounds exactly like
// acc + (the exponent-field add on p) -- bit-identical to shift_pow2 + FADD, 3 instructions
// instead of 9.  EXP_ZERO (-128) is clamped to -127, whose bit pattern is +0.0: the group
// contributes 0.
__device__ __forceinline__ float pow2_bits(int e) {
  return __int_as_float((e < -127 ? -127 : e) * (1 << 23) + 0x3f800000);
}

// a3 + a4 for one unit (16 rows x 256 k, Q planes) read from a ring stage: per plane the 16
// lookups of the lane's 16 key bytes (4 chains, fixed tree), scaled by 2^e and accumulated.
template <int Q, uint32_t HOFF>
__device__ __forceinline__ float unit_dot(uint32_t sp, uint32_t se, const uint32_t (&cst)[4]) {
  uint4 w[Q];
  int e[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = lds_u4(sp + i * kTileBytes);
#pragma unroll
  for (int i = 0; i < Q; ++i) e[i] = lds_s8(se + i * kTileExps);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float p[4];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float v = lds_f32(kDynBase + HOFF + prmt(word, cst[j >> 2], step_sel(j)));
      p[j & 3] = j < 4 ? v : p[j & 3] + v;
    }
    acc = __fmaf_rn((p[0] + p[1]) + (p[2] + p[3]), pow2_bits(e[i]), acc);
  }
  return acc;
}

// Ring position: slot j and its use count k (the phase parity is k & 1).
struct RingPos {
  int j, k;
  __device__ __forceinline__ void next(int nst) {
    if (++j == nst) { j = 0; ++k; }
  }
};

// a3 + a4 for two units at once (ILP: the two lookup streams interleave, hiding LDS latency
// and the per-unit wait/emit of the other).  v1 = false: unit 1 absent (acc[1] = 0).
template <int Q, uint32_t HOFF>
__device__ __forceinline__ void unit_dot2(uint32_t sp0, uint32_t se0, uint32_t sp1, uint32_t se1, bool v1,
                                          const uint32_t (&cst)[4], float (&acc)[2]) {
  uint4 w[2][Q];
  int e[2][Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    w[0][i] = lds_u4(sp0 + i * kTileBytes);
    e[0][i] = lds_s8(se0 + i * kTileExps);
  }
  if (v1) {
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      w[1][i] = lds_u4(sp1 + i * kTileBytes);
      e[1][i] = lds_s8(se1 + i * kTileExps);
    }
  } else {
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      w[1][i] = make_uint4(0, 0, 0, 0);
      e[1][i] = SHIFTADD_EXP_ZERO;   // contributes +0
    }
  }
  acc[0] = 0.f;
  acc[1] = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float p[2][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t word = (j < 4) ? w[u][i].x : (j < 8) ? w[u][i].y : (j < 12) ? w[u][i].z : w[u][i].w;
        const float v = lds_f32(kDynBase + HOFF + prmt(word, cst[j >> 2], step_sel(j)));
        p[u][j & 3] = j < 4 ? v : p[u][j & 3] + v;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      acc[u] = __fmaf_rn((p[u][0] + p[u][1]) + (p[u][2] + p[u][3]), pow2_bits(e[u][i]), acc[u]);
  }
}


// Position in the unit order of a launch (P: the kernel's parameter block, with S, nseg, Ws and
// seg[].{q, RG, woff}): slice s, segment g, row group rg of that segment.
struct Pos {
  int s, g, rg;
};

// First unit whose weight offset is >= w (units are assigned by their starting offset).
// floor(c W / G) for c <= G <= 256 and W < 2^31 without 64-bit division:
// c W / G = c (W / G) + c (W % G) / G, every product below 2^31.
__device__ __forceinline__ long long split_point(long long c, long long W, long long G) {
  const unsigned q = (unsigned)W / (unsigned)G, rm = (unsigned)W % (unsigned)G;
  return (long long)((unsigned)c * q + ((unsigned)c * rm) / (unsigned)G);
}

template <class P>
__device__ __forceinline__ Pos pos_at(const P& p, long long w) {
  Pos r;
  // w <= S x Ws < 2^31 (S <= 256, Ws <= 4 x 65536 x segments): 32-bit division (a 64-bit
  // one is a ~100-instruction routine on the launch's critical path)
  r.s = (int)((unsigned)w / (unsigned)p.Ws);
  int wi = (int)w - r.s * p.Ws;
  r.g = 0;
  while (r.g + 1 < p.nseg && p.seg[r.g + 1].woff <= wi) ++r.g;
  const int q = p.seg[r.g].q;
  r.rg = (wi - p.seg[r.g].woff + q - 1) / q;
  if (r.rg >= p.seg[r.g].RG) {
    r.rg = 0;
    if (++r.g == p.nseg) { r.g = 0; ++r.s; }
  }
  return r;
}
__device__ __forceinline__ bool before(const Pos& a, const Pos& b) {
  return a.s != b.s ? a.s < b.s : (a.g != b.g ? a.g < b.g : a.rg < b.rg);
}
// End (exclusive) row group of the run (a.s, a.g) inside [a, end); moving to the next run.
template <class P>
__device__ __forceinline__ int run_end(const P& p, const Pos& a, const Pos& end) {
  return (a.s == end.s && a.g == end.g) ? end.rg : p.seg[a.g].RG;
}
template <class P>
__device__ __forceinline__ void next_run(const P& p, Pos& a, int re) {
  a.rg = re;
  if (a.rg >= p.seg[a.g].RG) {
    a.rg = 0;
    if (++a.g == p.nseg) { a.g = 0; ++a.s; }
  }
}

}  // namespace stream_dev
}  // namespace shiftadd
