// lut_stream.cu -- the all-SM streaming LUT-GEMV for the tiled layout (§8 a2-a6; kernel id 8).
//
// y = sum_i alpha_i (.) (B_i x) with LUT queries and exponent-add shifts,
// for one or several output "segments" that share the activations x (fused projections:
// LLaMA q/k/v or gate/up), each with its own bit width q (mixed 2/3/4-bit dispatch, §8 a6,
// PAPER.md:286-292).
//
// Decomposition.  A unit is (256-k slice s, segment, 16-row group rg); units are numbered
// slice-major.  A unit of a q-bit segment weighs q (its bytes).  The grid is one CTA per SM
// and CTA c takes the units whose weight offset falls in [c W/G, (c+1) W/G): one contiguous
// byte range per (slice, segment), at most two slices per CTA (S <= G), so the CTA builds at
// most two LUTs (a2), once, in the two column halves of one 64 KB slab.
//
// Weights.  Warp 16 is a producer: one thread streams the CTA's units through a ring of
// shared-memory stages with 1-D bulk copies (cp.async.bulk, the TMA engine), 16 units per
// stage, each stage completing on its "full" mbarrier and released by the 16 consumer warps on
// its "empty" one.  It starts at kernel entry, before griddepcontrol.wait: the weights never
// depend on the upstream kernel (SHIFTADD_FLAG_PDL contract), so HBM is busy while the
// previous call drains.  The consumers wait, fetch x, build the LUTs, then take one unit per
// warp per stage: LDS.128 of the lane's 16 key bytes per plane (the tiled layout's rotation
// makes every lookup step hit 32 different LUT columns: conflict-free), one PRMT + one
// LDS [R+imm] + one FADD per key byte (a3), the chunk sum times 2^e by an exponent-field add
// (a4).
//
// Split-K reduction (a5) without fences or counters.  Every (slice, row) partial goes to the
// workspace as one 64-bit word {epoch, fp32 bits}, stored with a single relaxed store, so a
// reader that sees the call's epoch sees the value.  CTA c owns an equal share of the row
// groups; after its own units it polls the S words of each owned row until all carry this
// call's epoch, sums them in slice order (deterministic) and stores fp16 (RNE).  The epoch is
// the call count: a 64-bit counter in the workspace to which every call's CTAs add exactly
// 2^32 in total (CTA 0 adds 2^32 - (G-1), the others 1, fire-and-forget at their end) -- any
// proper subset of the adds stays below the next multiple of 2^32, so every CTA of a call,
// reading it after griddepcontrol.wait, sees the same epoch (counter >> 32) + 1, and stale
// words of earlier calls never match.
#include <mutex>

#include "common.cuh"
#include "stream_dev.cuh"

namespace shiftadd {
namespace {
using namespace stream_dev;

constexpr int kLutSlab = kLutBytes;          // 64 KB: two slices' LUTs (column halves)
constexpr int kBarBytes = 512;               // full[16] at +0, empty[16] at +128, epoch at +256

#ifdef SHIFTADD_DEV_TRACE
// development builds only (tools/dev_build.sh): per-CTA phase timestamps
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ void trace_at(int k) {
  if (g_trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[16 * blockIdx.x + k] = t;
  }
}
__device__ __forceinline__ void trace_clk(int k, long long c0) {   // cycles since c0 (same SM)
  if (g_trace && threadIdx.x == 0) g_trace[16 * blockIdx.x + k] = (unsigned long long)(clock64() - c0);
}
#else
__device__ __forceinline__ void trace_at(int) {}
__device__ __forceinline__ void trace_clk(int, long long) {}
#endif

struct SegDev {
  const uint8_t* planes;
  const int8_t* exps;
  __half* y;
  int q, RG, N, rgoff, woff;
};

struct StreamParams {
  const __half* x;
  int M, ldx, ldy;          // batch rows (<= 8 per launch), row strides of x and of every y
  int one_slice;            // 1: G = S x cps CTAs, CTA c covers 1/cps of slice c / cps (MW = 8)
  int lut_bytes;            // LUT region at kDynBase (64 KB or 128 KB); the ring follows
  int S, nseg, RGtot, Ws;   // Ws = sum over segments of q * RG (weight of one slice)
  SegDev seg[kMaxSegments];
  unsigned long long* done;   // epoch counter (workspace)
  unsigned long long* part;   // {epoch, fp32} [M][RGtot][S][16]
  int nst, slot, slot_planes;
  int su;    // units per stage (16, 8 or 4); consumer warp w serves stages t with
             // t % (16 / su) == w / su, unit w % su
  int pdl;
  int skew;   // offset the two warp halves' stage pairs (see consume_run)
  const int8_t* exps_bw;   // NEXT-f1 block-wise exponents [q][8][K/8] (BW kernels; planes only in the ring)
  int bw_rows;             // rows per block, N / 8
  int bw_rgb;              // BW = 2: row groups per block (N / 128)
  GatherArgs ga;           // NEXT-f3 fused all-gather epilogue (P == 0: off)
  int dev_mode;            // development builds only (co-roof experiments), 0 otherwise
  const unsigned long long* part_end;   // end of the partial region (bounds-checked builds)
  const int8_t* exps2;     // NEXT-f2 (BW = 5): second-term codes, streamed as a third array
  int slot_exps2;          // its offset in a ring slot
};

// A split-K partial word store (bounds-checked builds: inside [part, part_end)).
__device__ __forceinline__ void st_part(const StreamParams& p, unsigned long long* q, unsigned long long v) {
#ifdef SHIFTADD_BOUNDS_CHECK
  if (q < p.part || q >= p.part_end) __trap();
#endif
  stream_dev::st_relaxed_u64(q, v);
}

#ifdef SHIFTADD_DEV_TRACE
// co-roof experiment (dev builds): the lookups and adds of unit_dot2 with key words made in
// registers -- no LDS.128 of the staged key bytes (results meaningless)
template <int Q, uint32_t HOFF>
__device__ __forceinline__ void unit_dot2_regs(int lane, int seed, const uint32_t (&cst)[4], float (&acc)[2]) {
  acc[0] = 0.f;
  acc[1] = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float pp[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t b = (uint32_t)(lane * 0x01030507 + seed * 0x0b0d1113 + i * 0x11111111 + u * 0x2f2f2f2f);
      const uint4 w = make_uint4(b, b * 3u, b * 5u, b * 7u);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t word = (j < 4) ? w.x : (j < 8) ? w.y : (j < 12) ? w.z : w.w;
        const float v = lds_f32(kDynBase + HOFF + prmt(word, cst[j >> 2], step_sel(j)));
        pp[u][j & 3] = j < 4 ? v : pp[u][j & 3] + v;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) acc[u] += (pp[u][0] + pp[u][1]) + (pp[u][2] + pp[u][3]);
  }
}
#endif

// NEXT-f2, additive PoT with two terms (Eq. 2): per plane the 128-k chunk
// sum p gives v1 = p 2^{P1} (exponent add) plus the second term sign(c2) v1 2^{-|c2|}
// (shift_apot2, common.cuh) -- the cluster kernel's arithmetic, on two units at once.
template <int Q, uint32_t HOFF>
__device__ __forceinline__ void unit_dot2_ap2(uint32_t sp0, uint32_t se0, uint32_t sq0, uint32_t sp1, uint32_t se1,
                                              uint32_t sq1, bool v1, const uint32_t (&cst)[4], float (&acc)[2]) {
  uint4 w[2][Q];
  int e[2][Q], c[2][Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    w[0][i] = lds_u4(sp0 + i * kTileBytes);
    e[0][i] = lds_s8(se0 + i * kTileExps);
    c[0][i] = lds_s8(sq0 + i * kTileExps);
    if (v1) {
      w[1][i] = lds_u4(sp1 + i * kTileBytes);
      e[1][i] = lds_s8(se1 + i * kTileExps);
      c[1][i] = lds_s8(sq1 + i * kTileExps);
    } else {
      w[1][i] = make_uint4(0, 0, 0, 0);
      e[1][i] = SHIFTADD_EXP_ZERO;
      c[1][i] = 0;
    }
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float pp[2][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t word = (j < 4) ? w[u][i].x : (j < 8) ? w[u][i].y : (j < 12) ? w[u][i].z : w[u][i].w;
        const float v = lds_f32(kDynBase + HOFF + prmt(word, cst[j >> 2], step_sel(j)));
        pp[u][j & 3] = j < 4 ? v : pp[u][j & 3] + v;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float t1 = shift_pow2((pp[u][0] + pp[u][1]) + (pp[u][2] + pp[u][3]), e[u][i]);
      const float vt = t1 + shift_apot2(t1, c[u][i]);
      acc[u] = i == 0 ? vt : acc[u] + vt;
    }
  }
}

// Consumer side of one run (slice s, segment sg, row groups [rga, re)): the run's stages of su
// units, taken two at a time -- warp w processes unit w of stage t and unit w of stage t + 1
// together, then releases both.
template <int Q, uint32_t HOFF, bool AP2 = false>
__device__ __forceinline__ void consume_run(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                            RingPos& rp, int& t, uint32_t ring, uint32_t full, uint32_t empty,
                                            const uint32_t (&cst)[4], int wu, int lane, unsigned long long ep,
                                            bool skew) {
  const int r = lane >> 1, h = lane & 1;
  // partial words [flat row group][slice][16 rows]: a unit's 16 sums are one 128-B line, and an
  // owner's (row group, all slices) block is S contiguous lines
  unsigned long long* prow = p.part + ((size_t)sg.rgoff * p.S + s) * kTileRows + r;
  // Warps of the upper half take the run's first stage alone and then pairs: the two halves'
  // pairs are offset by one stage, so one half's barrier waits and stores overlap the other
  // half's lookups instead of the whole CTA stalling in lockstep.
  bool single = skew;
  for (int rg = rga; rg < re;) {
    const int n0 = re - rg < p.su ? re - rg : p.su;
    const int left = re - rg - n0;
    const int n1 = single ? 0 : (left < p.su ? left : p.su);   // may be <= 0: no second stage
    single = false;
    const RingPos r0 = rp;
    rp.next(p.nst);
    const RingPos r1 = rp;
    if (n1 > 0) rp.next(p.nst);
    t += n1 > 0 ? 2 : 1;
    const uint32_t slot0 = ring + (uint32_t)(r0.j * p.slot), slot1 = ring + (uint32_t)(r1.j * p.slot);
    const long long c0 = clock64();
    mbar_wait(full + 8 * r0.j, (uint32_t)(r0.k & 1));
    if (n1 > 0) mbar_wait(full + 8 * r1.j, (uint32_t)(r1.k & 1));
    if (rg == rga) trace_clk(8, c0);
    const bool u0 = wu < n0, u1 = wu < n1;
    float acc[2] = {0.f, 0.f};
#ifdef SHIFTADD_DEV_TRACE
    if (u0 && (p.dev_mode & 8)) unit_dot2_regs<Q, HOFF>(lane, rg, cst, acc); else
#endif
    if (u0 && AP2)
      unit_dot2_ap2<Q, HOFF>(slot0 + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                             slot0 + (uint32_t)(p.slot_planes + wu * Q * kTileExps + lane),
                             slot0 + (uint32_t)(p.slot_exps2 + wu * Q * kTileExps + lane),
                             slot1 + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                             slot1 + (uint32_t)(p.slot_planes + wu * Q * kTileExps + lane),
                             slot1 + (uint32_t)(p.slot_exps2 + wu * Q * kTileExps + lane), u1, cst, acc);
    else if (u0)
      unit_dot2<Q, HOFF>(slot0 + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                         slot0 + (uint32_t)(p.slot_planes + wu * Q * kTileExps + lane),
                         slot1 + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                         slot1 + (uint32_t)(p.slot_planes + wu * Q * kTileExps + lane), u1, cst, acc);
    if (rg == rga) trace_clk(9, c0);
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(empty + 8 * r0.j);
      if (n1 > 0) mbar_arrive(empty + 8 * r1.j);
    }
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
    acc[1] += __shfl_xor_sync(0xffffffffu, acc[1], 1);
    if (h == 0) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k == 0 ? u0 : u1) {
          const int u = rg + k * p.su + wu;
          if (p.S == 1) {
            const int nl = u * kTileRows + r;
            if (nl < sg.N) sg.y[nl] = __float2half_rn(acc[k]);
          } else {
            st_part(p, prow + (size_t)u * p.S * kTileRows, ep | __float_as_uint(acc[k]));
          }
        }
      }
    }
    if (rg == rga) trace_clk(10, c0);
    rg += n0 + (n1 > 0 ? n1 : 0);
  }
}

template <uint32_t HOFF, bool AP2 = false>
__device__ __forceinline__ void consume_run_q(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                              RingPos& rp, int& t, uint32_t ring, uint32_t full, uint32_t empty,
                                              const uint32_t (&cst)[4], int wu, int lane, unsigned long long ep,
                                              bool skew) {
  switch (sg.q) {
    case 1: consume_run<1, HOFF, AP2>(p, sg, s, rga, re, rp, t, ring, full, empty, cst, wu, lane, ep, skew); break;
    case 2: consume_run<2, HOFF, AP2>(p, sg, s, rga, re, rp, t, ring, full, empty, cst, wu, lane, ep, skew); break;
    case 3: consume_run<3, HOFF, AP2>(p, sg, s, rga, re, rp, t, ring, full, empty, cst, wu, lane, ep, skew); break;
    default: consume_run<4, HOFF, AP2>(p, sg, s, rga, re, rp, t, ring, full, empty, cst, wu, lane, ep, skew); break;
  }
}

// ------------------------------------------------------------------------------------------
// a7 small batch (App. D): M-wide LUT entries, one weight pass for M rows.
// A LUT entry holds MW fp16 partial sums -- rows 0..MW-1 of x against the same 8-k group and
// key -- built in fp32 and rounded once (the paper's FP16 LUT; reading R8/C10),
// so one LDS.{32,64,128} per key byte serves MW rows, and each half is accumulated into fp32
// by one FHADD (fp32 + fp16 -> fp32, the .H0/.H1 half selected in the instruction).
//   MW = 2: 4-B entries, the M = 1 slab layout (two slices in the column halves; 64 KB)
//   MW = 4: 8-B entries, slice t at +64K t, group g at 8-B slot 16(g>>4) + ((g&15) ^ 8(g>>4))
//   MW = 8: 16-B entries, one slice, groups 16h..16h+15 at +64K h, slot (g&15) ^ 4h
// The slots make every LDS phase (32/16/8 lanes) hit distinct banks for any keys.
template <int MW>
__host__ __device__ constexpr uint32_t mw_col(int g) {   // byte offset of group g in a key row
  return MW == 2 ? 4u * (uint32_t)g
                 : MW == 4 ? 8u * (uint32_t)(16 * (g >> 4) + ((g & 15) ^ (8 * (g >> 4))))
                           : 16u * (uint32_t)((g & 15) ^ (4 * (g >> 4)));
}
template <int MW>
__host__ __device__ constexpr uint32_t mw_hi(int g) {   // 64 KB block of group g (MW = 8)
  return MW == 8 ? (uint32_t)(g >> 4) : 0u;
}
// LUT base of slice t (0 or 1) of the CTA
template <int MW>
__host__ __device__ constexpr uint32_t mw_slice_base(int t) {
  return kDynBase + (MW == 2 ? 128u * t : MW == 4 ? 65536u * t : 0u);
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// a2 for MW rows: lane = group g; warp w writes keys with hi nibble w (+ NWC ...).
template <int NWC, int MW>
__device__ __forceinline__ void build_lut_mw(const StreamParams& p, int s, int t, int warp, int lane) {
  float sa[MW], da[MW], sb[MW], db[MW], x4[MW], x5[MW], x6[MW], x7[MW];
  const uint64_t pol_keep = policy_evict_last();
#pragma unroll
  for (int m = 0; m < MW; ++m) {
    uint4 xv = make_uint4(0, 0, 0, 0);
    if (m < p.M) xv = ldg_keep(p.x + (size_t)m * p.ldx + (size_t)s * kTileK + 8 * lane, pol_keep);
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
    const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
    const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
    sa[m] = f01.x + f01.y; da[m] = f01.x - f01.y;
    sb[m] = f23.x + f23.y; db[m] = f23.x - f23.y;
    x4[m] = f45.x; x5[m] = f45.y; x6[m] = f67.x; x7[m] = f67.y;
  }
  const uint32_t row0 = mw_slice_base<MW>(t) + 65536u * mw_hi<MW>(lane) + mw_col<MW>(lane);
#pragma unroll
  for (int hh = 0; hh < 16 / NWC; ++hh) {
    const int hi = warp + hh * NWC;
    float H[MW];
#pragma unroll
    for (int m = 0; m < MW; ++m)
      H[m] = ((hi & 1 ? x4[m] : -x4[m]) + (hi & 2 ? x5[m] : -x5[m])) + ((hi & 4 ? x6[m] : -x6[m]) + (hi & 8 ? x7[m] : -x7[m]));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) {
      // A[lo&3] = {-s, d, -d, s}(x0, x1), B[lo>>2] likewise from (x2, x3): key bit b -> +-x_b
      float e[MW];
#pragma unroll
      for (int m = 0; m < MW; ++m) {
        const int a = lo & 3, b = lo >> 2;
        const float A = a == 0 ? -sa[m] : a == 1 ? da[m] : a == 2 ? -da[m] : sa[m];
        const float B = b == 0 ? -sb[m] : b == 1 ? db[m] : b == 2 ? -db[m] : sb[m];
        e[m] = (A + B) + H[m];
      }
      const uint32_t addr = row0 + ((uint32_t)(hi * 16 + lo) << 8);
      if (MW == 2) {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(pack_h2(e[0], e[1])) : "memory");
      } else if (MW == 4) {
        asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(addr), "r"(pack_h2(e[0], e[1])),
                     "r"(pack_h2(e[2 % MW], e[3 % MW])) : "memory");
      } else {
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(pack_h2(e[0], e[1])),
                     "r"(pack_h2(e[2 % MW], e[3 % MW])), "r"(pack_h2(e[4 % MW], e[5 % MW])),
                     "r"(pack_h2(e[6 % MW], e[7 % MW])) : "memory");
      }
    }
  }
}

// Lookup address of step j: byte 0 = column byte (cst byte j&1), byte 1 = key byte (word byte
// j&3), byte 2 = 64 KB block (cst byte 2), byte 3 = 0.
__host__ __device__ constexpr uint32_t step_sel_mw(int j) {
  return (7u << 12) | (6u << 8) | ((uint32_t)(j & 3) << 4) | (4u + (j & 1));
}

__device__ __forceinline__ void fhadd_lo(float& acc, uint32_t v) {
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; add.rn.f32.f16 %0, l, %0;}" : "+f"(acc) : "r"(v));
}
__device__ __forceinline__ void fhadd_hi(float& acc, uint32_t v) {
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; add.rn.f32.f16 %0, h, %0;}" : "+f"(acc) : "r"(v));
}

// a3 + a4 for one unit, MW rows: per plane 16 lookups (2 chains of MW fp32 sums), scaled by
// 2^e into acc[MW].
template <int Q, uint32_t BASE, int MW>
__device__ __forceinline__ void unit_dot_mw(uint32_t sp, uint32_t se, const uint32_t (&cst)[8], float (&acc)[MW]) {
  uint4 w[Q];
  int e[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = lds_u4(sp + i * kTileBytes);
#pragma unroll
  for (int i = 0; i < Q; ++i) e[i] = lds_s8(se + i * kTileExps);
#pragma unroll
  for (int m = 0; m < MW; ++m) acc[m] = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float c[2][MW];
#pragma unroll
    for (int m = 0; m < MW; ++m) c[0][m] = c[1][m] = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const uint32_t a = BASE + prmt(word, cst[j >> 1], step_sel_mw(j));
      uint32_t v[4];
      if (MW == 2) {
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v[0]) : "r"(a));
      } else if (MW == 4) {
        asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(a));
      } else {
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(a));
      }
#pragma unroll
      for (int m = 0; m < MW; m += 2) {
        fhadd_lo(c[j & 1][m], v[m >> 1]);
        fhadd_hi(c[j & 1][m + 1], v[m >> 1]);
      }
    }
    const float sc = pow2_bits(e[i]);
#pragma unroll
    for (int m = 0; m < MW; ++m) acc[m] = __fmaf_rn(c[0][m] + c[1][m], sc, acc[m]);
  }
}

// Consumer side of one run for MW rows: one unit per warp per stage.
template <int Q, uint32_t BASE, int MW>
__device__ __forceinline__ void consume_run_mw(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                               RingPos& rp, uint32_t ring, uint32_t full, uint32_t empty,
                                               const uint32_t (&cst)[8], int wu, int lane, unsigned long long ep) {
  const int r = lane >> 1, h = lane & 1;
  for (int rg = rga; rg < re; rg += p.su, rp.next(p.nst)) {
    const int n = re - rg < p.su ? re - rg : p.su;
    const uint32_t slot = ring + (uint32_t)(rp.j * p.slot);
    mbar_wait(full + 8 * rp.j, (uint32_t)(rp.k & 1));
    if (wu < n) {
      float acc[MW];
      unit_dot_mw<Q, BASE, MW>(slot + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                               slot + (uint32_t)(p.slot_planes + wu * Q * kTileExps + lane), cst, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * rp.j);
#pragma unroll
      for (int m = 0; m < MW; ++m) acc[m] += __shfl_xor_sync(0xffffffffu, acc[m], 1);
      if (h == 0) {
        const int u = rg + wu;
#pragma unroll
        for (int m = 0; m < MW; ++m) {
          if (m < p.M) {
            if (p.S == 1) {
              const int nl = u * kTileRows + r;
              if (nl < sg.N) sg.y[(size_t)m * p.ldy + nl] = __float2half_rn(acc[m]);
            } else {
              const size_t w = ((((size_t)m * p.RGtot + sg.rgoff + u) * p.S) + s) * kTileRows + r;
              st_part(p, p.part + w, ep | __float_as_uint(acc[m]));
            }
          }
        }
      }
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * rp.j);
    }
  }
}

template <uint32_t BASE, int MW>
__device__ __forceinline__ void consume_run_mw_q(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                                 RingPos& rp, uint32_t ring, uint32_t full, uint32_t empty,
                                                 const uint32_t (&cst)[8], int wu, int lane, unsigned long long ep) {
  switch (sg.q) {
    case 1: consume_run_mw<1, BASE, MW>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
    case 2: consume_run_mw<2, BASE, MW>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
    case 3: consume_run_mw<3, BASE, MW>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
    default: consume_run_mw<4, BASE, MW>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
  }
}

// ------------------------------------------------------------------------------------------
// NEXT-f1 block-wise scales, "Ours (Lat.)": one PoT scale per (row block
// of N/8 rows, 8-column group) -- the 8 weights of a key byte share it, so each LUT query is
// scaled once: acc = fma(T[key], 2^e, acc), the 2^e formed by an integer add on the exponent
// field of 1.0 (pow2_bits).  A lane's 16 queries of a plane touch 16 column groups (the tiled
// rotation), so it keeps those 16 q scale factors in registers for the current (slice, row
// block) and reloads them (16 q bytes of the compact [q][8][K/8] array, L1/L2 resident) only
// when its row block changes.  The exponent array is never streamed: q K bytes per call.
// The 16 q scale factors of a lane are kept as bf16 pairs (2^e is exact in bf16: an 8-bit
// exponent and no mantissa), 8 q registers; a query widens its factor back to fp32 with one
// shift or mask (the high half is already an fp32 bit pattern once the low half is cleared).
template <int Q>
__device__ __forceinline__ void load_bw_scales(const int8_t* __restrict__ exps_bw, int KB, int s, int b, int r, int h,
                                               uint32_t (&S2)[Q][8]) {
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    // the lane's 16 groups 32s + 16h + 0..15 are one aligned 16-B load; step j uses group
    // (j + r) & 15, so rotate the 16 bytes right by r (words by r >> 2, then bytes by r & 3)
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(exps_bw + ((size_t)i * 8 + b) * KB + 32 * s + 16 * h));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const int rw = r >> 2, rb = r & 3;
    uint32_t t[4], e4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      t[k] = rw == 0 ? w[k] : rw == 1 ? w[(k + 1) & 3] : rw == 2 ? w[(k + 2) & 3] : w[(k + 3) & 3];
#pragma unroll
    for (int k = 0; k < 4; ++k) e4[k] = __funnelshift_r(t[k], t[(k + 1) & 3], 8 * rb);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t pr = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = 2 * k + u;
        const int e = (int)(int8_t)((e4[j >> 2] >> (8 * (j & 3))) & 0xffu);
        pr |= ((uint32_t)(e < -127 ? 0 : e + 127) << 7) << (16 * u);   // bf16 bits of 2^e (EXP_ZERO: +0)
      }
      S2[i][k] = pr;
    }
  }
}

template <int Q, uint32_t HOFF>
__device__ __forceinline__ float unit_dot_bw(uint32_t sp, const uint32_t (&cst)[4], const uint32_t (&S2)[Q][8]) {
  uint4 w[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = lds_u4(sp + i * kTileBytes);
  float pc[4];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float v = lds_f32(kDynBase + HOFF + prmt(word, cst[j >> 2], step_sel(j)));
      const float sc = __uint_as_float((j & 1) ? (S2[i][j >> 1] & 0xffff0000u) : (S2[i][j >> 1] << 16));
      pc[j & 3] = (i == 0 && j < 4) ? v * sc : __fmaf_rn(v, sc, pc[j & 3]);
    }
  }
  return (pc[0] + pc[1]) + (pc[2] + pc[3]);
}

template <int Q, uint32_t HOFF>
__device__ __forceinline__ void consume_run_bw(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                               RingPos& rp, uint32_t ring, uint32_t full, uint32_t empty,
                                               const uint32_t (&cst)[4], int wu, int lane, unsigned long long ep) {
  const int r = lane >> 1, h = lane & 1;
  uint32_t S[Q][8];
  int cur_b = -1;
  for (int rg = rga; rg < re; rg += p.su, rp.next(p.nst)) {
    const int n = re - rg < p.su ? re - rg : p.su;
    const uint32_t slot = ring + (uint32_t)(rp.j * p.slot);
    const int u = rg + wu;
    if (wu < n) {
      const int nrow = u * kTileRows + r;
      int b = nrow / p.bw_rows;
      b = b > 7 ? 7 : b;   // padding rows of the last row group
      if (b != cur_b) {
        load_bw_scales<Q>(p.exps_bw, p.S * (kTileK / 8), s, b, r, h, S);
        cur_b = b;
      }
    }
    mbar_wait(full + 8 * rp.j, (uint32_t)(rp.k & 1));
    if (wu < n) {
      float acc = unit_dot_bw<Q, HOFF>(slot + (uint32_t)(wu * Q * kTileBytes + 16 * lane), cst, S);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * rp.j);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (h == 0) {
        if (p.S == 1) {
          const int nl = u * kTileRows + r;
          if (nl < sg.N) sg.y[nl] = __float2half_rn(acc);
        } else {
          const size_t w = (((size_t)sg.rgoff + u) * p.S + s) * kTileRows + r;
          st_part(p, p.part + w, ep | __float_as_uint(acc));
        }
      }
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * rp.j);
    }
  }
}

template <uint32_t HOFF>
__device__ __forceinline__ void consume_run_bw_q(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                                 RingPos& rp, uint32_t ring, uint32_t full, uint32_t empty,
                                                 const uint32_t (&cst)[4], int wu, int lane, unsigned long long ep) {
  switch (sg.q) {
    case 1: consume_run_bw<1, HOFF>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
    case 2: consume_run_bw<2, HOFF>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
    case 3: consume_run_bw<3, HOFF>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
    default: consume_run_bw<4, HOFF>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep); break;
  }
}

// BW = 2 (N % 128 == 0: a row block is whole row groups): the block scales are folded into
// the LUT instead -- for the (slice, row block) a run of units lies in, plane i gets its own
// LUT T'_i[c][key] = 2^{e_i[b][c]} T_c[key] (an exact fp32 scaling by a power of two), so a
// query is PRMT + LDS + FADD as in the row-wise kernel and no shift remains per query or per
// chunk.  Plane i's LUT sits in slab i >> 1, column half i & 1 (the LDS immediate); the CTA
// rebuilds its q LUTs when its units cross into the next row block or slice (consumer warps
// meet on a named barrier before and after).
template <int NWC, int Q>
__device__ __forceinline__ void build_lut_scaled(const uint4 xv, const int8_t* __restrict__ exps_bw, int KB, int s, int b,
                                                 int warp, int lane) {
  const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
  const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
  const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
  const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
  const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
  const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
  float sc[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) sc[i] = pow2_bits((int)__ldg(exps_bw + ((size_t)i * 8 + b) * KB + 32 * s + lane));
#pragma unroll
  for (int hh = 0; hh < 16 / NWC; ++hh) {
    const int hi = warp + hh * NWC;
    const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                    ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) {
      const float t = (A[lo & 3] + B[lo >> 2]) + H;
#pragma unroll
      for (int i = 0; i < Q; ++i)
        sts_f32(kDynBase + (uint32_t)(i >> 1) * 65536u + (uint32_t)(i & 1) * 128u + 4u * lane + ((uint32_t)(hi * 16 + lo) << 8),
                t * sc[i]);
    }
  }
}

// NEXT-f1 column-wise scales, "Ours (Acc.)" (realisation SPEC.md:375,
// reading R18): plane i has one PoT scale per input column k, so the shift moves onto the
// activations -- plane i's LUT of the slice is built from x[k] 2^{e_i[k]} (an exact fp32
// multiply by a power of two; EXP_ZERO gives +0) and queried unscaled.  Same slab layout as
// the block-wise scaled LUTs (plane i in slab i >> 1, column half i & 1); lane = group of 8 k.
template <int NWC, int Q>
__device__ __forceinline__ void build_lut_colw(const uint4 xv, const int8_t* __restrict__ exps_col, int K, int s,
                                               int warp, int lane) {
  const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
  const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
  const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
  const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
  const float x8[8] = {f01.x, f01.y, f23.x, f23.y, f45.x, f45.y, f67.x, f67.y};
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const uint2 ev = __ldg(reinterpret_cast<const uint2*>(exps_col + (size_t)i * K + (size_t)s * kTileK + 8 * lane));
    float v[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int e = (int)(int8_t)(((b < 4 ? ev.x : ev.y) >> (8 * (b & 3))) & 0xffu);
      v[b] = x8[b] * pow2_bits(e);
    }
    const float A[4] = {-v[0] - v[1], v[0] - v[1], v[1] - v[0], v[0] + v[1]};
    const float B[4] = {-v[2] - v[3], v[2] - v[3], v[3] - v[2], v[2] + v[3]};
    const uint32_t col = kDynBase + (uint32_t)(i >> 1) * 65536u + (uint32_t)(i & 1) * 128u + 4u * lane;
#pragma unroll
    for (int hh = 0; hh < 16 / NWC; ++hh) {
      const int hi = warp + hh * NWC;
      const float H = ((hi & 1 ? v[4] : -v[4]) + (hi & 2 ? v[5] : -v[5])) + ((hi & 4 ? v[6] : -v[6]) + (hi & 8 ? v[7] : -v[7]));
#pragma unroll
      for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), (A[lo & 3] + B[lo >> 2]) + H);
    }
  }
}

template <int Q>
__device__ __forceinline__ float unit_dot_lut(uint32_t sp, const uint32_t (&cst)[4]) {
  uint4 w[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = lds_u4(sp + i * kTileBytes);
  float pc[4];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const uint32_t base = kDynBase + (uint32_t)(i >> 1) * 65536u + (uint32_t)(i & 1) * 128u;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float v = lds_f32(base + prmt(word, cst[j >> 2], step_sel(j)));
      pc[j & 3] = (i == 0 && j < 4) ? v : pc[j & 3] + v;
    }
  }
  return (pc[0] + pc[1]) + (pc[2] + pc[3]);
}

// Column-wise scales for two batch rows (a7 x NEXT-f1): plane i's LUT entry holds the fp16
// pair (row 0, row 1) of the sums of x_m[k] 2^{e_i[k]} -- built in fp32, rounded once -- at the
// address of the fp32 entry of the M = 1 layout, so one LDS.32 per key byte serves both rows
// (each half accumulated into fp32 by one FHADD).
template <int NWC, int Q>
__device__ __forceinline__ void build_lut_colw2(const StreamParams& p, int s, int warp, int lane) {
  const uint64_t pol_keep = policy_evict_last();
  float v[2][8];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    uint4 xv = make_uint4(0, 0, 0, 0);
    if (m < p.M) xv = ldg_keep(p.x + (size_t)m * p.ldx + (size_t)s * kTileK + 8 * lane, pol_keep);
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
    const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
    const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
    v[m][0] = f01.x; v[m][1] = f01.y; v[m][2] = f23.x; v[m][3] = f23.y;
    v[m][4] = f45.x; v[m][5] = f45.y; v[m][6] = f67.x; v[m][7] = f67.y;
  }
  const int K = p.S * kTileK;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const uint2 ev = __ldg(reinterpret_cast<const uint2*>(p.exps_bw + (size_t)i * K + (size_t)s * kTileK + 8 * lane));
    float w[2][8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const float sc = pow2_bits((int)(int8_t)(((b < 4 ? ev.x : ev.y) >> (8 * (b & 3))) & 0xffu));
      w[0][b] = v[0][b] * sc;
      w[1][b] = v[1][b] * sc;
    }
    const uint32_t col = kDynBase + (uint32_t)(i >> 1) * 65536u + (uint32_t)(i & 1) * 128u + 4u * lane;
#pragma unroll
    for (int hh = 0; hh < 16 / NWC; ++hh) {
      const int hi = warp + hh * NWC;
      float H[2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
        H[m] = ((hi & 1 ? w[m][4] : -w[m][4]) + (hi & 2 ? w[m][5] : -w[m][5])) +
               ((hi & 4 ? w[m][6] : -w[m][6]) + (hi & 8 ? w[m][7] : -w[m][7]));
#pragma unroll
      for (int lo = 0; lo < 16; ++lo) {
        float e[2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int a = lo & 3, b = lo >> 2;
          const float A = a == 0 ? -w[m][0] - w[m][1] : a == 1 ? w[m][0] - w[m][1] : a == 2 ? w[m][1] - w[m][0]
                                                                                              : w[m][0] + w[m][1];
          const float B = b == 0 ? -w[m][2] - w[m][3] : b == 1 ? w[m][2] - w[m][3] : b == 2 ? w[m][3] - w[m][2]
                                                                                              : w[m][2] + w[m][3];
          e[m] = (A + B) + H[m];
        }
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(col + ((uint32_t)(hi * 16 + lo) << 8)), "r"(pack_h2(e[0], e[1]))
                     : "memory");
      }
    }
  }
}

template <int Q>
__device__ __forceinline__ void unit_dot_lut2(uint32_t sp, const uint32_t (&cst)[4], float (&acc)[2]) {
  uint4 w[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = lds_u4(sp + i * kTileBytes);
  float c[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const uint32_t base = kDynBase + (uint32_t)(i >> 1) * 65536u + (uint32_t)(i & 1) * 128u;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      uint32_t v;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + prmt(word, cst[j >> 2], step_sel(j))));
      fhadd_lo(c[j & 1][0], v);
      fhadd_hi(c[j & 1][1], v);
    }
  }
  acc[0] = c[0][0] + c[1][0];
  acc[1] = c[0][1] + c[1][1];
}

template <int NWC, int Q, bool COLW, bool MW2 = false>
__device__ __forceinline__ void consume_run_lut(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                                RingPos& rp, uint32_t ring, uint32_t full, uint32_t empty,
                                                const uint32_t (&cst)[4], int wu, int lane, unsigned long long ep,
                                                const uint4 xv, int& cur) {
  const int r = lane >> 1, h = lane & 1;
  const int KB = p.S * (kTileK / 8);
  for (int r0 = rga; r0 < re;) {
    const int b = r0 / p.bw_rgb;
    const int r1 = (b + 1) * p.bw_rgb < re ? (b + 1) * p.bw_rgb : re;
    const int key = s * 8 + b;
    if (key != cur) {   // rebuild the q scaled LUTs for (s, b) (column-wise: for s)
      asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");
      if (MW2)
        build_lut_colw2<NWC, Q>(p, s, wu, lane);
      else if (COLW)
        build_lut_colw<NWC, Q>(xv, p.exps_bw, p.S * kTileK, s, wu, lane);
      else
        build_lut_scaled<NWC, Q>(xv, p.exps_bw, KB, s, b, wu, lane);
      asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");
      cur = key;
    }
    for (int rg = r0; rg < r1; rg += p.su, rp.next(p.nst)) {
      const int n = r1 - rg < p.su ? r1 - rg : p.su;
      const uint32_t slot = ring + (uint32_t)(rp.j * p.slot);
      mbar_wait(full + 8 * rp.j, (uint32_t)(rp.k & 1));
      if (wu < n && MW2) {
        float acc[2];
        unit_dot_lut2<Q>(slot + (uint32_t)(wu * Q * kTileBytes + 16 * lane), cst, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * rp.j);
#pragma unroll
        for (int m = 0; m < 2; ++m) acc[m] += __shfl_xor_sync(0xffffffffu, acc[m], 1);
        if (h == 0) {
          const int u = rg + wu;
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            if (m < p.M) {
              if (p.S == 1) {
                const int nl = u * kTileRows + r;
                if (nl < sg.N) sg.y[(size_t)m * p.ldy + nl] = __float2half_rn(acc[m]);
              } else {
                st_part(p, p.part + ((((size_t)m * p.RGtot + sg.rgoff + u) * p.S) + s) * kTileRows + r,
                               ep | __float_as_uint(acc[m]));
              }
            }
          }
        }
      } else if (wu < n) {
        float acc = unit_dot_lut<Q>(slot + (uint32_t)(wu * Q * kTileBytes + 16 * lane), cst);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * rp.j);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (h == 0) {
          const int u = rg + wu;
          if (p.S == 1) {
            const int nl = u * kTileRows + r;
            if (nl < sg.N) sg.y[nl] = __float2half_rn(acc);
          } else {
            st_part(p, p.part + (((size_t)sg.rgoff + u) * p.S + s) * kTileRows + r, ep | __float_as_uint(acc));
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * rp.j);
      }
    }
    r0 = r1;
  }
}

template <int NWC, bool COLW, bool MW2 = false>
__device__ __forceinline__ void consume_run_lut_q(const StreamParams& p, const SegDev& sg, int s, int rga, int re,
                                                  RingPos& rp, uint32_t ring, uint32_t full, uint32_t empty,
                                                  const uint32_t (&cst)[4], int wu, int lane, unsigned long long ep,
                                                  const uint4 xv, int& cur) {
  switch (sg.q) {
    case 1: consume_run_lut<NWC, 1, COLW, MW2>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep, xv, cur); break;
    case 2: consume_run_lut<NWC, 2, COLW, MW2>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep, xv, cur); break;
    case 3: consume_run_lut<NWC, 3, COLW, MW2>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep, xv, cur); break;
    default: consume_run_lut<NWC, 4, COLW, MW2>(p, sg, s, rga, re, rp, ring, full, empty, cst, wu, lane, ep, xv, cur); break;
  }
}

// MINB = 2: registers capped so that two CTAs fit one SM -- with <= 113 KB of shared memory
// the next call's CTA becomes resident (and streams its weights) while this one finishes.
template <int NWC, int MINB, int MW, int BW = 0>
__global__ void __launch_bounds__((NWC + 1) * 32, MINB) lut_stream_kernel(const __grid_constant__ StreamParams p) {
  constexpr int kNT = (NWC + 1) * 32;
  if (threadIdx.x == 0) check_dyn_base();
  trace_at(0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (p.pdl) pdl_launch_dependents();
  const long long G = gridDim.x, W = (long long)p.S * p.Ws, c = blockIdx.x;
  long long wlo = split_point(c, W, G), whi = split_point(c + 1, W, G);
  if (p.one_slice) {   // G = S x cps: CTA c covers part c % cps of slice c / cps
    const unsigned cps = (unsigned)G / (unsigned)p.S, sl = (unsigned)c / cps, sub = (unsigned)c % cps;
    wlo = (long long)sl * p.Ws + split_point(sub, p.Ws, cps);
    whi = (long long)sl * p.Ws + split_point(sub + 1, p.Ws, cps);
  }
  const Pos start = pos_at(p, wlo);
  const Pos end = pos_at(p, whi);
  const uint32_t ring = kDynBase + (uint32_t)p.lut_bytes;
  const uint32_t bars = ring + (uint32_t)(p.nst * p.slot);
  const uint32_t full = bars, empty = bars + 128;
  const uint32_t s_epoch = bars + 256;   // this call's epoch (shared, written once)
  if (tid == 0) {
    for (int j = 0; j < p.nst; ++j) {
      mbar_init(full + 8 * j, 1);
      mbar_init(empty + 8 * j, p.su);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWC) {
    // producer: one thread streams the CTA's runs into the ring, su units per stage
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos rp{0, 0};
      int t = 0;
      for (Pos a = start; before(a, end);) {
        const int re = run_end(p, a, end);
        const SegDev& sg = p.seg[a.g];
        const size_t ub = (size_t)a.s * sg.RG;
        for (int rg = a.rg; rg < re; ++t, rp.next(p.nst)) {
          if (rp.k > 0) mbar_wait(empty + 8 * rp.j, (uint32_t)((rp.k - 1) & 1));
          int n = re - rg < p.su ? re - rg : p.su;
          if (BW == 2 || BW == 3) {   // stages do not cross a row-block boundary (column-wise: one block)
            const int bend = (rg / p.bw_rgb + 1) * p.bw_rgb;
            n = bend - rg < n ? bend - rg : n;
          }
          const uint32_t bp = (uint32_t)(n * sg.q * kTileBytes);
          const uint32_t be = (BW && BW != 5) ? 0u : (uint32_t)(n * sg.q * kTileExps);
          const uint32_t fb = full + 8 * rp.j;
#ifdef SHIFTADD_DEV_TRACE
          if (p.dev_mode & 16) {   // co-roof experiment: no copies (no HBM, no TMA writes)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
            rg += n;
            continue;
          }
#endif
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                       "r"(bp + (BW == 5 ? 2u : 1u) * be) : "memory");
          const uint32_t dst = ring + (uint32_t)(rp.j * p.slot);
          bulk_g2s(dst, sg.planes + (ub + rg) * sg.q * kTileBytes, bp, fb, pol);
          if (!BW || BW == 5) bulk_g2s(dst + (uint32_t)p.slot_planes, sg.exps + (ub + rg) * sg.q * kTileExps, be, fb, pol);
          if (BW == 5) bulk_g2s(dst + (uint32_t)p.slot_exps2, p.exps2 + (ub + rg) * sg.q * kTileExps, be, fb, pol);
          rg += n;
        }
        next_run(p, a, re);
      }
    }
  } else {
    // consumers: x of the (at most two) slices, their LUTs, the epoch, then the ring.  x into
    // L2 before the PDL wait (a hint; the loads come after it)
    if (MW == 1 && tid < 8 && before(start, end) && start.s + (tid >> 2) < p.S)
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.x + (size_t)(start.s + (tid >> 2)) * kTileK + 64 * (tid & 3)));
    if (p.pdl) pdl_wait();
    trace_at(1);
    const int s0 = start.s;
    const bool any = before(start, end);
    const bool two = end.s > s0 && !(end.s == s0 + 1 && end.g == 0 && end.rg == 0);
    if (any) {
      if (tid == 32 && p.S > 1)   // a lane whose x does not gate warp 0
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(s_epoch), "r"((unsigned)(ld_relaxed_u64(p.done) >> 32) + 1u)
                     : "memory");
      if (MW == 1 && (BW < 2 || BW == 5)) {
        const uint64_t pol_keep = policy_evict_last();
        const uint4 xa = ldg_keep(p.x + (size_t)s0 * kTileK + 8 * lane, pol_keep);
        uint4 xb = xa;
        if (two) xb = ldg_keep(p.x + (size_t)(s0 + 1) * kTileK + 8 * lane, pol_keep);
        build_lut<NWC>(xa, 0u, warp, lane);
        if (two) build_lut<NWC>(xb, 128u, warp, lane);
      } else if (MW != 1 && BW != 3) {
        build_lut_mw<NWC, MW>(p, s0, 0, warp, lane);
        if (two && MW < 8) build_lut_mw<NWC, MW>(p, s0 + 1, 1, warp, lane);
      }
    } else if (tid == 32 && p.S > 1) {
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(s_epoch), "r"((unsigned)(ld_relaxed_u64(p.done) >> 32) + 1u)
                   : "memory");
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");   // consumer warps only
    trace_at(2);
#ifdef SHIFTADD_DEV_TRACE
    const long long c2 = clock64();
#endif
    unsigned ep32;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ep32) : "r"(s_epoch) : "memory");
    const unsigned long long ep = (unsigned long long)ep32 << 32;
    const int r = lane >> 1, h = lane & 1;
    const int wu = warp;
    RingPos rp{0, 0};
    if (MW == 1 || BW == 3) {   // (column-wise M = 2: fp16-pair entries at the M = 1 addresses)
      uint32_t cst[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) v |= (4u * (uint32_t)(16 * h + ((4 * k + b + r) & 15))) << (8 * b);
        cst[k] = v;
      }
      const bool skew = p.skew && warp >= NWC / 2;
      int t = 0;
      uint4 xs[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
      if (BW >= 2 && BW <= 3 && MW == 1 && any) {
        const uint64_t pol_keep = policy_evict_last();
        xs[0] = ldg_keep(p.x + (size_t)s0 * kTileK + 8 * lane, pol_keep);
        if (two) xs[1] = ldg_keep(p.x + (size_t)(s0 + 1) * kTileK + 8 * lane, pol_keep);
      }
      int cur = -1;
      for (Pos a = start; before(a, end);) {
        const int re = run_end(p, a, end);
        if (BW == 2 || BW == 3) {
          consume_run_lut_q<NWC, BW == 3, MW == 2>(p, p.seg[a.g], a.s, a.rg, re, rp, ring, full, empty, cst, wu,
                                                   lane, ep, a.s == s0 ? xs[0] : xs[1], cur);
        } else if (BW == 1) {
          if (a.s == s0)
            consume_run_bw_q<0u>(p, p.seg[a.g], a.s, a.rg, re, rp, ring, full, empty, cst, wu, lane, ep);
          else
            consume_run_bw_q<128u>(p, p.seg[a.g], a.s, a.rg, re, rp, ring, full, empty, cst, wu, lane, ep);
        } else if (a.s == s0) {
          consume_run_q<0u, BW == 5>(p, p.seg[a.g], a.s, a.rg, re, rp, t, ring, full, empty, cst, wu, lane, ep, skew);
        } else {
          consume_run_q<128u, BW == 5>(p, p.seg[a.g], a.s, a.rg, re, rp, t, ring, full, empty, cst, wu, lane, ep,
                                       skew);
        }
        next_run(p, a, re);
      }
    } else {
      // column bytes of the 16 steps (2 per constant) and the 64 KB block of the lane's groups
      uint32_t cst[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int g0 = 16 * h + ((2 * k + r) & 15), g1 = 16 * h + ((2 * k + 1 + r) & 15);
        cst[k] = mw_col<MW>(g0) | (mw_col<MW>(g1) << 8) | (mw_hi<MW>(g0) << 16);
      }
      for (Pos a = start; before(a, end);) {
        const int re = run_end(p, a, end);
        if (a.s == s0)
          consume_run_mw_q<mw_slice_base<MW>(0), MW>(p, p.seg[a.g], a.s, a.rg, re, rp, ring, full, empty, cst, wu,
                                                      lane, ep);
        else
          consume_run_mw_q<mw_slice_base<MW>(1), MW>(p, p.seg[a.g], a.s, a.rg, re, rp, ring, full, empty, cst, wu,
                                                      lane, ep);
        next_run(p, a, re);
      }
    }
#ifdef SHIFTADD_DEV_TRACE
    trace_clk(11, c2);
#endif
  }
  trace_at(4);
#ifdef SHIFTADD_DEV_TRACE
  if (g_trace && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_trace[16 * blockIdx.x + 15] = sm;
  }
#endif
  if (p.S == 1) return;

  // a5 owner phase: rows of the flattened row groups [c RGtot / G, (c+1) RGtot / G)
  __syncthreads();
  trace_at(6);

  unsigned ep;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ep) : "r"(s_epoch) : "memory");
  // (G <= 256 and RGtot <= 65536: 32-bit products, so a 32-bit division on the critical path)
  const int og0 = (int)((unsigned)c * (unsigned)p.RGtot / (unsigned)G);
  const int og1 = (int)((unsigned)(c + 1) * (unsigned)p.RGtot / (unsigned)G);
  const int R = (og1 - og0) * kTileRows;
  const int MR = p.M * R;   // (batch row m, output row) pairs owned
  // T threads per row; thread it takes row it % MR (consecutive lanes: consecutive rows of one
  // 128-B line) and slices it / MR, it / MR + T, ... in order, loading <= 8 words at once and
  // re-polling only the stale ones.  The T partial sums of a row then meet in shared memory
  // (the drained ring) and are added in part order: deterministic for a launch shape.
  int T = MR > 0 ? kNT / MR : 1;
  T = T < 1 ? 1 : (T > p.S ? p.S : T);
  float* red = reinterpret_cast<float*>(shiftadd_dyn_smem + p.lut_bytes);   // ring area, drained
  for (int base = 0; base < MR * T; base += kNT) {
    const int it = base + tid;
    if (it < MR * T) {
      const int rl = it % MR, part = it / MR;
      const int m = rl / R, row = rl % R;
      const unsigned long long* pp =
          p.part + (((size_t)m * p.RGtot + og0 + row / kTileRows) * p.S) * kTileRows + (row % kTileRows);
      float sum = 0.f;
      for (int s0 = part; s0 < p.S; s0 += 8 * T) {
        unsigned long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          v[k] = s0 + k * T < p.S ? ld_relaxed_u64(pp + (size_t)(s0 + k * T) * kTileRows) : 0ull;
        unsigned spins = 0;
        for (;;) {
          bool stale = false;
#pragma unroll
          for (int k = 0; k < 8; ++k) stale |= s0 + k * T < p.S && (unsigned)(v[k] >> 32) != ep;
          if (!stale) break;
          if (++spins > (1u << 24)) __trap();   // a non-resident CTA: never hang silently
          __nanosleep(64);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (s0 + k * T < p.S && (unsigned)(v[k] >> 32) != ep)
              v[k] = ld_relaxed_u64(pp + (size_t)(s0 + k * T) * kTileRows);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (s0 + k * T < p.S) sum += __uint_as_float((unsigned)v[k]);
      }
      red[it] = sum;
    }
  }
#ifdef SHIFTADD_DEV_TRACE
  if (tid == 0) trace_at(7);
#endif
  __syncthreads();
  for (int rl = tid; rl < MR; rl += kNT) {
    float sum = red[rl];
    for (int part = 1; part < T; ++part) sum += red[part * MR + rl];
    const int m = rl / R, row = rl % R;
    const int nf = og0 * kTileRows + row;
    const int rgf = nf / kTileRows;
    int g = 0;
    while (g + 1 < p.nseg && p.seg[g + 1].rgoff <= rgf) ++g;
    const int nl = nf - p.seg[g].rgoff * kTileRows;
    if (nl < p.seg[g].N) {
      const __half hv = __float2half_rn(sum);
      if (p.ga.P == 0) {
        p.seg[g].y[(size_t)m * p.ldy + nl] = hv;
      } else {   // NEXT-f3: straight into every rank's gathered y [M][P N] (peer memory), buffer by call parity
        const int b = (int)((*p.ga.epoch + 1u) & 1u);
        const size_t o = ((size_t)m * p.ga.P + p.ga.rank) * p.seg[0].N + nl;
        for (int rr = 0; rr < p.ga.P; ++rr) p.ga.y_peers[b * p.ga.P + rr][o] = hv;
      }
    }
  }
  if (p.ga.P > 0) gather_signal(p.ga);   // (starts with __syncthreads)
  __syncthreads();
  trace_at(5);
  // this CTA's share of the call's 2^32 (see the header comment)
  if (tid == 0) {
    const unsigned long long add = c == 0 ? (1ull << 32) - (unsigned long long)(G - 1) : 1ull;
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p.done), "l"(add) : "memory");
  }
}

}  // namespace

#ifdef SHIFTADD_DEV_TRACE
int g_dev_variant = 0;
void dev_set_variant(int v) { g_dev_variant = v; }
cudaError_t dev_set_trace(void* buf) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(g_trace, &p, sizeof p);
}
#endif

// LUT bytes for entries of MW rows (MW = 1: fp32 entries, two slices; 2, 4: fp16, two
// slices; 8: fp16, one slice)
int stream_lut_bytes(int MW) { return MW <= 2 ? kLutSlab : 2 * kLutSlab; }

int stream_smem_bytes(int qmax, int nst, int su, int MW) {
  return stream_lut_bytes(MW) + nst * su * qmax * (kTileBytes + kTileExps) + kBarBytes;
}

// Ring depth: as many su-unit stages as fit `budget` bytes of shared memory (<= 16).
int stream_stages(int qmax, int budget, int su, int MW) {
  const int slot = su * qmax * (kTileBytes + kTileExps);
  int n = (budget - stream_lut_bytes(MW) - kBarBytes) / slot;
  return n > 16 ? 16 : n;
}

size_t stream_workspace_bytes(int M, int S, int RGtot) {
  if (S <= 1) return 0;   // no split-K: the kernel touches no workspace
  return kPartOff + (size_t)M * S * RGtot * kTileRows * sizeof(unsigned long long);
}

bool stream_shape_ok(int K, int sms) {
  const int S = K / kTileK;
  return S >= 1 && S <= sms;
}

cudaError_t launch_lut_stream(const StreamLaunch& L, cudaStream_t stream) {
  // kernel attributes are per device: set them once on each device that launches
  static std::once_flag once[64];
  static cudaError_t attr_err[64];
  int dev = 0;
  cudaError_t de = cudaGetDevice(&dev);
  if (de != cudaSuccess) return de;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    const int big = 227 * 1024;
    cudaError_t e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lut_stream_kernel<8, 1, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lut_stream_kernel<16, 1, 1, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lut_stream_kernel<8, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
    attr_err[dev] = e;
  });
  if (attr_err[dev] != cudaSuccess) return attr_err[dev];
  if (L.nseg < 1 || L.nseg > kMaxSegments || L.nst < 1 || L.nst > 16 || (L.su != 8 && L.su != 16))
    return cudaErrorInvalidValue;
  StreamParams p = {};
  p.x = L.x;
  p.M = L.M < 1 ? 1 : L.M;
  p.ldx = L.ldx;
  p.ldy = L.ldy;
  p.S = L.K / kTileK;
  const int MW = p.M == 1 ? 1 : p.M == 2 ? 2 : p.M <= 4 ? 4 : 8;
  if (p.M > 8) return cudaErrorInvalidValue;
  p.one_slice = (MW == 8 || (L.one_slice && MW == 1 && !L.exps_bw)) ? 1 : 0;
  p.lut_bytes = stream_lut_bytes(MW);
  p.nseg = L.nseg;
  int rg = 0, w = 0, qmax = 1;
  for (int i = 0; i < L.nseg; ++i) {
    SegDev& d = p.seg[i];
    d.planes = L.seg[i].planes;
    d.exps = L.seg[i].exps;
    d.y = L.seg[i].y;
    d.q = L.seg[i].q;
    d.N = L.seg[i].N;
    d.RG = (d.N + kTileRows - 1) / kTileRows;
    d.rgoff = rg;
    d.woff = w;
    rg += d.RG;
    w += d.q * d.RG;
    qmax = d.q > qmax ? d.q : qmax;
  }
  p.RGtot = rg;
  p.Ws = w;
  if (p.S > 1) {
    char* ws = static_cast<char*>(L.workspace) + kStreamWsOff;
    p.done = reinterpret_cast<unsigned long long*>(ws);
    p.part = reinterpret_cast<unsigned long long*>(ws + (kPartOff - kStreamWsOff));
    p.part_end = p.part + (size_t)p.M * p.S * p.RGtot * kTileRows;
  }
  p.nst = L.nst;
  p.su = L.su;
  p.slot = L.su * qmax * (kTileBytes + kTileExps);
  p.slot_planes = L.su * qmax * kTileBytes;
  p.exps2 = L.exps2;
  p.slot_exps2 = p.slot;
  if (L.exps2) p.slot += L.su * qmax * kTileExps;   // the second-term codes after the exponents
  p.pdl = L.pdl;
  p.exps_bw = L.exps_bw;
  p.ga = L.gather;
  p.bw_rows = L.seg[0].N / 8;
  p.bw_rgb = (L.exps_bw && L.seg[0].N % 128 == 0) ? L.seg[0].N / 128 : 0;
  if (L.exps_bw && L.colwise) p.bw_rgb = (L.seg[0].N + kTileRows - 1) / kTileRows;   // one row block
  if (p.bw_rgb > 0) p.lut_bytes = qmax <= 2 ? kLutSlab : 2 * kLutSlab;
  p.skew = 1;
#ifdef SHIFTADD_DEV_TRACE
  if (g_dev_variant & 2) p.skew = 0;
  p.dev_mode = g_dev_variant & (8 | 16);
#endif
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(L.grid);
#ifdef SHIFTADD_DEV_TRACE
  if ((g_dev_variant & 128) && MW == 1 && !L.exps_bw && p.S > 1 && p.S <= L.grid) {   // experiment: one slice per CTA
    p.one_slice = 1;
    c.gridDim = dim3(p.S * (L.grid / p.S));
  }
#endif
  c.blockDim = dim3((L.half || (L.exps_bw && p.bw_rgb == 0)) ? 9 * 32 : 17 * 32);
  c.dynamicSmemBytes = p.lut_bytes + L.nst * p.slot + kBarBytes;
  c.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = attr;
  c.numAttrs = L.pdl ? 1 : 0;
  if (L.exps_bw && L.colwise && MW == 2) {   // column-wise, two batch rows
    if (L.nseg != 1) return cudaErrorInvalidValue;
    p.lut_bytes = qmax <= 2 ? kLutSlab : 2 * kLutSlab;
    c.dynamicSmemBytes = p.lut_bytes + L.nst * p.slot + kBarBytes;
    return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 2, 3>, p);
  }
  if (L.exps_bw) {
    if (MW != 1 || L.nseg != 1) return cudaErrorInvalidValue;
    // N % 128 == 0: scaled LUTs per (slice, row block); else the per-query scale (8 consumer
    // warps: room for the 8 q scale registers per lane)
    if (L.colwise) return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 1, 3>, p);
    if (p.bw_rgb > 0) return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 1, 2>, p);
    if (L.su != 8) return cudaErrorInvalidValue;
    return cudaLaunchKernelEx(&c, lut_stream_kernel<8, 1, 1, 1>, p);
  }
  if (L.exps2) {   // NEXT-f2: M = 1, one segment
    if (MW != 1 || L.nseg != 1 || L.exps_bw) return cudaErrorInvalidValue;
    c.dynamicSmemBytes = p.lut_bytes + L.nst * p.slot + kBarBytes;
    return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 1, 5>, p);
  }
  if (L.half && MW == 1) return cudaLaunchKernelEx(&c, lut_stream_kernel<8, 2, 1>, p);
  switch (MW) {
    case 1: return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 1>, p);
    case 2: return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 2>, p);
    case 4: return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 4>, p);
    default: return cudaLaunchKernelEx(&c, lut_stream_kernel<16, 1, 8>, p);
  }
}

}  // namespace shiftadd
