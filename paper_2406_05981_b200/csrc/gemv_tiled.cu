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
//    bank-conflict free for any keys.  One PRMT forms key*256 + col*4 -- the per-lane column
//    bytes of 4 steps share one register, and the two zero high bytes come from PRMT's
//    sign-replicate selector -- then one LDS [R + imm] (LUT base and column half are
//    compile-time immediates) and one FADD per key byte.
// a4 shift: the chunk sum (16 lookups, inside one scale group since 128 | g) is scaled by
//    2^e with an exponent-field integer add.
// a5 reduce: lanes h=0,1 combine with one shuffle; split-K partials (one fp32 per slice and
//    row) go to the workspace; per row group an arrival counter (one fence per CTA, then
//    relaxed reds) tells the group's owner CTA -- every CTA owns an equal share of the row
//    groups -- when its S partials are stored; the owner sums them in fixed slice order
//    (several threads per row, one round trip), stores fp16 (RNE) and zeroes the counter.
// PDL: dependents are released at kernel start; the first unit's weights are requested
//    before griddepcontrol.wait, x after it.
#include <mutex>

#include "common.cuh"

namespace shiftadd {
namespace {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// a2: build the 32 LUTs of one 256-k slice into column half `hoff` (0 or 128 bytes) from the
// 8 activations of group `lane` (xv = x[256 s + 8 lane .. +7]).
template <int NW>
__device__ __forceinline__ void build_lut(const uint4 xv, uint32_t hoff, int warp, int lane) {
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
  const uint32_t col = kDynBase + hoff + 4 * lane;
#pragma unroll
  for (int hh = 0; hh < (16 + NW - 1) / NW; ++hh) {
    const int hi = warp + NW * hh;
    if (NW > 16 && hi >= 16) break;
    // hi is warp-dependent: select the signs instead of indexing (keeps it in registers)
    const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                    ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), L[lo] + H);
  }
}

// PRMT selector for step j: byte0 <- column byte (j&3) of cst[j>>2], byte1 <- key byte (j&3)
// of the weight word, bytes 2,3 <- sign of the column byte (< 0x80, so 0x00).
__host__ __device__ constexpr uint32_t step_sel(int j) {
  return ((8u | (4u + (j & 3))) << 12) | ((8u | (4u + (j & 3))) << 8) | ((uint32_t)(j & 3) << 4) |
         (4u + (j & 3));
}

// a3 + a4 for one unit: sum over planes of 2^e * (16 LUT lookups).  LUT byte address of a
// lookup = kDynBase + HOFF + (key << 8 | col*4); the constant part is the LDS immediate.
template <int Q, int MODE, uint32_t HOFF>
__device__ __forceinline__ float unit_dot(const uint4 (&w)[Q], const int (&e)[Q], const uint32_t (&cst)[4]) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    // 4 chains seeded with the first 4 lookups (no 0 + v adds), summed as a fixed tree
    float p[4];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const uint32_t off = prmt(word, cst[j >> 2], step_sel(j));
      const float v = lds_f32(kDynBase + HOFF + off);
      p[j & 3] = j < 4 ? v : p[j & 3] + v;
    }
    const float vt = shift_pow2((p[0] + p[1]) + (p[2] + p[3]), e[i]);
    acc = i == 0 ? vt : acc + vt;
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

struct SegCtx {
  const uint4* planes;
  const int8_t* exps;
  int N, S, Npad;
  long long rg_base;   // first unit of the slice
  __half* y;
  float* partial;
  unsigned* cnt;       // per-row-group arrival counters
  int unit_release;    // 1: each warp releases its unit's arrival right after storing it
};

template <int Q, int MODE>
__device__ __forceinline__ void emit(float acc, const SegCtx& c, int s, long long u, int r, int h) {
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  const int rg = (int)(u - c.rg_base);
  const int n = rg * kTileRows + r;
  if (h == 0) {
    if (c.S == 1) { if (n < c.N) c.y[n] = __float2half_rn(acc); }
    else c.partial[(size_t)s * c.Npad + n] = acc;
  }
  if (c.unit_release && c.S > 1 && MODE != 3) {
    // the warp's 16 stores, then one release-add by lane 0 (cumulative after __syncwarp)
    __syncwarp();
    if (r == 0 && h == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c.cnt + rg) : "memory");
  }
}

// Register budget and pipeline depth.  A unit in flight costs Q x (4 + 1) registers; the
// rest of the loop needs ~36.  D units per warp are kept in flight (a ring of D register
// buffers), which is what hides the HBM latency at ~1-2 us under load.
__host__ __device__ constexpr int ring_depth(int Q, int REGS) {
  return (REGS - 36) / (5 * Q) < 1 ? 1 : ((REGS - 36) / (5 * Q) > 8 ? 8 : (REGS - 36) / (5 * Q));
}

// Process the units [uu, seg_end) (warp stride NW) of one slice; ring slot k holds unit
// uu + k*NW on entry (loaded by the caller before the LUT build).
template <int Q, int NW, int MODE, uint32_t HOFF, int D>
__device__ __forceinline__ void run_segment(const SegCtx& c, int s, long long uu, long long seg_end,
                                            int lane, uint64_t pol, uint4 (&w)[D][Q], int (&e)[D][Q]) {
  const int r = lane >> 1, h = lane & 1;
  uint32_t cst[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) v |= (4u * (uint32_t)(16 * h + ((4 * k + b + r) & 15))) << (8 * b);
    cst[k] = v;
  }
  for (long long base = uu; base < seg_end; base += (long long)D * NW) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const long long cur = base + (long long)k * NW;
      if (cur < seg_end) {
        const float acc = (MODE == 3) ? unit_xor<Q>(w[k], e[k]) : unit_dot<Q, MODE, HOFF>(w[k], e[k], cst);
        const long long nxt = cur + (long long)D * NW;
        if (nxt < seg_end) load_unit<Q>(c.planes, c.exps, nxt, lane, pol, w[k], e[k]);
        emit<Q, MODE>(acc, c, s, cur, r, h);
      }
    }
  }
}

// Dynamic variant of run_segment for slice-aligned grids (kc CTAs per slice): the slice's RG
// units are a queue.  Ring slot k of warp gw = p*NW + w starts on local unit gw + k*kc*NW
// (static prefix of kc*NW*D units); afterwards each refill takes the next unit from the
// slice's claim counter.  Every slot's claim is issued one ring cycle before its result is
// needed (lane 0 holds it; it is broadcast when the slot is refilled), so the atomic's
// latency hides behind D units of work.  SM-to-SM speed differences then even out inside the
// slice group.  Returns the number of units this warp processed.
template <int Q, int NW, int MODE, int D>
__device__ __forceinline__ int run_dynamic(const SegCtx& c, int s, int RG, int kc, int gw, int lane,
                                           uint64_t pol, unsigned* claim, uint4 (&w)[D][Q], int (&e)[D][Q]) {
  const int r = lane >> 1, h = lane & 1;
  uint32_t cst[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) v |= (4u * (uint32_t)(16 * h + ((4 * k + b + r) & 15))) << (8 * b);
    cst[k] = v;
  }
  const int base_dyn = kc * NW * D;
  int cur[D];
  unsigned pend[D];   // lane 0: pending claim for the slot's next refill
#pragma unroll
  for (int k = 0; k < D; ++k) {
    cur[k] = gw + k * kc * NW;
    pend[k] = 0u;
    if (lane == 0 && cur[k] < RG) pend[k] = atomicAdd(claim, 1u);
  }
  int done = 0;
  bool any = true;
  while (any) {
    any = false;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (cur[k] < RG) {
        const float acc = (MODE == 3) ? unit_xor<Q>(w[k], e[k]) : unit_dot<Q, MODE, 0u>(w[k], e[k], cst);
        const int unit = cur[k];
        const int nxt = base_dyn + (int)__shfl_sync(0xffffffffu, pend[k], 0);
        cur[k] = nxt;
        if (nxt < RG) {
          load_unit<Q>(c.planes, c.exps, c.rg_base + nxt, lane, pol, w[k], e[k]);
          if (lane == 0) pend[k] = atomicAdd(claim, 1u);
          any = true;
        }
        emit<Q, MODE>(acc, c, s, c.rg_base + unit, r, h);
        ++done;
      }
    }
  }
  return done;
}

// MODE: 0 = product; 3 = loads only; 4 = product + per-CTA phase timestamps written after the
// partials in the workspace.  Modes 3-4 are internal experiments (SHIFTADD_EXP).
template <int Q, int NW, int REGS, int MODE>
__global__ void __launch_bounds__(NW * 32) __maxnreg__(REGS)
gemv_tiled_kernel(const __half* __restrict__ x, const uint4* __restrict__ planes,
                  const int8_t* __restrict__ exps, int N, int S, int RG, long long U,
                  __half* __restrict__ y, float* __restrict__ partial, unsigned* __restrict__ cnt,
                  int pdl, int pre_wait, int pre_build, int unit_release, int dyn_kc) {
  constexpr int D = ring_depth(Q, REGS);
  if (threadIdx.x == 0) check_dyn_base();
  unsigned long long* trace = (MODE >= 4) ? reinterpret_cast<unsigned long long*>(
      partial + (size_t)S * RG * kTileRows) + (size_t)blockIdx.x * 16 : nullptr;
  if (MODE >= 4 && threadIdx.x == 0) trace[0] = gtimer();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long G = gridDim.x;
  // u0 = floor(c*U/G) in 32-bit arithmetic (c*U = c*(U/G)*G + c*(U%G), c*(U%G) < G*G)
  const unsigned Uu = (unsigned)U, Gu = (unsigned)G, qq = Uu / Gu, rr = Uu % Gu, cb = blockIdx.x;
  const long long u0 = (long long)(cb * qq + (cb * rr) / Gu);
  const long long u1 = (long long)((cb + 1) * qq + ((cb + 1) * rr) / Gu);
  const int Npad = RG * kTileRows;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  // All CTAs of this grid are resident once each has passed this point, so the dependent
  // grid may launch now and start fetching its own weights while this one works.
  if (pdl) pdl_launch_dependents();

  SegCtx c{planes, exps, N, S, Npad, 0, y, partial, cnt, unit_release};
  uint4 w[D][Q];
  int e[D][Q];
  long long u = u0;
  int seg = 0;
  // Dynamic mode (slice-aligned grid, dyn_kc CTAs per slice): one segment, units claimed.
  int* dyn_total = reinterpret_cast<int*>(shiftadd_dyn_smem + kLutBytes);
  const int dyn_s = dyn_kc > 0 ? (int)(cb / (unsigned)dyn_kc) : 0;
  if (dyn_kc > 0) {
    const int gw = (int)(cb % (unsigned)dyn_kc) * NW + warp;
    if (tid == 0) *dyn_total = 0;
    c.rg_base = (long long)dyn_s * RG;
    const __half* xs = x + (size_t)dyn_s * kTileK + 8 * lane;
    if (pdl) pdl_wait();
    const uint4 xv = ldg_keep(xs, pol_keep);
    if (MODE >= 4 && tid == 0) trace[8] = gtimer() + (xv.x & 0u);
    if (MODE != 3) build_lut<NW>(xv, 0u, warp, lane);
    if (MODE >= 4 && tid == 0) trace[9] = gtimer();
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int lu = gw + k * dyn_kc * NW;
      if (lu < RG) load_unit<Q>(planes, exps, c.rg_base + lu, lane, pol_stream, w[k], e[k]);
    }
    __syncthreads();
    if (MODE >= 4 && tid == 0) trace[1] = gtimer();
    const int done = run_dynamic<Q, NW, MODE, D>(c, dyn_s, RG, dyn_kc, gw, lane, pol_stream, cnt + dyn_s, w, e);
    if (lane == 0) atomicAdd(dyn_total, done);
    u = u1;
    seg = 1;
  }
  while (u < u1) {
    const int s = (int)((unsigned)u / (unsigned)RG);
    const long long seg_end = min(u1, (long long)(s + 1) * RG);
    const long long uu = u + warp;
    uint4 xv;
    const __half* xs = x + (size_t)s * kTileK + 8 * lane;
    // Ring slots k < early are requested before the LUT build, the rest right after this
    // warp's share of it: LDG traffic in flight delays the build's shared-memory stores, and
    // the build is on the critical path.  Weights never depend on the upstream kernel, x may
    // (it is its output), so under PDL the early slots go out before griddepcontrol.wait.
    const int early = (seg == 0 && pdl) ? pre_wait : pre_build;
    if (seg == 0 && pdl) {
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (k < early && uu + (long long)k * NW < seg_end)
          load_unit<Q>(planes, exps, uu + (long long)k * NW, lane, pol_stream, w[k], e[k]);
      pdl_wait();
      xv = ldg_keep(xs, pol_keep);
    } else {
      xv = ldg_keep(xs, pol_keep);
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (k < early && uu + (long long)k * NW < seg_end)
          load_unit<Q>(planes, exps, uu + (long long)k * NW, lane, pol_stream, w[k], e[k]);
    }
    if (MODE >= 4 && tid == 0 && seg == 0) trace[8] = gtimer() + (xv.x & 0u);   // x arrived
    if (MODE != 3) build_lut<NW>(xv, (seg & 1) ? 128u : 0u, warp, lane);
    if (MODE >= 4 && tid == 0 && seg == 0) trace[9] = gtimer();                 // own part built
#pragma unroll
    for (int k = 0; k < D; ++k)
      if (k >= early && uu + (long long)k * NW < seg_end)
        load_unit<Q>(planes, exps, uu + (long long)k * NW, lane, pol_stream, w[k], e[k]);
    __syncthreads();
    if (MODE >= 4 && tid == 0 && seg == 0) trace[1] = gtimer();
    c.rg_base = (long long)s * RG;
    if (seg & 1) run_segment<Q, NW, MODE, 128u, D>(c, s, uu, seg_end, lane, pol_stream, w, e);
    else run_segment<Q, NW, MODE, 0u, D>(c, s, uu, seg_end, lane, pol_stream, w, e);
    u = seg_end;
    ++seg;
  }
  if (MODE >= 4) {
    __syncthreads();
    if (tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[2] = gtimer();
      trace[5] = smid;
      trace[6] = (unsigned long long)seg;
      trace[7] = (unsigned long long)u0;
    }
  }
  if (S == 1 || MODE == 3) return;

  // Dynamic mode: one arrival per CTA on its slice's done word (units processed + 2^20, so
  // the word also counts the CTAs that finished claiming); every owner waits until each
  // slice shows RG units from all dyn_kc CTAs, then finalizes as below.  The last CTA to
  // depart resets the claim / done / departure words.
  unsigned* const dyn_done = cnt + 1024;
  unsigned* const dyn_dep = cnt + 2048;
  if (dyn_kc > 0) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(dyn_done + dyn_s),
                   "r"((unsigned)*dyn_total + (1u << 20)) : "memory");
    }
    const unsigned target = (unsigned)RG + ((unsigned)dyn_kc << 20);
    for (int t = tid; t < S; t += NW * 32)
      while (ld_acquire_gpu(dyn_done + t) != target) {
      }
    __syncthreads();
  }
  // a5: deterministic split-K reduction, balanced over the grid.  CTA c owns the final sums
  // of row groups [c*RG/G, (c+1)*RG/G) (whole groups, so every counter has one owner).  Per
  // row group an arrival counter cnt[rg] counts the (slice, rg) units whose partials are
  // stored: each CTA fences once after its main loop (cumulative over its threads' stores,
  // after bar.sync) and then adds 1 per unit with a relaxed red -- no grid-wide barrier, no
  // single hot address.  An owner waits (one acquire poller per row group) only for its own
  // counters, sums the S partials of each row in a fixed order, stores fp16 and zeroes the
  // counters.  All CTAs are co-resident (gridDim <= #SMs x CTAs-per-SM the kernel fits), so
  // the wait always completes.  (Measured alternatives: a red/acquire grid
  // barrier, and polling self-validating partial words, were both slower on B200.)
  const int own0 = (int)(((long long)blockIdx.x * RG) / G);
  const int own1 = (int)(((long long)(blockIdx.x + 1) * RG) / G);
  const int n0 = own0 * kTileRows;
  const int R = (own1 - own0) * kTileRows;
  if (dyn_kc == 0) {
    if (!unit_release) {
      __syncthreads();
      if (tid == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");   // release: the CTA's partials before its arrivals
      __syncthreads();
      for (long long uq = u0 + tid; uq < u1; uq += NW * 32)
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + ((unsigned)uq % (unsigned)RG)) : "memory");
    }
    for (int rg = own0 + tid; rg < own1; rg += NW * 32)
      while (ld_acquire_gpu(cnt + rg) < (unsigned)S) {
      }
    __syncthreads();
  }
  if (MODE >= 4 && tid == 0) trace[3] = gtimer();
  // T threads per row (power of two <= 32, <= S): each sums its strided share of the S
  // partials (up to 16 loads in flight per thread), then a fixed butterfly combines them.
  int T = 1;
  while (T < 32 && 2 * T <= S && (R * 2 * T <= NW * 32 || S > 16 * T)) T *= 2;
  const int items = R * T;
  const int items_pad = (items + 31) & ~31;
  for (int it = tid; it < items_pad; it += NW * 32) {
    const bool live = it < items;
    const int n = n0 + it / T;
    const int part = it & (T - 1);
    float sum = 0.f;
    if (live) {
      const float* p = partial + n;
      for (int s = part; s < S; s += 16 * T) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
          v[k] = (MODE != 5 && s + k * T < S) ? __ldcg(p + (size_t)(s + k * T) * Npad) : 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) sum += v[k];
      }
    }
    for (int off = T >> 1; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (live && part == 0 && n < N) y[n] = __float2half_rn(sum);
  }
  if (MODE >= 4) {
    __syncthreads();
    if (tid == 0) trace[4] = gtimer();
  }
  if (dyn_kc == 0) {
    for (int rg = own0 + tid; rg < own1; rg += NW * 32) cnt[rg] = 0u;   // for the next call
  } else {
    __syncthreads();
    if (tid == 0 && atomicAdd(dyn_dep, 1u) == (unsigned)G - 1) {
      for (int t = 0; t < S; ++t) {
        cnt[t] = 0u;
        dyn_done[t] = 0u;
      }
      *dyn_dep = 0u;
    }
  }
}

// Launch configurations (warps per CTA, register cap).  Variant 0 is the product default;
// the others exist for measurement (SHIFTADD_VARIANT) and are documented in DESIGN.md.
struct Variant {
  int nw, regs;
};
constexpr Variant kVariants[] = {{16, 128}, {8, 128}, {16, 64}, {24, 80}};

struct Cfg {
  int variant;     // index into kVariants
  int per_sm;      // CTAs per SM; 0 = choose by problem size
  int mode;        // experiment mode (0 = product)
  int no_align;    // 1 = plain linear split (experiment)
  int pre_wait;    // ring slots requested before griddepcontrol.wait (PDL)
  int pre_build;   // ring slots requested before the LUT build (no PDL)
  int align_min;   // min % of CTA slots a slice-aligned grid must keep
  int unit_release;  // split-K arrival: 1 = per unit by each warp, 0 = once per CTA at the end
  int dyn;           // 1 = dynamic unit claiming inside slice groups (slice-aligned grids)
};

// Fixed at the measured defaults: variant 2 (16 warps x 64 registers), CTAs per
// SM by problem size, slice-aligned grids keeping >= 85% of the slots.  No environment is read.
constexpr Cfg kCfg{2, 0, 0, 0, 0, 0, 85, 0, 0};

const Cfg& cfg() { return kCfg; }

constexpr int kDynSmem = kLutBytes + 16;  // 64 KB LUT + the dynamic mode's unit count

template <int Q, int NW, int REGS, int MODE>
cudaError_t launch_k(const GemmArgs& a, const LaunchPlan& p) {
  const cudaError_t attr_err = once_per_device([] {
    cudaError_t attr_err = cudaSuccess;
    attr_err = cudaFuncSetAttribute(gemv_tiled_kernel<Q, NW, REGS, MODE>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
    return attr_err;
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const long long U = (long long)S * RG;
  unsigned* sync = S > 1 ? reinterpret_cast<unsigned*>(a.workspace) : nullptr;
  float* partial = S > 1 ? reinterpret_cast<float*>(reinterpret_cast<char*>(a.workspace) + kPartOff) : nullptr;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  const int dyn_kc = (cfg().dyn && S > 1 && S <= 1024 && p.grid % S == 0 && p.grid / S >= 2) ? p.grid / S : 0;

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
  return cudaLaunchKernelEx(&c, gemv_tiled_kernel<Q, NW, REGS, MODE>, a.x,
                            reinterpret_cast<const uint4*>(a.planes), a.exps, a.N, S, RG, U, a.y, partial, sync,
                            pdl, cfg().pre_wait, cfg().pre_build, cfg().unit_release, dyn_kc);
}

template <int Q, int V>
cudaError_t launch_v(const GemmArgs& a, const LaunchPlan& p) {
  constexpr int NW = kVariants[V].nw, REGS = kVariants[V].regs;
  return launch_k<Q, NW, REGS, 0>(a, p);
}

template <int Q>
cudaError_t launch_q(const GemmArgs& a, const LaunchPlan& p) {
  switch (cfg().variant) {
    case 1: return launch_v<Q, 1>(a, p);
    case 2: return launch_v<Q, 2>(a, p);
    case 3: return launch_v<Q, 3>(a, p);
    default: return launch_v<Q, 0>(a, p);
  }
}


// ------------------------------------------------------------------------------------------
// TMA-ring variant for large layers (kernel id 4).  Same units, LUTs, lookup loop, shift and
// split-K reduction as gemv_tiled_kernel; what changes is how the weights reach the SM.  The
// register-ring kernel keeps at most D units per warp in flight (48 KB per SM at q = 3 with
// 64 registers), which caps a long layer at bytes-in-flight / HBM latency.  Here one producer
// thread streams the CTA's contiguous chunk of units with bulk copies (cp.async.bulk, the TMA
// engine) into a ring of NST shared-memory stages of 16 units (~157 KB in flight at q = 3),
// completing on a per-stage "full" mbarrier; 16 consumer warps take one unit each per stage
// (LDS.128 of the lane's 16 key bytes per plane: conflict-free), look it up and release the
// stage on its "empty" mbarrier.  One CTA per SM, grid = #SMs; a chunk spans at most two
// slices (S < gridDim), whose LUTs are both built up front in the two column halves.
constexpr int kStreamNWC = 16;     // consumer warps
constexpr int kStageUnits = 16;    // units per stage: one per consumer warp

template <int Q>
struct StreamSmem {
  static constexpr int lut = kLutBytes;
  static constexpr int stage_planes = kStageUnits * Q * kTileBytes;
  static constexpr int stage_exps = kStageUnits * Q * kTileExps;
  static constexpr int stage = stage_planes + stage_exps;
  static constexpr int budget = 227 * 1024 - lut - 256;
  static constexpr int nst = budget / stage > 8 ? 8 : budget / stage;
  static constexpr int ring = nst * stage;
  static constexpr int bars = 128;   // full[8] at +0, empty[8] at +64
  static constexpr int total = lut + ring + bars;
};

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ int lds_s8(uint32_t addr) {
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

template <int Q>
__global__ void __launch_bounds__((kStreamNWC + 1) * 32, 1)
gemv_stream_kernel(const __half* __restrict__ x, const uint8_t* __restrict__ planes,
                   const int8_t* __restrict__ exps, int N, int S, int RG, long long U,
                   __half* __restrict__ y, float* __restrict__ partial, unsigned* __restrict__ cnt, int pdl,
                   int npre, unsigned long long* __restrict__ trace, int nown) {
  using SM = StreamSmem<Q>;
  unsigned long long* tr = trace ? trace + 16 * blockIdx.x : nullptr;   // dev trace
  if (tr && threadIdx.x == 0) tr[0] = gtimer();
  constexpr int NST = SM::nst;
  constexpr int NWC = kStreamNWC;
  if (threadIdx.x == 0) check_dyn_base();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (NWC + 1) * 32;
  const long long G = gridDim.x;
  const unsigned Uu = (unsigned)U, Gu = (unsigned)G, qq = Uu / Gu, rr = Uu % Gu, cb = blockIdx.x;
  const long long u0 = (long long)(cb * qq + (cb * rr) / Gu);
  const long long u1 = (long long)((cb + 1) * qq + ((cb + 1) * rr) / Gu);
  const int Npad = RG * kTileRows;
  const uint32_t ring = kDynBase + SM::lut;
  const uint32_t full = ring + SM::ring, empty = full + 64;
  if (tid == 0) {
    for (int j = 0; j < NST; ++j) {
      mbar_init(full + 8 * j, 1);
      mbar_init(empty + 8 * j, NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (pdl) pdl_launch_dependents();
  const int nstages = (int)((u1 - u0 + kStageUnits - 1) / kStageUnits);

  if (warp == NWC) {
    // producer: stages [0, npre) before griddepcontrol.wait (weights never depend on the
    // upstream kernel; more would only queue x behind them), the rest as slots free up
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < nstages; ++t) {
        if (t == npre && pdl) pdl_wait();
        const int j = t % NST;
        if (t >= NST) mbar_wait(empty + 8 * j, (uint32_t)((t / NST - 1) & 1));
        const long long ub = u0 + (long long)t * kStageUnits;
        const int n = (int)min((long long)kStageUnits, u1 - ub);
        const uint32_t bp = (uint32_t)(n * Q * kTileBytes), be = (uint32_t)(n * Q * kTileExps);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * j), "r"(bp + be)
                     : "memory");
        bulk_g2s(ring + j * SM::stage, planes + (size_t)ub * Q * kTileBytes, bp, full + 8 * j, pol);
        bulk_g2s(ring + j * SM::stage + SM::stage_planes, exps + (size_t)ub * Q * kTileExps, be, full + 8 * j, pol);
      }
    }
  } else {
    // consumers: the LUTs of the (at most two) slices of the chunk, then the ring
    const int s_first = (int)((unsigned)u0 / (unsigned)RG);
    const int s_last = u1 > u0 ? (int)((unsigned)(u1 - 1) / (unsigned)RG) : s_first;
    const uint64_t pol_keep = policy_evict_last();
    if (pdl) pdl_wait();
    if (tr && tid == 0) tr[1] = gtimer();
    const uint4 xa = ldg_keep(x + (size_t)s_first * kTileK + 8 * lane, pol_keep);
    uint4 xb = xa;
    if (s_last != s_first) xb = ldg_keep(x + (size_t)s_last * kTileK + 8 * lane, pol_keep);
    build_lut<NWC>(xa, 0u, warp, lane);
    if (s_last != s_first) build_lut<NWC>(xb, 128u, warp, lane);
    asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");   // consumer warps only
    if (tr && tid == 0) tr[2] = gtimer();
    const int r = lane >> 1, h = lane & 1;
    uint32_t cst[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) v |= (4u * (uint32_t)(16 * h + ((4 * k + b + r) & 15))) << (8 * b);
      cst[k] = v;
    }
    SegCtx c{nullptr, nullptr, N, S, Npad, 0, y, partial, cnt, 0};
    for (int t = 0; t < nstages; ++t) {
      const int j = t % NST;
      const long long u = u0 + (long long)t * kStageUnits + warp;
      mbar_wait(full + 8 * j, (uint32_t)((t / NST) & 1));
      if (tr && tid == 0 && t == 0) tr[3] = gtimer();
      if (u < u1) {
        uint4 w[Q];
        int e[Q];
        const uint32_t sp = ring + j * SM::stage + warp * Q * kTileBytes + 16 * lane;
        const uint32_t se = ring + j * SM::stage + SM::stage_planes + warp * Q * kTileExps + lane;
#pragma unroll
        for (int i = 0; i < Q; ++i) w[i] = lds_u4(sp + i * kTileBytes);
#pragma unroll
        for (int i = 0; i < Q; ++i) e[i] = lds_s8(se + i * kTileExps);
        const int s = (int)((unsigned)u / (unsigned)RG);
        const float acc = s == s_first ? unit_dot<Q, 0, 0u>(w, e, cst) : unit_dot<Q, 0, 128u>(w, e, cst);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * j);   // the unit's bytes are consumed
        c.rg_base = (long long)s * RG;
        emit<Q, 0>(acc, c, s, u, r, h);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * j);
      }
    }
  }
  if (tr && tid == 0) tr[4] = gtimer();
  if (S == 1) return;
  // a5 as in gemv_tiled_kernel: one fence per CTA, relaxed arrivals per unit, owners poll
  // their row groups' counters, sum the S partials in slice order, store fp16, re-arm.
  // Only the first nown CTAs own row groups: the others leave right after their arrivals, and
  // their SMs take the next kernel's CTAs (PDL), whose weight streams then overlap this
  // kernel's reduction.
  const bool owner = (int)blockIdx.x < nown;
  const int own0 = owner ? (int)(((long long)blockIdx.x * RG) / nown) : 0;
  const int own1 = owner ? (int)(((long long)(blockIdx.x + 1) * RG) / nown) : 0;
  const int n0 = own0 * kTileRows;
  const int R = (own1 - own0) * kTileRows;
  __syncthreads();
  if (tid == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");   // release: the CTA's partials before its arrivals
  __syncthreads();
  for (long long uq = u0 + tid; uq < u1; uq += NT)
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + ((unsigned)uq % (unsigned)RG)) : "memory");
  if (tr && tid == 0) tr[5] = gtimer();
  if (!owner) return;
  for (int rg = own0 + tid; rg < own1; rg += NT)
    while (ld_acquire_gpu(cnt + rg) < (unsigned)S) {
    }
  __syncthreads();
  if (tr && tid == 0) tr[6] = gtimer();
  int T = 1;
  while (T < 32 && 2 * T <= S && (R * 2 * T <= NT || S > 16 * T)) T *= 2;
  const int items = R * T;
  const int items_pad = (items + 31) & ~31;
  for (int it = tid; it < items_pad; it += NT) {
    const bool live = it < items;
    const int n = n0 + it / T;
    const int part = it & (T - 1);
    float sum = 0.f;
    if (live) {
      const float* p = partial + n;
      for (int s = part; s < S; s += 16 * T) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = s + k * T < S ? __ldcg(p + (size_t)(s + k * T) * Npad) : 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) sum += v[k];
      }
    }
    for (int off = T >> 1; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (live && part == 0 && n < N) y[n] = __float2half_rn(sum);
  }
  for (int rg = own0 + tid; rg < own1; rg += NT) cnt[rg] = 0u;   // for the next call
  if (tr) {
    __syncthreads();
    if (tid == 0) tr[7] = gtimer();
  }
}

template <int Q>
cudaError_t launch_stream_q(const GemmArgs& a, const LaunchPlan& p) {
  const cudaError_t attr_err = once_per_device([] {
    cudaError_t attr_err = cudaSuccess;
    attr_err = cudaFuncSetAttribute(gemv_stream_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    StreamSmem<Q>::total);
    return attr_err;
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const long long U = (long long)S * RG;
  unsigned* sync = reinterpret_cast<unsigned*>(a.workspace);
  float* partial = reinterpret_cast<float*>(reinterpret_cast<char*>(a.workspace) + kPartOff);
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  constexpr int npre = 1;   // stages requested before griddepcontrol.wait (measured best)
  unsigned long long* trace = nullptr;
  const int nown = p.grid;
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
  return cudaLaunchKernelEx(&c, gemv_stream_kernel<Q>, a.x, a.planes, a.exps, a.N, S, RG, U, a.y, partial, sync,
                            pdl, npre, trace, nown);
}

int stream_smem(int q) {
  switch (q) {
    case 1: return StreamSmem<1>::total;
    case 2: return StreamSmem<2>::total;
    case 3: return StreamSmem<3>::total;
    default: return StreamSmem<4>::total;
  }
}

}  // namespace

LaunchPlan plan_gemv_tiled(int N, int K, int q, int sms) {
  (void)q;
  const long long S = K / kTileK;
  const long long RG = (N + kTileRows - 1) / kTileRows;
  const long long U = S * RG;
  // Default (measured): 16-warp CTAs capped at 64 registers.  Small problems
  // run one CTA per SM, leaving room for the next call's CTAs under PDL; problems with >= 64
  // units per SM run two (32 warps per SM keep more loads in flight).
  int per_sm = cfg().per_sm;
  if (per_sm == 0) per_sm = (U >= 64LL * sms && kVariants[cfg().variant].nw * 32 * kVariants[cfg().variant].regs <= 32768) ? 2 : 1;
  const long long want = (long long)sms * per_sm;
  long long grid = U < want ? U : want;
  // Slice-aligned split: with gridDim a multiple of S every CTA's chunk lies in one slice
  // (one LUT build, no mid-chunk barrier).  Taken when it idles <= 15% of the CTA slots.
  if (grid == want && S > 1 && !cfg().no_align) {
    const long long k = want / S;
    if (k >= 1 && S * k * 100 >= want * cfg().align_min) grid = S * k;
  }
  return LaunchPlan{(int)grid, kVariants[cfg().variant].nw * 32, kDynSmem, 1};
}

// Large layers (more than ~64 units per SM, chunks within two slices) stream through the
// TMA ring (kernel 4); SHIFTADD_STREAM=0 keeps them on the register-ring kernel.
bool stream_applicable(int N, int K, int q, int sms) {
  if (q < 1 || q > 4) return false;
  const long long S = K / kTileK;
  const long long RG = (N + kTileRows - 1) / kTileRows;
  return S > 1 && S < sms && S * RG >= 64LL * sms;
}

LaunchPlan plan_gemv_stream(int N, int K, int q, int sms) {
  (void)N; (void)K;
  return LaunchPlan{sms, (kStreamNWC + 1) * 32, stream_smem(q), 4};
}

size_t workspace_gemv_tiled(int N, int K) {
  const size_t S = K / kTileK;
  if (S <= 1) return 0;
  const size_t RG = (N + kTileRows - 1) / kTileRows;
  return kPartOff + S * RG * kTileRows * sizeof(float);
}

cudaError_t launch_gemv_tiled(const GemmArgs& a, const LaunchPlan& p) {
  if (p.kernel == 4) {
    switch (a.q) {
      case 1: return launch_stream_q<1>(a, p);
      case 2: return launch_stream_q<2>(a, p);
      case 3: return launch_stream_q<3>(a, p);
      case 4: return launch_stream_q<4>(a, p);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.q) {
    case 1: return launch_q<1>(a, p);
    case 2: return launch_q<2>(a, p);
    case 3: return launch_q<3>(a, p);
    case 4: return launch_q<4>(a, p);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace shiftadd
