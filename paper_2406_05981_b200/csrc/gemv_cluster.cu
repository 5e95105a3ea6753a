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
//    the band) with st.async stores that complete transaction bytes on the owner's
//    mbarrier; each owner waits for exactly its bytes, sums ranks 0..C-1 in that order and
//    stores fp16 (RNE).  Deterministic; no workspace, no global atomics, no cluster-wide
//    barrier at the end.
//  * The grid is (max co-resident clusters) x C, from cudaOccupancyMaxActiveClusters, so it
//    never needs a second wave.
// In a cluster a CTA's shared addresses carry its rank in bits 24+ (a rank-0 address used by
// rank 1 is an illegal instruction -- measured), so the PRMT that forms a lookup address
// takes byte 3 = rank from the constant registers (see step_sel_c).
#include <mutex>

#include "common.cuh"

namespace shiftadd {
namespace {

constexpr int kMaxSc = 4;                 // resident LUT slots (slices per CTA)
constexpr int kMaxC = 8;                  // portable cluster size
constexpr int kMaxCColw = 16;             // column-wise kernel: non-portable clusters of <= 16
constexpr int kMaxRGb = 128;              // row groups per band
constexpr int kMaxRGbColw = 4 * kMaxRGb;  // column-wise: one slice per CTA

// Shared-memory map of a variant with SCM LUT slots: LUT slabs, staged x, receive buffer
// recv[slice s][row of the owner's chunk] (every (slice, row) partial sum of the owner's rows,
// pushed by the CTA that streamed it), the owner's receive mbarrier.
template <int SCM>
struct Smem {
  static constexpr int lut = SCM <= 2 ? kLutBytes : 2 * kLutBytes;
  static constexpr int xstage = SCM * kTileK * 2;
  // chunks are whole row groups: S * chunk <= SCM * (RGb + C) * 16 rows (regular variants);
  // the column-wise kernel (4-slot map, one slice per CTA) has S = C and bands up to 4x taller
  static constexpr int recv_rows = SCM * (kMaxRGb + kMaxC) * kTileRows;
  static constexpr int recv_rows_colw = (kMaxRGbColw + kMaxCColw) * kTileRows;
  static constexpr int recv = 4 * (SCM == 4 && recv_rows_colw > recv_rows ? recv_rows_colw : recv_rows);
  static constexpr int part = SCM * kMaxRGb * kTileRows * 4;   // push-at-end mode: part[t][row]
  static constexpr int mbar = 16;   // the owner's receive mbarrier (8-byte aligned)
  static constexpr int total = lut + xstage + recv + part + mbar;
};
static_assert(Smem<2>::total <= 113 * 1024, "two half-SM CTAs must fit one SM");

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
// Split cluster barrier: arrive early (relaxed; a preceding fence supplies the release),
// wait (acquire) right before the first DSMEM access.
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
// Owner-side receive barrier: one arrival (the owner's own expect_tx) + the bytes its peers
// push with st.async ... complete_tx.
__device__ __forceinline__ void mbar_init_expect(uint32_t bar, uint32_t tx_bytes) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx_bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity0(uint32_t bar) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar) : "memory");
  } while (!done);
}
// x staging by the bulk-copy engine (TMA, 1-D): `bytes` from global `src` into this CTA's
// shared `dst`, completing on `xbar` (already armed with expect_tx).  It does not queue behind
// the LSU's weight loads.
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_load_x(uint32_t dst, const void* src, uint32_t bytes, uint32_t xbar,
                                            uint64_t pol, bool expect = true) {
  smem_check(dst, bytes);
  smem_check(xbar, 8);
  if (expect)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(xbar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(xbar), "l"(pol) : "memory");
}

// Asynchronous 4-byte store into CTA `rank`'s shared memory that completes 4 transaction
// bytes on that CTA's mbarrier (both addresses given in this CTA's window, mapped here).
__device__ __forceinline__ void st_async_f32(uint32_t local_addr, uint32_t local_bar, uint32_t rank, float v) {
  smem_check(local_addr, 4);
  smem_check(local_bar, 8);
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(local_bar), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
               "r"(__float_as_uint(v)), "r"(rb) : "memory");
}


// a2 from staged x: LUT slot at `slot_base` (slab base + 0 / 128 B half) from the 256
// activations at shared address xaddr; warp = hi nibble, lane = 8-k group (column).
template <int NW>
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
  float L[16];
#pragma unroll
  for (int lo = 0; lo < 16; ++lo) L[lo] = A[lo & 3] + B[lo >> 2];
  const uint32_t col = slot_base + 4 * lane;
#pragma unroll
  for (int k = 0; k < 16 / NW; ++k) {   // hi nibbles warp, warp + NW, ...
    const int hi = warp + k * NW;
    const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                    ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), L[lo] + H);
  }
}

// a2 for the column-wise variant (NEXT-f1): the LUT of plane i is built from the
// pre-shifted activations x[k] * 2^{e_i[k]} (SPEC.md:375 ColumnWisePerPlane; the shift is an
// exact fp32 multiply by a power of two: |x| < 2^17 and e in [-100, 100] keep it normal).
__device__ __forceinline__ float pow2_or_zero(int e) {
  return e == SHIFTADD_EXP_ZERO ? 0.f : __int_as_float((e + 127) << 23);
}
template <int NW>
__device__ __forceinline__ void build_lut_slot_colw(uint32_t slot_base, uint32_t xaddr, const int8_t* e8, int warp,
                                                    int lane) {
  uint4 xv;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xv.x), "=r"(xv.y), "=r"(xv.z), "=r"(xv.w)
               : "r"(xaddr + 16 * lane));
  const uint2 ev = __ldg(reinterpret_cast<const uint2*>(e8) + lane);
  const float2 g01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
  const float2 g23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
  const float2 g45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
  const float2 g67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
  auto ex = [&](int b) { return (int)(int8_t)(((b < 4 ? ev.x : ev.y) >> (8 * (b & 3))) & 0xffu); };
  const float2 f01 = make_float2(g01.x * pow2_or_zero(ex(0)), g01.y * pow2_or_zero(ex(1)));
  const float2 f23 = make_float2(g23.x * pow2_or_zero(ex(2)), g23.y * pow2_or_zero(ex(3)));
  const float2 f45 = make_float2(g45.x * pow2_or_zero(ex(4)), g45.y * pow2_or_zero(ex(5)));
  const float2 f67 = make_float2(g67.x * pow2_or_zero(ex(6)), g67.y * pow2_or_zero(ex(7)));
  const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
  const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
  float L[16];
#pragma unroll
  for (int lo = 0; lo < 16; ++lo) L[lo] = A[lo & 3] + B[lo >> 2];
  const uint32_t col = slot_base + 4 * lane;
#pragma unroll
  for (int k = 0; k < 16 / NW; ++k) {
    const int hi = warp + k * NW;
    const float H = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
                    ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) sts_f32(col + ((hi * 16 + lo) << 8), L[lo] + H);
  }
}

// Lookup address of step j: byte 0 = column byte (cst byte j&1), byte 1 = key byte (word
// byte j&3), byte 2 = 0 (cst byte 3), byte 3 = cluster rank (cst byte 2).
__host__ __device__ constexpr uint32_t step_sel_c(int j) {
  return (6u << 12) | (7u << 8) | ((uint32_t)(j & 3) << 4) | (4u + (j & 1));
}

template <int Q, uint32_t IMM, bool AP2 = false>
__device__ __forceinline__ float unit_dot_c(const uint4 (&w)[Q], const int (&e)[Q], const int (&e2)[Q],
                                            const uint32_t (&cst)[8]) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    // 4 chains seeded with the first 4 lookups (no 0 + v adds), summed as a fixed tree
    float p[4];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float v = lds_f32(IMM + prmt(word, cst[j >> 1], step_sel_c(j)));
      p[j & 3] = j < 4 ? v : p[j & 3] + v;
    }
    const float v1 = shift_pow2((p[0] + p[1]) + (p[2] + p[3]), e[i]);
    const float vt = AP2 ? v1 + shift_apot2(v1, e2[i]) : v1;   // NEXT-f2: second additive-PoT term
    acc = i == 0 ? vt : acc + vt;
  }
  return acc;
}

// Column-wise (NEXT-f1): plane i queries its own LUT slot i (slab i >> 1 as the LDS
// immediate, half i & 1 as the constant set) and the sums need no shift.
template <int Q>
__device__ __forceinline__ float unit_dot_colw(const uint4 (&w)[Q], const uint32_t (&cstE)[8],
                                               const uint32_t (&cstO)[8]) {
  float p0 = 0.f, p1 = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    constexpr uint32_t kSlab = kLutBytes;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const uint32_t c = (i & 1) ? cstO[j >> 1] : cstE[j >> 1];
      const uint32_t off = prmt(word, c, step_sel_c(j));
      const float v = (i >> 1) ? lds_f32(kDynBase + kSlab + off) : lds_f32(kDynBase + off);
      if (j & 1) p1 += v; else p0 += v;
    }
  }
  return p0 + p1;
}

template <int Q>
__device__ __forceinline__ void load_planes_unit(const uint4* __restrict__ planes, long long u, int lane, uint64_t pol,
                                                 uint4 (&w)[Q]) {
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = ldg_stream(planes + (u * Q + i) * 32 + lane, pol);
}

// column-wise: no exponent registers, 4 per plane per slot
__host__ __device__ constexpr int cl_ring_colw(int Q, int REGS) {
  return (REGS - 56) / (4 * Q) < 1 ? 1 : ((REGS - 56) / (4 * Q) > 8 ? 8 : (REGS - 56) / (4 * Q));
}
// additive PoT K = 2: one more exponent register per plane per slot
__host__ __device__ constexpr int cl_ring_ap2(int Q, int REGS) {
  return (REGS - 56) / (6 * Q) < 1 ? 1 : ((REGS - 56) / (6 * Q) > 8 ? 8 : (REGS - 56) / (6 * Q));
}
__host__ __device__ constexpr int cl_ring(int Q, int REGS) {
  return (REGS - 56) / (5 * Q) < 1 ? 1 : ((REGS - 56) / (5 * Q) > 8 ? 8 : (REGS - 56) / (5 * Q));
}

// NEXT-f3 completion signal: gather_signal (common.cuh).  Causality is transitive through the
// two synchronising pairs (gpu scope inside this GPU, system scope to the peers), so a consumer
// that acquires all P flags == epoch sees every rank's whole y shard.  (A system-scope fence
// or atomic in every CTA measured 6-12 us per launch; one in the last CTA is cheap.)

// Items of a CTA: i = t * RGb + rgl (slice t of its Sc, row group rgl of the band), warp w
// takes i = w, w + NW, ...; item i is tiled-layout unit (s0 + t) * RG + rg0 + rgl.  The
// warp walks its items with (t, rgl) cursors (no division per item).
struct Cursor {
  int t, rgl;
  template <int NW>
  __device__ __forceinline__ void advance(int RGb) {
    rgl += NW;
    while (rgl >= RGb) { rgl -= RGb; ++t; }
  }
};

constexpr int kFlagPdl = 1, kFlagXFirst = 2, kFlagPushEnd = 4, kFlagXTma = 8;
constexpr int kPreShift = 8;   // flags bits 8..15: ring slots prefilled before griddepcontrol.wait

template <int Q, int SCM, int NW, int REGS, bool COLW, bool AP2 = false>
__global__ void __launch_bounds__(NW * 32) __maxnreg__(REGS)
gemv_cluster_kernel(const __half* __restrict__ x, const uint4* __restrict__ planes,
                    const int8_t* __restrict__ exps, int N, int S, int RG, int C, __half* __restrict__ y,
                    int flags, unsigned long long* __restrict__ trace, const int8_t* __restrict__ exps2,
                    GatherArgs ga) {
  constexpr int D = COLW ? cl_ring_colw(Q, REGS) : (AP2 ? cl_ring_ap2(Q, REGS) : cl_ring(Q, REGS));
  static_assert(!(COLW && AP2), "column-wise and additive-PoT-2 layers are separate formats");
  static_assert(!COLW || (SCM == 4 && Q <= 4), "column-wise: one LUT slot per plane");
  const bool pdl = flags & kFlagPdl;
  const int pre = (flags >> kPreShift) & 0xff;
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
  const int Mw = Mc > warp ? (Mc - warp + NW - 1) / NW : 0;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  if (pdl) pdl_launch_dependents();

  const uint32_t base = dyn_smem_base_cluster();   // kDynBase | rank << 24
  const uint32_t xs = base + Smem<SCM>::lut;
  const uint32_t recv = xs + Smem<SCM>::xstage;
  const uint32_t part = recv + Smem<SCM>::recv;
  const uint32_t bar = part + Smem<SCM>::part;
  const bool push_end = flags & kFlagPushEnd;
  // a5 set-up: the band's rows are cut into C chunks of whole row groups; rank o owns rows
  // [o*chunk, o*chunk + cnt) and receives the S slice partials of each, recv[s][row - o*chunk],
  // (S - Sc) * cnt of them pushed by its peers.
  const int chunk_rg = (RGb + C - 1) / C;
  const int chunk = chunk_rg * kTileRows;
  const int rows = RGb * kTileRows;
  const int own_lo = (int)rank * chunk;
  const int cnt = rows - own_lo < chunk ? (rows - own_lo > 0 ? rows - own_lo : 0) : chunk;
  const float inv_chunk_rg = 1.f / (float)chunk_rg;   // owner of row group g: (g + .5) / chunk_rg
  const bool xtma = flags & kFlagXTma;
  const uint32_t xbar = bar + 8;
  if (tid == 0) {
    mbar_init_expect(bar, (uint32_t)((push_end ? C - 1 : S - Sc) * cnt * 4));
    if (xtma) mbar_init1(xbar);
  }
  cluster_arrive_relaxed();
  const bool xthread = tid < Sc * (kTileK / 8);    // one 16-B chunk of x per thread
  static_assert(NW * 32 >= SCM * (kTileK / 8), "x staging: one chunk per thread");
  const uint4* xsrc = reinterpret_cast<const uint4*>(x + (size_t)s0 * kTileK) + tid;
  Cursor ld{warp / RGb, warp % RGb};
  Cursor pc = ld;
  uint4 w[D][Q];
  int e[D][Q];
  int e2[D][Q];
  auto load_e2 = [&](long long u, int k) {
    if (AP2) {
#pragma unroll
      for (int i = 0; i < Q; ++i) e2[k][i] = ldg_s8_stream(exps2 + (u * Q + i) * 32 + lane, pol_stream);
    }
  };
  // ring slots [k0, k1) of the first D items
  auto prefill = [&](int k0, int k1) {
#pragma unroll
    for (int k = 0; k < D; ++k)
      if (k >= k0 && k < k1 && k < Mw) {
        if (COLW) load_planes_unit<Q>(planes, (long long)(s0 + ld.t) * RG + rg0 + ld.rgl, lane, pol_stream, w[k]);
        else load_unit<Q>(planes, exps, (long long)(s0 + ld.t) * RG + rg0 + ld.rgl, lane, pol_stream, w[k], e[k]);
        load_e2((long long)(s0 + ld.t) * RG + rg0 + ld.rgl, k);
        ld.advance<NW>(RGb);
      }
  };
  // Weights do not depend on the upstream kernel: under PDL the first `pre` ring slots are
  // requested before griddepcontrol.wait -- no more than HBM delivers during the wait, since
  // x queues behind every weight request issued before it (measured: 1.1 us late on FC1
  // with the whole ring in flight) -- and the rest right behind x's request.
  const int pre_n = pdl ? pre : ((flags & kFlagXFirst) ? 0 : D);
  prefill(0, pre_n);
  if (pdl) pdl_wait();
  if (tr && threadIdx.x == 0) tr[8] = gtimer_ns();
  uint4 xv = make_uint4(0, 0, 0, 0);
  if (xtma) {
    if (tid == 0) bulk_load_x(xs, x + (size_t)s0 * kTileK, (uint32_t)(Sc * kTileK * 2), xbar, pol_keep);
  } else if (xthread) {
    xv = ldg_keep(xsrc, pol_keep);
  }
  prefill(pre_n, D);
  if (xtma) {
    mbar_wait_parity0(xbar);
    if (tr && threadIdx.x == 0) tr[9] = gtimer_ns();
  } else if (xthread) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(xs + 16 * tid), "r"(xv.x), "r"(xv.y), "r"(xv.z),
                 "r"(xv.w) : "memory");
    if (tr && threadIdx.x == 0) tr[9] = gtimer_ns();
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[1] = gtimer_ns();
  if (COLW) {   // one slice, one slot per plane built from x * 2^{e_i[k]}
    const int K = S * kTileK;
#pragma unroll
    for (int i = 0; i < Q; ++i)
      build_lut_slot_colw<NW>(base + (uint32_t)(i >> 1) * kLutBytes + (uint32_t)(i & 1) * 128u, xs,
                              exps + (size_t)i * K + (size_t)s0 * kTileK, warp, lane);
  } else {
#pragma unroll
    for (int t = 0; t < SCM; ++t)
      if (t < Sc)
        build_lut_slot<NW>(base + (uint32_t)(t >> 1) * kLutBytes + (uint32_t)(t & 1) * 128u, xs + t * (kTileK * 2),
                           warp, lane);
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[2] = gtimer_ns();
  cluster_wait();   // every peer's receive mbarrier is initialised (arrived at kernel start)

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
      if (COLW) {
        v = unit_dot_colw<Q>(w[k], cstE, cstO);
      } else if (SCM <= 2) {
        v = (pc.t & 1) ? unit_dot_c<Q, kDynBase, AP2>(w[k], e[k], e2[k], cstO)
                       : unit_dot_c<Q, kDynBase, AP2>(w[k], e[k], e2[k], cstE);
      } else {
        switch (pc.t) {   // slot t: slab t >> 1 (LDS immediate), half t & 1 (constant set)
          case 0: v = unit_dot_c<Q, kDynBase, AP2>(w[k], e[k], e2[k], cstE); break;
          case 1: v = unit_dot_c<Q, kDynBase, AP2>(w[k], e[k], e2[k], cstO); break;
          case 2: v = unit_dot_c<Q, kDynBase + kLutBytes, AP2>(w[k], e[k], e2[k], cstE); break;
          default: v = unit_dot_c<Q, kDynBase + kLutBytes, AP2>(w[k], e[k], e2[k], cstO); break;
        }
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      // a5, pushed as soon as the item is done: row pc.rgl*16 + r's partial of slice s0 + t
      // goes to recv[s0 + t][row - o*chunk] of its owner o (st.async completes 4 bytes on the
      // owner's mbarrier; the owner's own rows are plain stores, covered by its bar.sync)
      if (h == 0 && push_end) {
        sts_f32(part + 4u * (uint32_t)((pc.t * RGb + pc.rgl) * kTileRows + r), v);
      } else if (h == 0) {
        const int o = (int)(((float)pc.rgl + 0.5f) * inv_chunk_rg);
        const uint32_t dst =
            recv + 4u * (uint32_t)((s0 + pc.t) * chunk + (pc.rgl - o * chunk_rg) * kTileRows + r);
        if (o == (int)rank) sts_f32(dst, v);
        else st_async_f32(dst, bar, (uint32_t)o, v);
      }
      pc.advance<NW>(RGb);
      if (m + D < Mw) {
        if (COLW) load_planes_unit<Q>(planes, (long long)(s0 + ld.t) * RG + rg0 + ld.rgl, lane, pol_stream, w[k]);
        else load_unit<Q>(planes, exps, (long long)(s0 + ld.t) * RG + rg0 + ld.rgl, lane, pol_stream, w[k], e[k]);
        load_e2((long long)(s0 + ld.t) * RG + rg0 + ld.rgl, k);
        ld.advance<NW>(RGb);
      }
    }
  }
  __syncthreads();         // the CTA's own partials
  if (tr && threadIdx.x == 0) tr[3] = gtimer_ns();
  if (push_end) {   // 3-4 slices per CTA: sum them per row first, push one value per row
    for (int i = tid; i < rows; i += NW * 32) {
      float v = 0.f;
      for (int t = 0; t < Sc; ++t) v += lds_f32(part + 4u * (uint32_t)(t * rows + i));
      const int o = i / chunk;
      const uint32_t dst = recv + 4u * (uint32_t)(rank * chunk + (i - o * chunk));
      if (o == (int)rank) sts_f32(dst, v);
      else st_async_f32(dst, bar, (uint32_t)o, v);
    }
    __syncthreads();
  }
  mbar_wait_parity0(bar);  // the peers' partials
  if (tr && threadIdx.x == 0) tr[4] = gtimer_ns();
  // the owner sums slices 0..S-1 of each of its rows in order (deterministic) and stores
  for (int j = tid; j < cnt; j += NW * 32) {
    float v = lds_f32(recv + 4u * (uint32_t)j);
    const int nsrc = push_end ? C : S;   // ranks 0..C-1, or slices 0..S-1, in order
    for (int s = 1; s < nsrc; ++s) v += lds_f32(recv + 4u * (uint32_t)(s * chunk + j));
    const int n = rg0 * kTileRows + own_lo + j;
    if (n < N) {
      const __half hv = __float2half_rn(v);
      if (ga.P == 0) {
        y[n] = hv;
      } else {   // NEXT-f3: store straight into every rank's gathered y (peer memory)
        const int b = (int)((*ga.epoch + 1u) & 1u);
        for (int r = 0; r < ga.P; ++r) ga.y_peers[b * ga.P + r][(size_t)ga.rank * N + n] = hv;
      }
    }
  }
  if (ga.P > 0) gather_signal(ga);
  if (tr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[5] = gtimer_ns();
    tr[6] = smid;
    tr[7] = (unsigned long long)Mw;
  }
}


// ------------------------------------------------------------------------------------------
// TMA-ring variant of the 2-slot cluster kernel (the default for K <= 4096).  Same items,
// LUT slots, lookups, in-loop DSMEM push and owner reduction as gemv_cluster_kernel; the
// weights reach shared memory through the bulk-copy engine instead of a per-warp register
// ring of LDGs.  Measured on the register ring: with ~96 KB of weight loads in the LSU queue
// when griddepcontrol.wait returns, x (and so the LUT build) waited ~1 us behind them on
// FC1, and shrinking the ring left HBM idle during the wait.  Here one producer thread
// (warp 16) streams the CTA's items -- for each of its slices a contiguous range of units --
// in stages of 16 items (one per consumer warp) into a ring of NST stages, completing on the
// stage's "full" mbarrier, from kernel start on (weights never depend on the upstream
// kernel); the 16 consumer warps fetch x with nothing ahead of it, build the LUTs and take
// one item per stage (LDS.128 of the lane's 16 key bytes per plane, conflict-free), then
// release the stage on its "empty" mbarrier.
constexpr int kRingNW = 16;                       // consumer warps
constexpr int kRingBytes = 124 * 1024;            // stages + their 2 x 8 mbarriers
// Map below the ring: one 64 KB LUT slab -- 2 slices of fp32 entries, or (H16) 4 slices of
// fp16 entries, two slices per 32-bit word -- staged x of up to 4 slices, receive buffer
// recv[slice][row] for up to 4 slices per CTA, the owner's receive mbarrier.
struct RingMap {
  static constexpr int lut = kLutBytes;
  static constexpr int xstage = 4 * kTileK * 2;
  static constexpr int recv = 4 * (4 * (kMaxRGb + kMaxC) * kTileRows);
  static constexpr int bar = lut + xstage + recv;
  static constexpr int total = bar + 16;
};
constexpr int kRingBase = (RingMap::total + 127) & ~127;
static_assert(kRingBase + kRingBytes <= 227 * 1024, "ring must fit");

// a2 for the fp16-pair LUT (H16): word (key, col) of column half `hoff` holds slice ta's entry
// in its low half and slice tb's in its high half (fp32 sums rounded once to fp16, RNE), so a
// 64 KB slab holds 4 slices and a build stores half the bytes (store-bandwidth bound:
// tools/lutbuild.cu, 310 vs 595 cycles per 2 slices).  A lookup of slice t reads the 16-bit
// half 2*(t&1) of the fp32 layout's address -- an LDS.U16 immediate -- and converts it.
template <int NW>
__device__ __forceinline__ void build_lut_pair16(uint32_t slot_base, uint32_t xa, uint32_t xb, bool has_b,
                                                 int warp, int lane) {
  float L[2][16], H[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    uint4 xv = make_uint4(0, 0, 0, 0);
    if (u == 0 || has_b)
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xv.x), "=r"(xv.y), "=r"(xv.z), "=r"(xv.w)
                   : "r"((u ? xb : xa) + 16 * lane));
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
    const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
    const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
    const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
    const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) L[u][lo] = A[lo & 3] + B[lo >> 2];
    const int hi = warp;   // NW == 16: one hi nibble per warp
    H[u] = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
           ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
  }
  static_assert(NW == 16, "one hi nibble per warp");
  const uint32_t col = slot_base + 4 * lane;
#pragma unroll
  for (int lo = 0; lo < 16; ++lo) {
    const __half2 v = __floats2half2_rn(L[0][lo] + H[0], L[1][lo] + H[1]);
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(col + ((warp * 16 + lo) << 8)),
                 "r"(*reinterpret_cast<const uint32_t*>(&v)) : "memory");
  }
}

__device__ __forceinline__ float lds_h16(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return __half2float(__ushort_as_half(v));
}

// a3 + a4 with fp16 LUT entries: slice half `IMM2` (0 or 2 bytes) of the words addressed as
// in unit_dot_c.
template <int Q, uint32_t IMM>
__device__ __forceinline__ float unit_dot_h16(const uint4 (&w)[Q], const int (&e)[Q], const uint32_t (&cst)[8]) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float p0 = 0.f, p1 = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float v = lds_h16(IMM + prmt(word, cst[j >> 1], step_sel_c(j)));
      if (j & 1) p1 += v; else p0 += v;
    }
    acc += shift_pow2(p0 + p1, e[i]);
  }
  return acc;
}

template <int Q>
struct RingCfg {
  static constexpr int items = kRingNW;              // items per stage: one per consumer warp
  static constexpr int stage_planes = items * Q * kTileBytes;
  static constexpr int stage = items * Q * (kTileBytes + kTileExps);
  static constexpr int nst = (kRingBytes - 128) / stage > 8 ? 8 : (kRingBytes - 128) / stage;
  static constexpr int bars = nst * stage;          // full[j] at +8j, empty[j] at +64+8j
  static constexpr int smem = kRingBase + kRingBytes;
};
static_assert(kRingBase + kRingBytes <= 227 * 1024, "ring must fit");

__device__ __forceinline__ void rmbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void rmbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}

template <int Q, bool H16>
__global__ void __launch_bounds__((kRingNW + 1) * 32, 1)
gemv_cluster_ring_kernel(const __half* __restrict__ x, const uint8_t* __restrict__ planes,
                         const int8_t* __restrict__ exps, int N, int S, int RG, int C, __half* __restrict__ y,
                         int flags, unsigned long long* __restrict__ trace, GatherArgs ga) {
  using RC = RingCfg<Q>;
  constexpr int NW = kRingNW, NST = RC::nst, SI = RC::items;
  const bool pdl = flags & kFlagPdl;
  if (threadIdx.x == 0) check_dyn_base();
  unsigned long long* tr = trace ? trace + 32 * blockIdx.x : nullptr;   // dev trace
  if (tr && threadIdx.x == 0) tr[0] = gtimer_ns();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (NW + 1) * 32;
  const int r = lane >> 1, h = lane & 1;
  const uint32_t rank = cluster_rank();
  const unsigned Cu = (unsigned)C, ncl = gridDim.x / Cu, cl = blockIdx.x / Cu;
  const int rg0 = (int)((cl * (unsigned)RG) / ncl);
  const int RGb = (int)(((cl + 1) * (unsigned)RG) / ncl) - rg0;
  const int s0 = (int)((rank * (unsigned)S) / Cu);
  const int Sc = (int)(((rank + 1) * (unsigned)S) / Cu) - s0;   // <= 2 (H16: <= 4)
  const int Mc = Sc * RGb;                                        // items: i = t * RGb + rgl
  if (pdl) pdl_launch_dependents();

  const uint32_t base = dyn_smem_base_cluster();   // kDynBase | rank << 24
  const uint32_t xs = base + RingMap::lut;
  const uint32_t recv = xs + RingMap::xstage;
  const uint32_t bar = base + RingMap::bar;
  const uint32_t ring = base + (uint32_t)kRingBase;
  const uint32_t full = ring + RC::bars, empty = full + 64;
  // a5 set-up as in gemv_cluster_kernel (in-loop push of every (slice, row) partial)
  const int chunk_rg = (RGb + C - 1) / C;
  const int chunk = chunk_rg * kTileRows;
  const int rows = RGb * kTileRows;
  const int own_lo = (int)rank * chunk;
  const int cnt = rows - own_lo < chunk ? (rows - own_lo > 0 ? rows - own_lo : 0) : chunk;
  const float inv_chunk_rg = 1.f / (float)chunk_rg;
  if (tid == 0) {
    mbar_init_expect(bar, (uint32_t)((S - Sc) * cnt * 4));
    for (int j = 0; j < NST; ++j) {
      rmbar_init(full + 8 * j, 1);
      rmbar_init(empty + 8 * j, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  cluster_arrive_relaxed();
  const int nstages = (Mc + SI - 1) / SI;

  if (warp == NW) {
    // producer: stage t = items [16t, 16t + 16), one contiguous unit range per slice
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < nstages; ++t) {
        const int j = t % NST;
        if (t >= NST) rmbar_wait(empty + 8 * j, (uint32_t)((t / NST - 1) & 1));
        const int i0 = t * SI, i1 = i0 + SI < Mc ? i0 + SI : Mc;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * j),
                     "r"((uint32_t)((i1 - i0) * Q * (kTileBytes + kTileExps))) : "memory");
        for (int a = i0; a < i1;) {
          const int ts = a / RGb;
          const int b = (ts + 1) * RGb < i1 ? (ts + 1) * RGb : i1;
          const long long u = (long long)(s0 + ts) * RG + rg0 + (a - ts * RGb);
          const uint32_t dst = ring + (uint32_t)(j * RC::stage);
          bulk_load_x(dst + (uint32_t)((a - i0) * Q * kTileBytes), planes + u * Q * kTileBytes,
                      (uint32_t)((b - a) * Q * kTileBytes), full + 8 * j, pol, false);
          bulk_load_x(dst + (uint32_t)(RC::stage_planes + (a - i0) * Q * kTileExps), exps + u * Q * kTileExps,
                      (uint32_t)((b - a) * Q * kTileExps), full + 8 * j, pol, false);
          a = b;
        }
      }
    }
  } else {
    // x into L2 before the PDL wait (a hint: L2 is the point of coherence and x is read after
    // the wait), so a cold x costs no miss on the call's dependent chain
    if (tid < Sc * 4)
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(x + (size_t)s0 * kTileK + 64 * tid));
    if (pdl) pdl_wait();
    if (tr && tid == 0) tr[8] = gtimer_ns();
    if (tid < Sc * (kTileK / 8)) {   // one 16-B chunk of x per thread
      const uint4 xv = ldg_keep(reinterpret_cast<const uint4*>(x + (size_t)s0 * kTileK) + tid, policy_evict_last());
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(xs + 16 * tid), "r"(xv.x), "r"(xv.y), "r"(xv.z),
                   "r"(xv.w) : "memory");
      if (tr && tid == 0) tr[9] = gtimer_ns();
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");   // consumer warps only
    if (tr && tid == 0) tr[1] = gtimer_ns();
    if (H16) {   // slices (0,1) in column half 0, (2,3) in half 1
      for (int t = 0; t < Sc; t += 2)
        build_lut_pair16<NW>(base + (uint32_t)(t >> 1) * 128u, xs + t * (kTileK * 2), xs + (t + 1) * (kTileK * 2),
                             t + 1 < Sc, warp, lane);
    } else {
      for (int t = 0; t < 2; ++t)
        if (t < Sc) build_lut_slot<NW>(base + (uint32_t)t * 128u, xs + t * (kTileK * 2), warp, lane);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    if (tr && tid == 0) tr[2] = gtimer_ns();
    cluster_wait();   // every peer's receive mbarrier is initialised
    uint32_t cstE[8], cstO[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t c0 = 4u * (uint32_t)(16 * h + ((2 * c + r) & 15));
      const uint32_t c1 = 4u * (uint32_t)(16 * h + ((2 * c + 1 + r) & 15));
      cstE[c] = c0 | (c1 << 8) | (rank << 16);
      cstO[c] = cstE[c] + 0x8080u;
    }
    for (int t = 0; t < nstages; ++t) {
      const int j = t % NST;
      const int i = t * NW + warp;
      rmbar_wait(full + 8 * j, (uint32_t)((t / NST) & 1));
      if (tr && tid == 0 && (t == 0 || t == nstages - 1)) tr[t == 0 ? 10 : 11] = gtimer_ns();
      if (i < Mc) {
        uint4 w[Q];
        int e[Q];
        const uint32_t sp = ring + (uint32_t)(j * RC::stage + warp * Q * kTileBytes + 16 * lane);
        const uint32_t se = ring + (uint32_t)(j * RC::stage + RC::stage_planes + warp * Q * kTileExps + lane);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          smem_check(sp + (uint32_t)(k * kTileBytes), 16);
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[k].x), "=r"(w[k].y), "=r"(w[k].z),
                       "=r"(w[k].w) : "r"(sp + (uint32_t)(k * kTileBytes)));
          smem_check(se + (uint32_t)(k * kTileExps), 1);
          asm volatile("ld.shared.s8 %0, [%1];" : "=r"(e[k]) : "r"(se + (uint32_t)(k * kTileExps)));
        }
        const int ts = H16 ? (i >= RGb) + (i >= 2 * RGb) + (i >= 3 * RGb) : (i >= RGb ? 1 : 0);
        const int rgl = i - ts * RGb;
        float v;
        if (H16) {
          switch (ts) {   // column half ts >> 1 (constant set), word half ts & 1 (LDS immediate)
            case 0: v = unit_dot_h16<Q, kDynBase>(w, e, cstE); break;
            case 1: v = unit_dot_h16<Q, kDynBase + 2>(w, e, cstE); break;
            case 2: v = unit_dot_h16<Q, kDynBase>(w, e, cstO); break;
            default: v = unit_dot_h16<Q, kDynBase + 2>(w, e, cstO); break;
          }
        } else {
          v = ts ? unit_dot_c<Q, kDynBase, false>(w, e, e, cstO) : unit_dot_c<Q, kDynBase, false>(w, e, e, cstE);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (h == 0) {   // a5 push, as in gemv_cluster_kernel
          const int o = (int)(((float)rgl + 0.5f) * inv_chunk_rg);
          const uint32_t dst = recv + 4u * (uint32_t)((s0 + ts) * chunk + (rgl - o * chunk_rg) * kTileRows + r);
          if (o == (int)rank) sts_f32(dst, v);
          else st_async_f32(dst, bar, (uint32_t)o, v);
        }
      } else {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
      }
    }
  }
  __syncthreads();         // the CTA's own partials
  if (tr && threadIdx.x == 0) tr[3] = gtimer_ns();
  mbar_wait_parity0(bar);  // the peers' partials
  if (tr && threadIdx.x == 0) tr[4] = gtimer_ns();
  for (int jj = tid; jj < cnt; jj += NT) {
    float v = lds_f32(recv + 4u * (uint32_t)jj);
    for (int s = 1; s < S; ++s) v += lds_f32(recv + 4u * (uint32_t)(s * chunk + jj));
    const int n = rg0 * kTileRows + own_lo + jj;
    if (n < N) {
      const __half hv = __float2half_rn(v);
      if (ga.P == 0) {
        y[n] = hv;
      } else {   // NEXT-f3: store straight into every rank's gathered y (peer memory)
        const int b = (int)((*ga.epoch + 1u) & 1u);
        for (int rr = 0; rr < ga.P; ++rr) ga.y_peers[b * ga.P + rr][(size_t)ga.rank * N + n] = hv;
      }
    }
  }
  if (ga.P > 0) gather_signal(ga);
  if (tr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[5] = gtimer_ns();
    tr[6] = smid;
    tr[7] = (unsigned long long)nstages;
  }
}


// ------------------------------------------------------------------------------------------
// Fused projections on the cluster TMA ring (kernel id 10): the segments of
// shiftadd_lut_gemv_fused (LLaMA q/k/v at 2/3/2 bits, gate/up at 2/3) in one launch of the
// ring kernel's decomposition.  A cluster's band is a range of the segments' concatenated row
// groups; per slice of the CTA the band splits into runs of one segment (one q), each streamed
// in stages of <= 16 items of q x 544 B; the consumers walk the same runs and dispatch on q.
// Reduction (in-loop DSMEM push, owner sums in slice order) as in gemv_cluster_ring_kernel.
struct FusedSeg {
  const uint8_t* planes;
  const int8_t* exps;
  __half* y;
  int q, N, RG, rgoff;
};
struct FusedArgs {
  const __half* x;
  FusedSeg seg[kMaxSegments];
  int nseg, S, RGtot, C, slot, slot_planes, nst, pdl;
};

// Run of the band [b0, b1) inside segment g: [max(b0, rgoff), min(b1, rgoff + RG)).
__device__ __forceinline__ bool fused_run(const FusedArgs& A, int g, int b0, int b1, int& ra, int& rb) {
  ra = b0 > A.seg[g].rgoff ? b0 : A.seg[g].rgoff;
  const int e = A.seg[g].rgoff + A.seg[g].RG;
  rb = b1 < e ? b1 : e;
  return ra < rb;
}

template <int Q>
__device__ __forceinline__ float fused_dot(uint32_t sp, uint32_t se, bool odd, const uint32_t (&cstE)[8],
                                           const uint32_t (&cstO)[8]) {
  uint4 w[Q];
  int e[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    smem_check(sp + (uint32_t)(k * kTileBytes), 16);
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[k].x), "=r"(w[k].y), "=r"(w[k].z), "=r"(w[k].w)
                 : "r"(sp + (uint32_t)(k * kTileBytes)));
    smem_check(se + (uint32_t)(k * kTileExps), 1);
    asm volatile("ld.shared.s8 %0, [%1];" : "=r"(e[k]) : "r"(se + (uint32_t)(k * kTileExps)));
  }
  return odd ? unit_dot_c<Q, kDynBase, false>(w, e, e, cstO) : unit_dot_c<Q, kDynBase, false>(w, e, e, cstE);
}

__global__ void __launch_bounds__((kRingNW + 1) * 32, 1) gemv_cluster_fused_kernel(const __grid_constant__ FusedArgs A) {
  constexpr int NW = kRingNW;
  if (threadIdx.x == 0) check_dyn_base();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (NW + 1) * 32;
  const int r = lane >> 1, h = lane & 1;
  const uint32_t rank = cluster_rank();
  const unsigned Cu = (unsigned)A.C, ncl = gridDim.x / Cu, cl = blockIdx.x / Cu;
  const int S = A.S;
  const int rg0 = (int)((cl * (unsigned)A.RGtot) / ncl);
  const int RGb = (int)(((cl + 1) * (unsigned)A.RGtot) / ncl) - rg0;
  const int s0 = (int)((rank * (unsigned)S) / Cu);
  const int Sc = (int)(((rank + 1) * (unsigned)S) / Cu) - s0;   // <= 2
  if (A.pdl) pdl_launch_dependents();

  const uint32_t base = dyn_smem_base_cluster();
  const uint32_t xs = base + RingMap::lut;
  const uint32_t recv = xs + RingMap::xstage;
  const uint32_t bar = base + RingMap::bar;
  const uint32_t ring = base + (uint32_t)kRingBase;
  const uint32_t full = ring + (uint32_t)(A.nst * A.slot), empty = full + 64;
  const int chunk_rg = (RGb + A.C - 1) / A.C;
  const int chunk = chunk_rg * kTileRows;
  const int rows = RGb * kTileRows;
  const int own_lo = (int)rank * chunk;
  const int cnt = rows - own_lo < chunk ? (rows - own_lo > 0 ? rows - own_lo : 0) : chunk;
  const float inv_chunk_rg = 1.f / (float)chunk_rg;
  if (tid == 0) {
    mbar_init_expect(bar, (uint32_t)((S - Sc) * cnt * 4));
    for (int j = 0; j < A.nst; ++j) {
      rmbar_init(full + 8 * j, 1);
      rmbar_init(empty + 8 * j, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  cluster_arrive_relaxed();

  if (warp == NW) {
    // producer: per slice t, per segment run of the band, stages of <= 16 items
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int st = 0;
      for (int t = 0; t < Sc; ++t) {
        for (int g = 0; g < A.nseg; ++g) {
          int ra, rb;
          if (!fused_run(A, g, rg0, rg0 + RGb, ra, rb)) continue;
          const FusedSeg& sg = A.seg[g];
          for (int a = ra; a < rb; a += NW, ++st) {
            const int n = rb - a < NW ? rb - a : NW;
            const int j = st % A.nst;
            if (st >= A.nst) rmbar_wait(empty + 8 * j, (uint32_t)((st / A.nst - 1) & 1));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * j),
                         "r"((uint32_t)(n * sg.q * (kTileBytes + kTileExps))) : "memory");
            const long long u = (long long)(s0 + t) * sg.RG + (a - sg.rgoff);
            const uint32_t dst = ring + (uint32_t)(j * A.slot);
            bulk_load_x(dst, sg.planes + u * sg.q * kTileBytes, (uint32_t)(n * sg.q * kTileBytes), full + 8 * j, pol,
                        false);
            bulk_load_x(dst + (uint32_t)A.slot_planes, sg.exps + u * sg.q * kTileExps,
                        (uint32_t)(n * sg.q * kTileExps), full + 8 * j, pol, false);
          }
        }
      }
    }
  } else {
    if (tid < Sc * 4)
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(A.x + (size_t)s0 * kTileK + 64 * tid));
    if (A.pdl) pdl_wait();
    if (tid < Sc * (kTileK / 8)) {
      const uint4 xv = ldg_keep(reinterpret_cast<const uint4*>(A.x + (size_t)s0 * kTileK) + tid, policy_evict_last());
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(xs + 16 * tid), "r"(xv.x), "r"(xv.y), "r"(xv.z),
                   "r"(xv.w) : "memory");
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    for (int t = 0; t < Sc; ++t) build_lut_slot<NW>(base + (uint32_t)t * 128u, xs + t * (kTileK * 2), warp, lane);
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    cluster_wait();
    uint32_t cstE[8], cstO[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t c0 = 4u * (uint32_t)(16 * h + ((2 * c + r) & 15));
      const uint32_t c1 = 4u * (uint32_t)(16 * h + ((2 * c + 1 + r) & 15));
      cstE[c] = c0 | (c1 << 8) | (rank << 16);
      cstO[c] = cstE[c] + 0x8080u;
    }
    int st = 0;
    for (int t = 0; t < Sc; ++t) {
      for (int g = 0; g < A.nseg; ++g) {
        int ra, rb;
        if (!fused_run(A, g, rg0, rg0 + RGb, ra, rb)) continue;
        const int q = A.seg[g].q;
        for (int a = ra; a < rb; a += NW, ++st) {
          const int n = rb - a < NW ? rb - a : NW;
          const int j = st % A.nst;
          rmbar_wait(full + 8 * j, (uint32_t)((st / A.nst) & 1));
          if (warp < n) {
            const uint32_t sp = ring + (uint32_t)(j * A.slot + warp * q * kTileBytes + 16 * lane);
            const uint32_t se = ring + (uint32_t)(j * A.slot + A.slot_planes + warp * q * kTileExps + lane);
            float v;
            switch (q) {
              case 1: v = fused_dot<1>(sp, se, t, cstE, cstO); break;
              case 2: v = fused_dot<2>(sp, se, t, cstE, cstO); break;
              case 3: v = fused_dot<3>(sp, se, t, cstE, cstO); break;
              default: v = fused_dot<4>(sp, se, t, cstE, cstO); break;
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            if (h == 0) {
              const int rgl = a + warp - rg0;   // band-local row group
              const int o = (int)(((float)rgl + 0.5f) * inv_chunk_rg);
              const uint32_t dst = recv + 4u * (uint32_t)((s0 + t) * chunk + (rgl - o * chunk_rg) * kTileRows + r);
              if (o == (int)rank) sts_f32(dst, v);
              else st_async_f32(dst, bar, (uint32_t)o, v);
            }
          } else {
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
          }
        }
      }
    }
  }
  __syncthreads();
  mbar_wait_parity0(bar);
  for (int jj = tid; jj < cnt; jj += NT) {
    float v = lds_f32(recv + 4u * (uint32_t)jj);
    for (int s = 1; s < S; ++s) v += lds_f32(recv + 4u * (uint32_t)(s * chunk + jj));
    const int nf = rg0 * kTileRows + own_lo + jj;   // row of the concatenated segments
    const int rgf = nf / kTileRows;
    int g = 0;
    while (g + 1 < A.nseg && A.seg[g + 1].rgoff <= rgf) ++g;
    const int nl = nf - A.seg[g].rgoff * kTileRows;
    if (nl < A.seg[g].N) A.seg[g].y[nl] = __float2half_rn(v);
  }
}

// ------------------------------------------------------------------------------------------
// §8 a7, M = 2 on the cluster TMA ring (kernel id 5).  The batch-1 ring kernel's
// decomposition, weight ring and DSMEM reduction, with float2 LUT entries holding the
// partial sums of both batch rows: one key byte from HBM, one LDS.64, two FADDs.  A slot is
// 256 keys x 32 groups x 8 B = 64 KB; group g of a slice sits at physical column
// pcol(g) = 16*(g>>4) + ((g & 15) ^ 8*(g>>4)), so each 16-lane LDS.64 phase (rows r..r+7,
// halves 0/1) covers all 32 banks (the XOR sends half 1 to the complementary 8 columns).
// Two slots (slices) per CTA -> 128 KB of LUT and a 60 KB weight ring.
constexpr int kM2RingBytes = 60 * 1024;
struct M2Map {
  static constexpr int lut = 2 * kLutBytes;
  static constexpr int xstage = 2 * 2 * kTileK * 2;                        // [row][slice][256] fp16
  static constexpr int recv = 4 * (2 * 2 * (kMaxRGb + kMaxC) * kTileRows);  // [row][slice][chunk row]
  static constexpr int bar = lut + xstage + recv;
  static constexpr int base = (bar + 16 + 127) & ~127;                      // the ring
  static constexpr int total = base + kM2RingBytes;
};
static_assert(M2Map::total <= 227 * 1024, "M = 2 ring kernel must fit");

template <int Q>
struct M2Cfg {
  static constexpr int stage_planes = kRingNW * Q * kTileBytes;
  static constexpr int stage = kRingNW * Q * (kTileBytes + kTileExps);
  static constexpr int nst = (kM2RingBytes - 128) / stage > 8 ? 8 : (kM2RingBytes - 128) / stage;
  static constexpr int bars = nst * stage;
};

__host__ __device__ constexpr int pcol2(int g) { return 16 * (g >> 4) + ((g & 15) ^ (8 * (g >> 4))); }

// a2 for M = 2: slot at slot_base from x rows 0/1 of one slice (xa, xb: shared addresses of
// the 256 activations of each row); warp = hi nibble, lane = group.
__device__ __forceinline__ void build_lut_slot_m2(uint32_t slot_base, uint32_t xa, uint32_t xb, int warp, int lane) {
  float L[2][16], H[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    uint4 xv;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xv.x), "=r"(xv.y), "=r"(xv.z), "=r"(xv.w)
                 : "r"((m ? xb : xa) + 16 * lane));
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
    const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
    const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
    const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
    const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) L[m][lo] = A[lo & 3] + B[lo >> 2];
    const int hi = warp;
    H[m] = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
           ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
  }
  const uint32_t col = slot_base + 8u * (uint32_t)pcol2(lane);
#pragma unroll
  for (int lo = 0; lo < 16; ++lo)
    asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(col + ((warp * 16 + lo) << 8)), "f"(L[0][lo] + H[0]),
                 "f"(L[1][lo] + H[1]) : "memory");
}

__device__ __forceinline__ float2 lds_f32x2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

// a3 + a4 for both rows of one unit; IMM = the slot's LUT base.
template <int Q, uint32_t IMM>
__device__ __forceinline__ float2 unit_dot_m2(const uint4 (&w)[Q], const int (&e)[Q], const uint32_t (&cst)[8]) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float2 p[2];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float2 v = lds_f32x2(IMM + prmt(word, cst[j >> 1], step_sel_c(j)));
      if (j < 2) {
        p[j & 1] = v;
      } else {
        p[j & 1].x += v.x;
        p[j & 1].y += v.y;
      }
    }
    const float v0 = shift_pow2(p[0].x + p[1].x, e[i]), v1 = shift_pow2(p[0].y + p[1].y, e[i]);
    acc.x = i == 0 ? v0 : acc.x + v0;
    acc.y = i == 0 ? v1 : acc.y + v1;
  }
  return acc;
}

template <int Q>
__global__ void __launch_bounds__((kRingNW + 1) * 32, 1)
gemm_cluster_ring_m2_kernel(const __half* __restrict__ x, int ldx, const uint8_t* __restrict__ planes,
                            const int8_t* __restrict__ exps, int N, int S, int RG, int C, __half* __restrict__ y,
                            int ldy, int flags) {
  using RC = M2Cfg<Q>;
  constexpr int NW = kRingNW, NST = RC::nst;
  const bool pdl = flags & kFlagPdl;
  if (threadIdx.x == 0) check_dyn_base();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (NW + 1) * 32;
  const int r = lane >> 1, h = lane & 1;
  const uint32_t rank = cluster_rank();
  const unsigned Cu = (unsigned)C, ncl = gridDim.x / Cu, cl = blockIdx.x / Cu;
  const int rg0 = (int)((cl * (unsigned)RG) / ncl);
  const int RGb = (int)(((cl + 1) * (unsigned)RG) / ncl) - rg0;
  const int s0 = (int)((rank * (unsigned)S) / Cu);
  const int Sc = (int)(((rank + 1) * (unsigned)S) / Cu) - s0;   // <= 2
  const int Mc = Sc * RGb;
  if (pdl) pdl_launch_dependents();

  const uint32_t base = dyn_smem_base_cluster();
  const uint32_t xs = base + M2Map::lut;
  const uint32_t recv = xs + M2Map::xstage;
  const uint32_t bar = base + M2Map::bar;
  const uint32_t ring = base + (uint32_t)M2Map::base;
  const uint32_t full = ring + RC::bars, empty = full + 64;
  const int chunk_rg = (RGb + C - 1) / C;
  const int chunk = chunk_rg * kTileRows;
  const int rows = RGb * kTileRows;
  const int own_lo = (int)rank * chunk;
  const int cnt = rows - own_lo < chunk ? (rows - own_lo > 0 ? rows - own_lo : 0) : chunk;
  const float inv_chunk_rg = 1.f / (float)chunk_rg;
  if (tid == 0) {
    mbar_init_expect(bar, (uint32_t)(2 * (S - Sc) * cnt * 4));
    for (int j = 0; j < NST; ++j) {
      rmbar_init(full + 8 * j, 1);
      rmbar_init(empty + 8 * j, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  cluster_arrive_relaxed();
  const int nstages = (Mc + NW - 1) / NW;

  if (warp == NW) {
    if (lane == 0) {   // producer, as in gemv_cluster_ring_kernel
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < nstages; ++t) {
        const int j = t % NST;
        if (t >= NST) rmbar_wait(empty + 8 * j, (uint32_t)((t / NST - 1) & 1));
        const int i0 = t * NW, i1 = i0 + NW < Mc ? i0 + NW : Mc;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * j),
                     "r"((uint32_t)((i1 - i0) * Q * (kTileBytes + kTileExps))) : "memory");
        for (int a = i0; a < i1;) {
          const int ts = a / RGb;
          const int b = (ts + 1) * RGb < i1 ? (ts + 1) * RGb : i1;
          const long long u = (long long)(s0 + ts) * RG + rg0 + (a - ts * RGb);
          const uint32_t dst = ring + (uint32_t)(j * RC::stage);
          bulk_load_x(dst + (uint32_t)((a - i0) * Q * kTileBytes), planes + u * Q * kTileBytes,
                      (uint32_t)((b - a) * Q * kTileBytes), full + 8 * j, pol, false);
          bulk_load_x(dst + (uint32_t)(RC::stage_planes + (a - i0) * Q * kTileExps), exps + u * Q * kTileExps,
                      (uint32_t)((b - a) * Q * kTileExps), full + 8 * j, pol, false);
          a = b;
        }
      }
    }
  } else {
    if (pdl) pdl_wait();
    if (tid < 2 * Sc * (kTileK / 8)) {   // x rows 0/1 of the CTA's slices -> xs[row][slice][256]
      const int m = tid / (Sc * 32), c = tid - m * (Sc * 32);
      const uint4 xv = ldg_keep(reinterpret_cast<const uint4*>(x + (size_t)m * ldx + (size_t)s0 * kTileK) + c,
                                policy_evict_last());
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(xs + (uint32_t)(m * 2 * kTileK * 2 + 16 * c)),
                   "r"(xv.x), "r"(xv.y), "r"(xv.z), "r"(xv.w) : "memory");
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    for (int t = 0; t < Sc; ++t)
      build_lut_slot_m2(base + (uint32_t)t * kLutBytes, xs + (uint32_t)(t * kTileK * 2),
                        xs + (uint32_t)(2 * kTileK * 2 + t * kTileK * 2), warp, lane);
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    cluster_wait();
    uint32_t cst[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t c0 = 8u * (uint32_t)pcol2(16 * h + ((2 * c + r) & 15));
      const uint32_t c1 = 8u * (uint32_t)pcol2(16 * h + ((2 * c + 1 + r) & 15));
      cst[c] = c0 | (c1 << 8) | (rank << 16);
    }
    for (int t = 0; t < nstages; ++t) {
      const int j = t % NST;
      const int i = t * NW + warp;
      rmbar_wait(full + 8 * j, (uint32_t)((t / NST) & 1));
      if (i < Mc) {
        uint4 w[Q];
        int e[Q];
        const uint32_t sp = ring + (uint32_t)(j * RC::stage + warp * Q * kTileBytes + 16 * lane);
        const uint32_t se = ring + (uint32_t)(j * RC::stage + RC::stage_planes + warp * Q * kTileExps + lane);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          smem_check(sp + (uint32_t)(k * kTileBytes), 16);
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[k].x), "=r"(w[k].y), "=r"(w[k].z),
                       "=r"(w[k].w) : "r"(sp + (uint32_t)(k * kTileBytes)));
          smem_check(se + (uint32_t)(k * kTileExps), 1);
          asm volatile("ld.shared.s8 %0, [%1];" : "=r"(e[k]) : "r"(se + (uint32_t)(k * kTileExps)));
        }
        const int ts = i >= RGb ? 1 : 0, rgl = i - ts * RGb;
        float2 v = ts ? unit_dot_m2<Q, kDynBase + kLutBytes>(w, e, cst) : unit_dot_m2<Q, kDynBase>(w, e, cst);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
        if (h == 0) {   // a5 push of both rows' partials: recv[m][slice][row - o*chunk] of owner o
          const int o = (int)(((float)rgl + 0.5f) * inv_chunk_rg);
          const uint32_t d0 = recv + 4u * (uint32_t)((s0 + ts) * chunk + (rgl - o * chunk_rg) * kTileRows + r);
          const uint32_t d1 = d0 + 4u * (uint32_t)(S * chunk);
          if (o == (int)rank) {
            sts_f32(d0, v.x);
            sts_f32(d1, v.y);
          } else {
            st_async_f32(d0, bar, (uint32_t)o, v.x);
            st_async_f32(d1, bar, (uint32_t)o, v.y);
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
      }
    }
  }
  __syncthreads();
  mbar_wait_parity0(bar);
  for (int it = tid; it < 2 * cnt; it += NT) {   // the owner: rows 0/1 of its chunk, slices in order
    const int m = it >= cnt ? 1 : 0, jj = it - m * cnt;
    const uint32_t rb = recv + 4u * (uint32_t)(m * S * chunk + jj);
    float v = lds_f32(rb);
    for (int s = 1; s < S; ++s) v += lds_f32(rb + 4u * (uint32_t)(s * chunk));
    const int n = rg0 * kTileRows + own_lo + jj;
    if (n < N) y[(size_t)m * ldy + n] = __float2half_rn(v);
  }
}

template <int Q>
cudaError_t launch_m2_q(const GemmArgs& a, const LaunchPlan& p, int C) {
  const cudaError_t err = once_per_device([] {
    cudaError_t err = cudaSuccess;
    err = cudaFuncSetAttribute(gemm_cluster_ring_m2_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               M2Map::total);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(gemm_cluster_ring_m2_kernel<Q>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return err;
  });
  if (err != cudaSuccess) return err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(p.grid);
  c.blockDim = dim3((kRingNW + 1) * 32);
  c.dynamicSmemBytes = M2Map::total;
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
  return cudaLaunchKernelEx(&c, gemm_cluster_ring_m2_kernel<Q>, a.x, a.ldx, a.planes, a.exps, a.N, S, RG, C, a.y,
                            a.ldy, pdl ? kFlagPdl : 0);
}


// ------------------------------------------------------------------------------------------
// §8 a7, M = 3..4 on the cluster TMA ring (kernel id 6).  float4 LUT entries (4 rows per
// lookup: one LDS.128, four FADDs).  A slot is 256 keys x 32 groups x 16 B = 128 KB in two
// 64 KB regions (group half h = g >> 4); group g sits at region h, key*256 + ((g & 15) ^ 4h)*16,
// so each 8-lane LDS.128 phase covers 8 distinct 16-B bank groups.  One slot (slice) per CTA:
// clusters of S (K <= 4096).  The PRMT forms the whole address from the key byte and a
// per-step constant (column byte, region byte, rank byte).
struct M4Map {
  static constexpr int lut = 2 * kLutBytes;
  static constexpr int xstage = 4 * kTileK * 2;                            // [row][256] fp16
  static constexpr int recv = 4 * (4 * (kMaxRGb + 2 * kMaxC) * kTileRows);  // [row][slice][chunk row]
  static constexpr int bar = lut + xstage + recv;
  static constexpr int base = (bar + 16 + 127) & ~127;
  static constexpr int total = base + kM2RingBytes;
};
static_assert(M4Map::total <= 227 * 1024, "M = 4 ring kernel must fit");

// step j: byte0 <- cst byte 0 (column), byte1 <- key byte j&3, byte2 <- cst byte 2 (region),
// byte3 <- cst byte 3 (rank)
__host__ __device__ constexpr uint32_t step_sel_m4(int j) { return (7u << 12) | (6u << 8) | ((uint32_t)(j & 3) << 4) | 4u; }

__device__ __forceinline__ void build_lut_slot_m4(uint32_t slot_base, uint32_t xs, int warp, int lane) {
  float L[4][16], H[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    uint4 xv;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xv.x), "=r"(xv.y), "=r"(xv.z), "=r"(xv.w)
                 : "r"(xs + (uint32_t)(m * kTileK * 2) + 16 * lane));
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
    const float2 f45 = __half22float2(*reinterpret_cast<const __half2*>(&xv.z));
    const float2 f67 = __half22float2(*reinterpret_cast<const __half2*>(&xv.w));
    const float A[4] = {-f01.x - f01.y, f01.x - f01.y, f01.y - f01.x, f01.x + f01.y};
    const float B[4] = {-f23.x - f23.y, f23.x - f23.y, f23.y - f23.x, f23.x + f23.y};
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) L[m][lo] = A[lo & 3] + B[lo >> 2];
    const int hi = warp;
    H[m] = ((hi & 1 ? f45.x : -f45.x) + (hi & 2 ? f45.y : -f45.y)) +
           ((hi & 4 ? f67.x : -f67.x) + (hi & 8 ? f67.y : -f67.y));
  }
  const int hh = lane >> 4;
  const uint32_t col = slot_base + (uint32_t)hh * 65536u + 16u * (uint32_t)((lane & 15) ^ (4 * hh));
#pragma unroll
  for (int lo = 0; lo < 16; ++lo)
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(col + ((warp * 16 + lo) << 8)), "f"(L[0][lo] + H[0]),
                 "f"(L[1][lo] + H[1]), "f"(L[2][lo] + H[2]), "f"(L[3][lo] + H[3]) : "memory");
}

template <int Q>
__device__ __forceinline__ float4 unit_dot_m4(const uint4 (&w)[Q], const int (&e)[Q], const uint32_t (&cst)[16]) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = (j < 4) ? w[i].x : (j < 8) ? w[i].y : (j < 12) ? w[i].z : w[i].w;
      const float4 v = lds_f32x4(kDynBase + prmt(word, cst[j], step_sel_m4(j)));
      if (j == 0) {
        p = v;
      } else {
        p.x += v.x; p.y += v.y; p.z += v.z; p.w += v.w;
      }
    }
    const float v0 = shift_pow2(p.x, e[i]), v1 = shift_pow2(p.y, e[i]);
    const float v2 = shift_pow2(p.z, e[i]), v3 = shift_pow2(p.w, e[i]);
    if (i == 0) {
      acc = make_float4(v0, v1, v2, v3);
    } else {
      acc.x += v0; acc.y += v1; acc.z += v2; acc.w += v3;
    }
  }
  return acc;
}

template <int Q>
__global__ void __launch_bounds__((kRingNW + 1) * 32, 1)
gemm_cluster_ring_m4_kernel(const __half* __restrict__ x, int ldx, int M, const uint8_t* __restrict__ planes,
                            const int8_t* __restrict__ exps, int N, int S, int RG, int C, __half* __restrict__ y,
                            int ldy, int flags) {
  using RC = M2Cfg<Q>;
  constexpr int NW = kRingNW, NST = RC::nst;
  const bool pdl = flags & kFlagPdl;
  if (threadIdx.x == 0) check_dyn_base();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (NW + 1) * 32;
  const int r = lane >> 1, h = lane & 1;
  const uint32_t rank = cluster_rank();
  const unsigned Cu = (unsigned)C, ncl = gridDim.x / Cu, cl = blockIdx.x / Cu;
  const int rg0 = (int)((cl * (unsigned)RG) / ncl);
  const int RGb = (int)(((cl + 1) * (unsigned)RG) / ncl) - rg0;
  const int s0 = (int)((rank * (unsigned)S) / Cu);
  const int Sc = (int)(((rank + 1) * (unsigned)S) / Cu) - s0;   // 1 (C = S)
  const int Mc = Sc * RGb;
  if (pdl) pdl_launch_dependents();

  const uint32_t base = dyn_smem_base_cluster();
  const uint32_t xs = base + M4Map::lut;
  const uint32_t recv = xs + M4Map::xstage;
  const uint32_t bar = base + M4Map::bar;
  const uint32_t ring = base + (uint32_t)M4Map::base;
  const uint32_t full = ring + RC::bars, empty = full + 64;
  const int chunk_rg = (RGb + C - 1) / C;
  const int chunk = chunk_rg * kTileRows;
  const int rows = RGb * kTileRows;
  const int own_lo = (int)rank * chunk;
  const int cnt = rows - own_lo < chunk ? (rows - own_lo > 0 ? rows - own_lo : 0) : chunk;
  const float inv_chunk_rg = 1.f / (float)chunk_rg;
  if (tid == 0) {
    mbar_init_expect(bar, (uint32_t)(4 * (S - Sc) * cnt * 4));
    for (int j = 0; j < NST; ++j) {
      rmbar_init(full + 8 * j, 1);
      rmbar_init(empty + 8 * j, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  cluster_arrive_relaxed();
  const int nstages = (Mc + NW - 1) / NW;

  if (warp == NW) {
    if (lane == 0) {   // producer: one slice, contiguous units
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < nstages; ++t) {
        const int j = t % NST;
        if (t >= NST) rmbar_wait(empty + 8 * j, (uint32_t)((t / NST - 1) & 1));
        const int i0 = t * NW, i1 = i0 + NW < Mc ? i0 + NW : Mc;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * j),
                     "r"((uint32_t)((i1 - i0) * Q * (kTileBytes + kTileExps))) : "memory");
        const long long u = (long long)s0 * RG + rg0 + i0;
        const uint32_t dst = ring + (uint32_t)(j * RC::stage);
        bulk_load_x(dst, planes + u * Q * kTileBytes, (uint32_t)((i1 - i0) * Q * kTileBytes), full + 8 * j, pol,
                    false);
        bulk_load_x(dst + (uint32_t)RC::stage_planes, exps + u * Q * kTileExps, (uint32_t)((i1 - i0) * Q * kTileExps),
                    full + 8 * j, pol, false);
      }
    }
  } else {
    if (pdl) pdl_wait();
    if (tid < 4 * (kTileK / 8)) {   // x rows 0..3 of the slice (rows >= M are zero)
      const int m = tid >> 5, c = tid & 31;
      uint4 xv = make_uint4(0, 0, 0, 0);
      if (m < M)
        xv = ldg_keep(reinterpret_cast<const uint4*>(x + (size_t)m * ldx + (size_t)s0 * kTileK) + c,
                      policy_evict_last());
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(xs + (uint32_t)(m * kTileK * 2 + 16 * c)),
                   "r"(xv.x), "r"(xv.y), "r"(xv.z), "r"(xv.w) : "memory");
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    build_lut_slot_m4(base, xs, warp, lane);
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    cluster_wait();
    uint32_t cst[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      cst[j] = (16u * (uint32_t)(((j + r) & 15) ^ (4 * h))) | ((uint32_t)h << 16) | (rank << 24);
    for (int t = 0; t < nstages; ++t) {
      const int j = t % NST;
      const int i = t * NW + warp;
      rmbar_wait(full + 8 * j, (uint32_t)((t / NST) & 1));
      if (i < Mc) {
        uint4 w[Q];
        int e[Q];
        const uint32_t sp = ring + (uint32_t)(j * RC::stage + warp * Q * kTileBytes + 16 * lane);
        const uint32_t se = ring + (uint32_t)(j * RC::stage + RC::stage_planes + warp * Q * kTileExps + lane);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          smem_check(sp + (uint32_t)(k * kTileBytes), 16);
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[k].x), "=r"(w[k].y), "=r"(w[k].z),
                       "=r"(w[k].w) : "r"(sp + (uint32_t)(k * kTileBytes)));
          smem_check(se + (uint32_t)(k * kTileExps), 1);
          asm volatile("ld.shared.s8 %0, [%1];" : "=r"(e[k]) : "r"(se + (uint32_t)(k * kTileExps)));
        }
        float4 v = unit_dot_m4<Q>(w, e, cst);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
        v.z += __shfl_xor_sync(0xffffffffu, v.z, 1);
        v.w += __shfl_xor_sync(0xffffffffu, v.w, 1);
        if (h == 0) {   // a5 push of the 4 rows' partials: recv[m][slice][row - o*chunk] of owner o
          const int rgl = i;
          const int o = (int)(((float)rgl + 0.5f) * inv_chunk_rg);
          const uint32_t d0 = recv + 4u * (uint32_t)(s0 * chunk + (rgl - o * chunk_rg) * kTileRows + r);
          const uint32_t ds = 4u * (uint32_t)(S * chunk);
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            if (o == (int)rank) sts_f32(d0 + m * ds, vv[m]);
            else st_async_f32(d0 + m * ds, bar, (uint32_t)o, vv[m]);
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * j) : "memory");
      }
    }
  }
  __syncthreads();
  mbar_wait_parity0(bar);
  for (int it = tid; it < M * cnt; it += NT) {   // the owner: rows 0..M-1 of its chunk, slices in order
    const int m = it / cnt, jj = it - m * cnt;
    const uint32_t rb = recv + 4u * (uint32_t)(m * S * chunk + jj);
    float v = lds_f32(rb);
    for (int s = 1; s < S; ++s) v += lds_f32(rb + 4u * (uint32_t)(s * chunk));
    const int n = rg0 * kTileRows + own_lo + jj;
    if (n < N) y[(size_t)m * ldy + n] = __float2half_rn(v);
  }
}

template <int Q>
cudaError_t launch_m4_q(const GemmArgs& a, const LaunchPlan& p, int C) {
  const cudaError_t err = once_per_device([] {
    cudaError_t err = cudaSuccess;
    err = cudaFuncSetAttribute(gemm_cluster_ring_m4_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               M4Map::total);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(gemm_cluster_ring_m4_kernel<Q>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return err;
  });
  if (err != cudaSuccess) return err;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(p.grid);
  c.blockDim = dim3((kRingNW + 1) * 32);
  c.dynamicSmemBytes = M4Map::total;
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
  return cudaLaunchKernelEx(&c, gemm_cluster_ring_m4_kernel<Q>, a.x, a.ldx, a.M, a.planes, a.exps, a.N, S, RG, C,
                            a.y, a.ldy, pdl ? kFlagPdl : 0);
}

// The launch choices below are fixed at their measured defaults; the library
// reads no environment.

// Variants (warps, LUT slots).  HALF: 8 warps x 128 registers and 2 slots (~90 KB of shared
// memory), so two CTAs share an SM -- when one finishes, a CTA of the next kernel on the
// stream takes its place and, under PDL, prefetches its weights while this kernel's tail
// (cluster barrier, reduction) runs.  FULL4: 16 warps, 4 slots (170 KB, one CTA per SM),
// for K up to 8192 with clusters of <= 8.
enum Variant { kHalf = 0, kFull2 = 1, kFull4 = 2, kColw = 3, kRing = 4, kRing16 = 5 };
struct ClusterShape {
  int variant;
  int sc;   // max slices per CTA
  int C;    // cluster size
};

ClusterShape cluster_shape(int N, int K, int q, bool allow16 = true) {
  (void)N; (void)q;
  (void)allow16;
  const int S = K / kTileK;
  const int sc = (S + 1) / 2 <= kMaxC ? 2 : kMaxSc;
  // (S + sc - 1) / sc may exceed the portable 8: clusters of up to 16 are non-portable
  const int variant = sc > 2 ? kFull4 : kRing;
  return ClusterShape{variant, sc, (S + sc - 1) / sc};
}

int variant_threads(int v) { return v == kHalf ? 8 * 32 : v >= kRing ? (kRingNW + 1) * 32 : 16 * 32; }
int variant_smem(int v) { return v == kFull4 ? Smem<4>::total : v >= kRing ? RingCfg<1>::smem : Smem<2>::total; }

template <int Q, bool H16 = false>
cudaError_t set_ring_attrs() {
  const cudaError_t err = once_per_device([] {
    cudaError_t err = cudaSuccess;
    err = cudaFuncSetAttribute(gemv_cluster_ring_kernel<Q, H16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               RingCfg<Q>::smem);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(gemv_cluster_ring_kernel<Q, H16>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return err;
  });
  return err;
}

int occupancy_ring_clusters(int C) {
  if (set_ring_attrs<2>() != cudaSuccess) return 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(C * 64);
  c.blockDim = dim3((kRingNW + 1) * 32);
  c.dynamicSmemBytes = RingCfg<2>::smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  c.attrs = &attr;
  c.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemv_cluster_ring_kernel<2, false>, &c) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return n;
}

template <int Q, int SCM, int NW, int REGS, bool COLW = false, bool AP2 = false>
cudaError_t set_attrs() {
  const cudaError_t err = once_per_device([] {
    cudaError_t err = cudaSuccess;
    err = cudaFuncSetAttribute(gemv_cluster_kernel<Q, SCM, NW, REGS, COLW, AP2>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<SCM>::total);
    if (err == cudaSuccess)   // clusters of up to 16 (column-wise; one slice per CTA)
      err = cudaFuncSetAttribute(gemv_cluster_kernel<Q, SCM, NW, REGS, COLW, AP2>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return err;
  });
  return err;
}

template <int SCM, int NW, bool COLW = false>
int occupancy_clusters(int C) {
  if (set_attrs<2, SCM, NW, 128, COLW>() != cudaSuccess) return 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(C * 64);
  c.blockDim = dim3(NW * 32);
  c.dynamicSmemBytes = Smem<SCM>::total;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  c.attrs = &attr;
  c.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemv_cluster_kernel<2, SCM, NW, 128, COLW, false>, &c) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return n;
}

// Max co-resident clusters of size C for a variant (cached).
int max_clusters(int variant, int C) {
  static int cache[6][kMaxCColw + 1] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  int& slot = cache[variant][C];
  if (slot) return slot;
  const int n = variant == kHalf    ? occupancy_clusters<2, 8>(C)
                : variant == kFull2 ? occupancy_clusters<2, 16>(C)
                : variant == kFull4 ? occupancy_clusters<4, 16>(C)
                : variant >= kRing  ? occupancy_ring_clusters(C)
                                    : occupancy_clusters<4, 16, true>(C);
  slot = n > 0 ? n : -1;
  return slot;
}


template <int Q, int SCM, int NW, int REGS, bool COLW = false, bool AP2 = false>
cudaError_t launch_cluster_q(const GemmArgs& a, const LaunchPlan& p, int C) {
  const cudaError_t ae = set_attrs<Q, SCM, NW, REGS, COLW, AP2>();
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
  // ring slots requested before griddepcontrol.wait: ~pre_kb KB per CTA (what HBM delivers
  // to an SM's share during the wait; more only delays x, which queues behind them)
  constexpr int D = COLW ? cl_ring_colw(Q, REGS) : (AP2 ? cl_ring_ap2(Q, REGS) : cl_ring(Q, REGS));
  constexpr int pre_kb = 1024;
  const int slot_bytes = (p.threads / 32) * Q * kTileBytes;
  int pre = (pre_kb * 1024 + slot_bytes / 2) / slot_bytes;
  pre = pre < 0 ? 0 : (pre > D ? D : pre);
  // pushes at the end for 4-slot CTAs (measured), in the loop otherwise
  const int flags = (pdl ? kFlagPdl : 0) | (pre << kPreShift) | (SCM > 2 ? kFlagPushEnd : 0);
  return cudaLaunchKernelEx(&c, gemv_cluster_kernel<Q, SCM, NW, REGS, COLW, AP2>, a.x,
                            reinterpret_cast<const uint4*>(a.planes), a.exps, a.N, S, RG, C, a.y, flags, trace,
                            a.exps2, a.gather);
}

template <int Q, bool H16>
cudaError_t launch_ring_q(const GemmArgs& a, const LaunchPlan& p, int C) {
  const cudaError_t ae = set_ring_attrs<Q, H16>();
  if (ae != cudaSuccess) return ae;
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const int pdl = (a.flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(p.grid);
  c.blockDim = dim3((kRingNW + 1) * 32);
  c.dynamicSmemBytes = RingCfg<Q>::smem;
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
  return cudaLaunchKernelEx(&c, gemv_cluster_ring_kernel<Q, H16>, a.x, a.planes, a.exps, a.N, S, RG, C, a.y,
                            pdl ? kFlagPdl : 0, trace, a.gather);
}

// Kernel 10 geometry: clusters of the ring kernel's shape for K; nullptr-free plan or C = 0.
int fused_cluster_grid(int K, int RGtot, int* C_out) {
  const int S = K / kTileK;
  if (S < 1 || (S + 1) / 2 > kMaxC) return 0;
  const int C = (S + 1) / 2;
  const int ncl = max_clusters(kRing, C);
  if (ncl <= 0) return 0;
  const int bands = ncl < RGtot ? ncl : RGtot;
  if ((RGtot + bands - 1) / bands > kMaxRGb) return 0;
  *C_out = C;
  return bands * C;
}

cudaError_t launch_fused_impl(const StreamLaunch& L, cudaStream_t stream) {
  const cudaError_t attr_err = once_per_device([] {
    cudaError_t attr_err = cudaSuccess;
    attr_err = cudaFuncSetAttribute(gemv_cluster_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    RingCfg<1>::smem);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(gemv_cluster_fused_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return attr_err;
  });
  if (attr_err != cudaSuccess) return attr_err;
  FusedArgs A = {};
  A.x = L.x;
  A.nseg = L.nseg;
  A.S = L.K / kTileK;
  int rg = 0, qmax = 1;
  for (int i = 0; i < L.nseg; ++i) {
    FusedSeg& d = A.seg[i];
    d.planes = L.seg[i].planes;
    d.exps = L.seg[i].exps;
    d.y = L.seg[i].y;
    d.q = L.seg[i].q;
    d.N = L.seg[i].N;
    d.RG = (d.N + kTileRows - 1) / kTileRows;
    d.rgoff = rg;
    rg += d.RG;
    qmax = d.q > qmax ? d.q : qmax;
  }
  A.RGtot = rg;
  int C = 0;
  const int grid = fused_cluster_grid(L.K, rg, &C);
  if (grid <= 0) return cudaErrorNotSupported;
  A.C = C;
  A.slot = kRingNW * qmax * (kTileBytes + kTileExps);
  A.slot_planes = kRingNW * qmax * kTileBytes;
  A.nst = (kRingBytes - 128) / A.slot > 8 ? 8 : (kRingBytes - 128) / A.slot;
  A.pdl = L.pdl;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(grid);
  c.blockDim = dim3((kRingNW + 1) * 32);
  c.dynamicSmemBytes = RingCfg<1>::smem;
  c.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = attr;
  c.numAttrs = L.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&c, gemv_cluster_fused_kernel, A);
}

template <int SCM, int NW, bool AP2 = false>
cudaError_t launch_cluster_v(const GemmArgs& a, const LaunchPlan& p, int C) {
  switch (a.q) {
    case 1: return launch_cluster_q<1, SCM, NW, 128, false, AP2>(a, p, C);
    case 2: return launch_cluster_q<2, SCM, NW, 128, false, AP2>(a, p, C);
    case 3: return launch_cluster_q<3, SCM, NW, 128, false, AP2>(a, p, C);
    case 4: return launch_cluster_q<4, SCM, NW, 128, false, AP2>(a, p, C);
    default: return cudaErrorInvalidValue;
  }
}

// NEXT-f3 consumer side: wait until every rank published call *epoch + 1 (acquire, system
// scope), then advance *epoch (the device call counter the producer reads).  Bounded: ~5 s
// without progress traps (an error, not a hung GPU).
__global__ void gather_wait_kernel(const uint32_t* __restrict__ flags, int P, uint32_t* __restrict__ epoch_ctr) {
  // Launched with PDL: it may start while the producing GEMV still runs (it only reads
  // flags, and this rank's own flag covers that GEMV's stores), and lets its dependents
  // start at once -- they call griddepcontrol.wait, i.e. wait for this kernel to finish.
  pdl_launch_dependents();
  // The epoch counter is advanced by the previous gather_wait and read by the GEMV it follows;
  // under PDL this kernel may start while that GEMV (and, transitively, the previous wait) is
  // still running, so read it only after griddepcontrol.wait.  (The wait itself is cheap: this
  // rank's own flag is published at the end of that GEMV anyway.)
  pdl_wait();
  const int r = threadIdx.x;
  const uint32_t epoch = *epoch_ctr + 1u;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (; r < P;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
    if ((int)(v - epoch) >= 0) break;
    __nanosleep(200);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 5000000000ull) __trap();
  }
  __syncwarp();
  if (r == 0) *epoch_ctr = epoch;
}

}  // namespace

// kernel 10 entry (shiftadd_lut_gemv_fused, K <= 4096): cudaErrorNotSupported if no cluster shape fits
cudaError_t launch_gemv_cluster_fused(const StreamLaunch& L, cudaStream_t stream) { return launch_fused_impl(L, stream); }
bool fused_cluster_ok(int K, int RGtot) {
  int C = 0;
  return fused_cluster_grid(K, RGtot, &C) > 0;
}

cudaError_t launch_gather_wait(const uint32_t* flags, int P, uint32_t* epoch, cudaStream_t stream) {
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(1);
  c.blockDim = dim3(32);
  c.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  c.attrs = &attr;
  c.numAttrs = 1;
  return cudaLaunchKernelEx(&c, gather_wait_kernel, flags, P, epoch);
}

// Clusters of <= 4 pack 132 of the 148 SMs; of 5-8 fewer (120 at C = 8, measured), which
// costs more than the grid split-K's hand-off once the layer streams long enough: C > 4 only
// for layers up to kBigC bytes of planes (measured: 2048x8192 q=3 6.2 vs 8.4 us, 8192^2 q=2
// a tie, 28672x8192 q=3 27.7 vs 24.3 us).
constexpr double kBigC = 12.0 * (1 << 20);

bool cluster_applicable(int N, int K, int q, int sms) {
  (void)sms;
  const int S = K / kTileK;
  if (S < 1) return false;
  const ClusterShape cs = cluster_shape(N, K, q);
  if (cs.C > kMaxCColw) return false;
  if (cs.variant == kFull4 && cs.C > 4 && (double)q * N * K / 8 > kBigC) return false;
  const int ncl = max_clusters(cs.variant, cs.C);
  if (ncl <= 0) return false;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int bands = ncl < RG ? ncl : RG;
  return (RG + bands - 1) / bands <= kMaxRGb;
}

// 4-slot (K > 4096) cluster shapes: the TMA-ring grid split-K kernel is faster where it
// applies (measured: LLaMA-2-7B down 4096x11008 q=2 8.5 vs 11.3 us).
bool cluster_is_4slot(int N, int K, int q) { return cluster_shape(N, K, q).variant == kFull4; }

LaunchPlan plan_gemv_cluster(int N, int K, int q, int sms) {
  (void)sms;
  const ClusterShape cs = cluster_shape(N, K, q);
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int ncl = max_clusters(cs.variant, cs.C);
  const int bands = ncl < RG ? ncl : RG;
  return LaunchPlan{bands * cs.C, variant_threads(cs.variant), variant_smem(cs.variant), 3};
}

// NEXT-f1: column-wise scales.  One slice per CTA (its q LUT slots are the q planes' banks),
// so C = S; clusters of up to 16 (non-portable) cover K <= 4096.
bool colwise_applicable(int N, int K, int q) {
  const int S = K / kTileK;
  if (K % kTileK || S < 1 || S > kMaxCColw || q < 1 || q > 4) return false;
  const int ncl = max_clusters(kColw, S);
  if (ncl <= 0) return false;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int bands = ncl < RG ? ncl : RG;
  return (RG + bands - 1) / bands <= kMaxRGbColw;
}

cudaError_t launch_gemv_colwise(const GemmArgs& a) {
  const int S = a.K / kTileK;
  const int RG = (a.N + kTileRows - 1) / kTileRows;
  const int ncl = max_clusters(kColw, S);
  if (ncl <= 0) return cudaErrorNotSupported;
  const int bands = ncl < RG ? ncl : RG;
  const LaunchPlan p{bands * S, 16 * 32, Smem<4>::total, 4};
  switch (a.q) {
    case 1: return launch_cluster_q<1, 4, 16, 128, true>(a, p, S);
    case 2: return launch_cluster_q<2, 4, 16, 128, true>(a, p, S);
    case 3: return launch_cluster_q<3, 4, 16, 128, true>(a, p, S);
    case 4: return launch_cluster_q<4, 4, 16, 128, true>(a, p, S);
    default: return cudaErrorInvalidValue;
  }
}

// §8 a7, M = 2 (kernel id 5): tiled layout, K <= 4096, q <= 3 (a 60 KB ring holds >= 2 stages).
bool m2_applicable(int N, int K, int q, int sms) {
  (void)sms;
  const int S = K / kTileK;
  if (S < 1 || S > 2 * kMaxC || q < 1 || q > 3) return false;
  const int C = (S + 1) / 2;
  const int ncl = max_clusters(kRing, C);
  if (ncl <= 0) return false;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int bands = ncl < RG ? ncl : RG;
  return (RG + bands - 1) / bands <= kMaxRGb;
}

LaunchPlan plan_gemm_m2(int N, int K, int q, int sms) {
  (void)q; (void)sms;
  const int S = K / kTileK, C = (S + 1) / 2;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int ncl = max_clusters(kRing, C);
  const int bands = ncl < RG ? ncl : RG;
  return LaunchPlan{bands * C, (kRingNW + 1) * 32, M2Map::total, 5};
}

cudaError_t launch_gemm_m2(const GemmArgs& a, const LaunchPlan& p) {
  const int C = (a.K / kTileK + 1) / 2;
  switch (a.q) {
    case 1: return launch_m2_q<1>(a, p, C);
    case 2: return launch_m2_q<2>(a, p, C);
    case 3: return launch_m2_q<3>(a, p, C);
    default: return cudaErrorInvalidValue;
  }
}

// §8 a7, M = 3..4 (kernel id 6): tiled layout, K <= 4096 (one slice per CTA), q <= 3.
bool m4_applicable(int N, int K, int q, int sms) {
  (void)sms;
  const int S = K / kTileK;
  if (S < 1 || S > kMaxCColw || q < 1 || q > 3) return false;
  const int ncl = max_clusters(kRing, S);
  if (ncl <= 0) return false;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int bands = ncl < RG ? ncl : RG;
  return (RG + bands - 1) / bands <= kMaxRGb;
}

LaunchPlan plan_gemm_m4(int N, int K, int q, int sms) {
  (void)q; (void)sms;
  const int S = K / kTileK;
  const int RG = (N + kTileRows - 1) / kTileRows;
  const int ncl = max_clusters(kRing, S);
  const int bands = ncl < RG ? ncl : RG;
  return LaunchPlan{bands * S, (kRingNW + 1) * 32, M4Map::total, 6};
}

cudaError_t launch_gemm_m4(const GemmArgs& a, const LaunchPlan& p) {
  const int C = a.K / kTileK;
  switch (a.q) {
    case 1: return launch_m4_q<1>(a, p, C);
    case 2: return launch_m4_q<2>(a, p, C);
    case 3: return launch_m4_q<3>(a, p, C);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemv_cluster(const GemmArgs& a, const LaunchPlan& p) {
  ClusterShape cs = cluster_shape(a.N, a.K, a.q);
  if ((cs.variant == kRing || cs.variant == kRing16) && !a.exps2 && !(reinterpret_cast<uintptr_t>(a.exps) & 15)) {
    const bool h16 = cs.variant == kRing16;
    switch (a.q) {   // the TMA ring (its bulk copies need 16-B aligned exponent tiles)
      case 1: return h16 ? launch_ring_q<1, true>(a, p, cs.C) : launch_ring_q<1, false>(a, p, cs.C);
      case 2: return h16 ? launch_ring_q<2, true>(a, p, cs.C) : launch_ring_q<2, false>(a, p, cs.C);
      case 3: return h16 ? launch_ring_q<3, true>(a, p, cs.C) : launch_ring_q<3, false>(a, p, cs.C);
      case 4: return h16 ? launch_ring_q<4, true>(a, p, cs.C) : launch_ring_q<4, false>(a, p, cs.C);
      default: return cudaErrorInvalidValue;
    }
  }
  LaunchPlan pp = p;
  if (cs.variant == kRing16) cs = cluster_shape(a.N, a.K, a.q, false);
  if (cs.variant == kRing) {   // register-ring kernel instead: its own launch shape
    const int RG = (a.N + kTileRows - 1) / kTileRows;
    const int ncl = max_clusters(kFull2, cs.C);
    if (ncl <= 0) return cudaErrorNotSupported;
    const int bands = ncl < RG ? ncl : RG;
    if ((RG + bands - 1) / bands > kMaxRGb) return cudaErrorNotSupported;
    pp = LaunchPlan{bands * cs.C, variant_threads(kFull2), variant_smem(kFull2), 3};
  }
  if (a.exps2)   // NEXT-f2: additive PoT K = 2 (16-warp variants only)
    return cs.sc <= 2 ? launch_cluster_v<2, 16, true>(a, pp, cs.C) : launch_cluster_v<4, 16, true>(a, pp, cs.C);
  switch (cs.variant) {
    case kHalf: return launch_cluster_v<2, 8>(a, pp, cs.C);
    case kFull2:
    case kRing: return launch_cluster_v<2, 16>(a, pp, cs.C);
    default: return launch_cluster_v<4, 16>(a, pp, cs.C);
  }
}

}  // namespace shiftadd
