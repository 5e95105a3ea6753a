// lut_program.cu -- a whole decode step of LUT-GEMV calls in one persistent launch (kernel id 9).
//
// A "program" is an ordered list of calls, each the fused-segment LUT-GEMV of lut_stream.cu
// (one x, 1..4 output segments with their own q: LLaMA q/k/v, o, gate/up, down), for one
// token's pass over the model (§8 a2-a6 over BASELINE configs[2]).  One CTA per SM runs
// every call in order:
//
//  * the producer warp streams the weights of call after call through the shared-memory
//    ring with 1-D bulk copies, never waiting on activations -- the weights of call j+1
//    land in the ring while call j is still being reduced, and HBM stays busy across the
//    call boundaries that a kernel-per-call chain pays for with a launch, a PDL wait and a
//    cold first stage;
//  * the 16 consumer warps, per call: wait for the call's dependency (SHIFTADD_CALL_WAIT:
//    every earlier call has stored its y -- a decoder's next projection reads the previous
//    one's output), read x, build the (at most two) slice LUTs (a2), query the ring (a3 +
//    a4), publish epoch-tagged split-K partials, reduce the rows they own in slice order and
//    store fp16 y (a5), then count the call complete.
//
// Work split, LUT build, lookup loop and split-K words are those of kernel 8 (lut_stream.cu):
// CTA c takes the units whose weight offset lies in [c W/G, (c+1) W/G) of the call.
//
// Completion counter (workspace word 0, 64 bit): every CTA adds 1 per call after storing its
// owned rows (release); a launch's adds total exactly 2^32 (CTA 0 adds 2^32 - ncalls G after
// its last call), so (counter >> 32) read at kernel start is the launch number L and every
// proper subset of a launch's adds stays below the next multiple of 2^32.  Call j's
// dependency is "counter >= (L << 32) + j G"; calls without SHIFTADD_CALL_WAIT still wait for
// call j-2 (its partial region is reused by call j).  Partial words carry the 32-bit tag
// L ncalls + j + 1 and alternate between two regions by call parity.
#include <mutex>

#include "stream_dev.cuh"

namespace shiftadd {
namespace {
using namespace stream_dev;

constexpr int kNWC = 16;                    // consumer warps
constexpr int kNC = kNWC * 32;              // consumer threads
constexpr int kRingOff = kLutBytes;         // ring after the 64 KB LUT slab
constexpr int kProgBarBytes = 256;          // full[16] at +0, empty[16] at +128
constexpr int kScratchFloats = kNC;         // owner-phase partial row sums
constexpr uint64_t kProgMagic = 0x3130325347525053ull;   // "SPRGS201"

#ifdef SHIFTADD_DEV_TRACE
// development builds only: globaltimer stamps [CTA][call][8] (tools/trace_program.py)
__device__ unsigned long long* g_ptrace = nullptr;
__device__ __forceinline__ void ptrace(long long c, int ncalls, int j, int k) {
  if (g_ptrace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_ptrace[((size_t)c * ncalls + j) * 8 + k] = t;
  }
}
__device__ int g_pvariant = 0;
#else
__device__ __forceinline__ void ptrace(long long, int, int, int) {}
#endif

struct ProgSeg {
  const uint8_t* planes;
  const int8_t* exps;
  __half* y;
  int q, N, RG, rgoff, woff, pad;
};
struct ProgCall {
  const __half* x;
  int S, nseg, RGtot, Ws, wait, pad;
  ProgSeg seg[kMaxSegments];
};
struct ProgHeader {
  uint64_t magic, hash;
  int ncalls, pad[11];
};
static_assert(sizeof(ProgHeader) == 64, "header size");

struct ProgParams {
  const ProgHeader* hdr;
  const ProgCall* calls;
  int ncalls;
  uint64_t hash;
  unsigned long long* ctr;
  unsigned long long* part[2];
  size_t part_words;   // words per region (bounds-checked builds)
  int nst, slot, slot_planes;
};

__device__ __forceinline__ uint4 ldg_cg_u4(const void* p) {   // L2 only: x may be written by this launch
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"r"(kNC) : "memory"); }

struct Ring {
  uint32_t base, full, empty;
  int nst, slot, slot_planes;
};

// Consumer side of one run (slice s, segment sg, row groups [rga, re)) -- kernel 8's pairing:
// warp w takes unit w of stages t and t + 1 together; the upper half of the warps starts with
// one stage alone so the two halves' barrier waits interleave.
template <int Q, uint32_t HOFF>
__device__ __forceinline__ void consume_run(const ProgSeg& sg, int S, int s, int rga, int re, RingPos& rp,
                                            const Ring& R, const uint32_t (&cst)[4], int wu, int lane,
                                            unsigned long long ep, unsigned long long* part, size_t part_words,
                                            bool skew) {
  const int r = lane >> 1, h = lane & 1;
  unsigned long long* prow = part + ((size_t)sg.rgoff * S + s) * kTileRows + r;
  bool single = skew;
  for (int rg = rga; rg < re;) {
    const int n0 = re - rg < 16 ? re - rg : 16;
    const int left = re - rg - n0;
    const int n1 = single ? 0 : (left < 16 ? left : 16);
    single = false;
    const RingPos r0 = rp;
    rp.next(R.nst);
    const RingPos r1 = rp;
    if (n1 > 0) rp.next(R.nst);
    const uint32_t slot0 = R.base + (uint32_t)(r0.j * R.slot), slot1 = R.base + (uint32_t)(r1.j * R.slot);
    mbar_wait(R.full + 8 * r0.j, (uint32_t)(r0.k & 1));
    if (n1 > 0) mbar_wait(R.full + 8 * r1.j, (uint32_t)(r1.k & 1));
    const bool u0 = wu < n0, u1 = wu < n1;
    float acc[2] = {0.f, 0.f};
    if (u0)
      unit_dot2<Q, HOFF>(slot0 + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                         slot0 + (uint32_t)(R.slot_planes + wu * Q * kTileExps + lane),
                         slot1 + (uint32_t)(wu * Q * kTileBytes + 16 * lane),
                         slot1 + (uint32_t)(R.slot_planes + wu * Q * kTileExps + lane), u1, cst, acc);
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(R.empty + 8 * r0.j);
      if (n1 > 0) mbar_arrive(R.empty + 8 * r1.j);
    }
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
    acc[1] += __shfl_xor_sync(0xffffffffu, acc[1], 1);
    if (h == 0) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k == 0 ? u0 : u1) {
          const int u = rg + k * 16 + wu;
          if (S == 1) {
            const int nl = u * kTileRows + r;
            if (nl < sg.N) sg.y[nl] = __float2half_rn(acc[k]);
          } else {
            unsigned long long* const q = prow + (size_t)u * S * kTileRows;
#ifdef SHIFTADD_BOUNDS_CHECK
            if (q < part || q >= part + part_words) __trap();
#endif
            st_relaxed_u64(q, ep | __float_as_uint(acc[k]));
          }
        }
      }
    }
    rg += n0 + (n1 > 0 ? n1 : 0);
  }
}

template <uint32_t HOFF>
__device__ __forceinline__ void consume_run_q(const ProgSeg& sg, int S, int s, int rga, int re, RingPos& rp,
                                              const Ring& R, const uint32_t (&cst)[4], int wu, int lane,
                                              unsigned long long ep, unsigned long long* part, size_t part_words,
                                              bool skew) {
  switch (sg.q) {
    case 1: consume_run<1, HOFF>(sg, S, s, rga, re, rp, R, cst, wu, lane, ep, part, part_words, skew); break;
    case 2: consume_run<2, HOFF>(sg, S, s, rga, re, rp, R, cst, wu, lane, ep, part, part_words, skew); break;
    case 3: consume_run<3, HOFF>(sg, S, s, rga, re, rp, R, cst, wu, lane, ep, part, part_words, skew); break;
    default: consume_run<4, HOFF>(sg, S, s, rga, re, rp, R, cst, wu, lane, ep, part, part_words, skew); break;
  }
}

// CTA c's weight range of call cl (units assigned by their starting weight offset)
__device__ __forceinline__ void cta_range(const ProgCall& cl, long long c, long long G, Pos& a, Pos& b) {
  const long long W = (long long)cl.S * cl.Ws;
  a = pos_at(cl, split_point(c, W, G));
  b = pos_at(cl, split_point(c + 1, W, G));
}

// x of a call into L2 ahead of its dependency wait: a prefetch is only a hint (L2 is the point
// of coherence, the real load comes after the acquire), so it is correct even when x is being
// written by the calls before it, and it takes the cold miss off the chain.  Threads 0..7: the
// 512 B of the CTA's first slice and of its second, 128 B each.
__device__ __forceinline__ void prefetch_x(const ProgCall& cl, long long c, long long G, int tid) {
  if (tid < 8) {
    Pos a, b;
    cta_range(cl, c, G, a, b);
    const int s = a.s + (tid >> 2);
    if (s < cl.S && before(a, b))
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(cl.x + (size_t)s * kTileK + 64 * (tid & 3)));
  }
}

__global__ void __launch_bounds__((kNWC + 1) * 32, 1) lut_program_kernel(const __grid_constant__ ProgParams pp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long G = gridDim.x, c = blockIdx.x;
  const Ring R{kDynBase + (uint32_t)kRingOff, kDynBase + (uint32_t)(kRingOff + pp.nst * pp.slot),
               kDynBase + (uint32_t)(kRingOff + pp.nst * pp.slot) + 128u, pp.nst, pp.slot, pp.slot_planes};
  float* red = reinterpret_cast<float*>(shiftadd_dyn_smem + kRingOff + pp.nst * pp.slot + kProgBarBytes);
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(red + kScratchFloats);
  // the consumers' copies of the current and the next call descriptor (global reads after an
  // acquire would miss in L1 on every field)
  ProgCall* s_call = reinterpret_cast<ProgCall*>(s_base + 8);
  constexpr int kCallWords = (int)(sizeof(ProgCall) / 4);
  static_assert(sizeof(ProgCall) % 16 == 0 && kCallWords <= kNC, "descriptor copy");
  if (tid == 0) {
    check_dyn_base();
    // the device copy of the program must be the encoding of the calls this launch was
    // validated against
    if (pp.hdr->magic != kProgMagic || pp.hdr->hash != pp.hash || pp.hdr->ncalls != pp.ncalls) __trap();
    for (int j = 0; j < pp.nst; ++j) {
      mbar_init(R.full + 8 * j, 1);
      mbar_init(R.empty + 8 * j, 16);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    *s_base = ld_acquire_u64(pp.ctr) & ~0xffffffffull;   // (launch number L) << 32
    s_base[1] = 0;
  }
  if (tid < kCallWords)
    reinterpret_cast<uint32_t*>(s_call)[tid] = __ldg(reinterpret_cast<const uint32_t*>(pp.calls) + tid);
  __syncthreads();
  prefetch_x(s_call[0], c, G, tid);

  if (warp == kNWC) {
    // producer: the weights of every call, in order, through the ring (16 units per stage)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos rp{0, 0};
      for (int j = 0; j < pp.ncalls; ++j) {
        const ProgCall& cl = pp.calls[j];
        Pos a, end;
        cta_range(cl, c, G, a, end);
        bool first = true;
#ifdef SHIFTADD_DEV_TRACE
        if ((g_pvariant & 1) && j > 0) {   // experiment: no prefetch across the call boundary
          volatile unsigned* cur = reinterpret_cast<volatile unsigned*>(s_base + 1);
          while (*cur < (unsigned)j) __nanosleep(20);
        }
#endif
        while (before(a, end)) {
          const int re = run_end(cl, a, end);
          const ProgSeg& sg = cl.seg[a.g];
          const size_t ub = (size_t)a.s * sg.RG;
          for (int rg = a.rg; rg < re; rp.next(pp.nst)) {
            if (rp.k > 0) mbar_wait(R.empty + 8 * rp.j, (uint32_t)((rp.k - 1) & 1));
            if (first) {
              ptrace(c, pp.ncalls, j, 6);
              first = false;
            }
#ifdef SHIFTADD_DEV_TRACE
            if (g_pvariant & 2) {   // experiment: no copies while the consumers are in a call's chain
              volatile unsigned* ph = reinterpret_cast<volatile unsigned*>(s_base + 1) + 1;
              while (*ph) __nanosleep(20);
            }
#endif
            const int n = re - rg < 16 ? re - rg : 16;
            const uint32_t bp = (uint32_t)(n * sg.q * kTileBytes), be = (uint32_t)(n * sg.q * kTileExps);
            const uint32_t fb = R.full + 8 * rp.j;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(bp + be) : "memory");
            const uint32_t dst = R.base + (uint32_t)(rp.j * pp.slot);
            bulk_g2s(dst, sg.planes + (ub + rg) * sg.q * kTileBytes, bp, fb, pol);
            bulk_g2s(dst + (uint32_t)pp.slot_planes, sg.exps + (ub + rg) * sg.q * kTileExps, be, fb, pol);
            rg += n;
          }
          next_run(cl, a, re);
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  const unsigned long long base = *s_base;
  const unsigned tag0 = (unsigned)((base >> 32) * (unsigned long long)pp.ncalls);
  const int r = lane >> 1, h = lane & 1;
  uint32_t cst[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) v |= (4u * (uint32_t)(16 * h + ((4 * k + b + r) & 15))) << (8 * b);
    cst[k] = v;
  }
  const bool skew = warp >= kNWC / 2;
  RingPos rp{0, 0};
  for (int j = 0; j < pp.ncalls; ++j) {
    const ProgCall& cl = s_call[j & 1];
    // the next descriptor, into registers now and into the other buffer after the LUT build
    uint32_t nxt = 0;
    if (j + 1 < pp.ncalls && tid < kCallWords)
      nxt = __ldg(reinterpret_cast<const uint32_t*>(pp.calls + j + 1) + tid);
    if (tid == 0) ptrace(c, pp.ncalls, j, 0);
    // dependency: calls 0..need-1 complete (need = j with SHIFTADD_CALL_WAIT, else j - 1 so
    // that call j - 2's partial region -- reused by this call -- has been read)
    const int need = cl.wait ? j : j - 1;
    if (need > 0) {
      if (tid == 0) {
        const unsigned long long target = base + (unsigned long long)need * (unsigned long long)G;
        unsigned spins = 0;
        while (ld_acquire_u64(pp.ctr) < target) {
          if (++spins > (1u << 26)) __trap();   // a non-resident CTA: never hang silently
          __nanosleep(32);
        }
      }
      consumers_sync();
    }
    if (tid == 0) ptrace(c, pp.ncalls, j, 1);
#ifdef SHIFTADD_DEV_TRACE
    if (tid == 0) *reinterpret_cast<volatile unsigned*>(s_base + 1) = (unsigned)j;
#endif
    Pos start, end;
    cta_range(cl, c, G, start, end);
    const int S = cl.S;
    const int s0 = start.s;
    const bool any = before(start, end);
    const bool two = end.s > s0 && !(end.s == s0 + 1 && end.g == 0 && end.rg == 0);
    if (any) {
      const uint4 xa = ldg_cg_u4(cl.x + (size_t)s0 * kTileK + 8 * lane);
      uint4 xb = xa;
      if (two) xb = ldg_cg_u4(cl.x + (size_t)(s0 + 1) * kTileK + 8 * lane);
#ifdef SHIFTADD_DEV_TRACE
      if (tid == 0 && xa.x + 1u != 0u) ptrace(c, pp.ncalls, j, 7);   // x arrived (tid 0)
#endif
      build_lut<kNWC>(xa, 0u, warp, lane);
      if (two) build_lut<kNWC>(xb, 128u, warp, lane);
    }
    if (j + 1 < pp.ncalls && tid < kCallWords) reinterpret_cast<uint32_t*>(s_call + ((j + 1) & 1))[tid] = nxt;
    consumers_sync();
    if (tid == 0) ptrace(c, pp.ncalls, j, 2);
#ifdef SHIFTADD_DEV_TRACE
    if (tid == 0) reinterpret_cast<volatile unsigned*>(s_base + 1)[1] = 0u;
#endif
    if (j + 1 < pp.ncalls) prefetch_x(s_call[(j + 1) & 1], c, G, tid);
    const unsigned tag = tag0 + (unsigned)j + 1u;
    const unsigned long long ep = (unsigned long long)tag << 32;
    unsigned long long* part = pp.part[j & 1];
    for (Pos a = start; before(a, end);) {
      const int re = run_end(cl, a, end);
      if (a.s == s0)
        consume_run_q<0u>(cl.seg[a.g], S, a.s, a.rg, re, rp, R, cst, warp, lane, ep, part, pp.part_words, skew);
      else
        consume_run_q<128u>(cl.seg[a.g], S, a.s, a.rg, re, rp, R, cst, warp, lane, ep, part, pp.part_words, skew);
      next_run(cl, a, re);
    }
    if (tid == 0) ptrace(c, pp.ncalls, j, 3);
#ifdef SHIFTADD_DEV_TRACE
    if (tid == 0) reinterpret_cast<volatile unsigned*>(s_base + 1)[1] = 1u;
#endif

    if (S > 1) {
      // a5 owner phase: rows of the flattened row groups [c RGtot / G, (c+1) RGtot / G), T
      // threads per row over the slices in order (kernel 8's scheme)
      const int og0 = (int)((unsigned)c * (unsigned)cl.RGtot / (unsigned)G);   // 32-bit: G <= 256, RGtot <= 65536
      const int og1 = (int)((unsigned)(c + 1) * (unsigned)cl.RGtot / (unsigned)G);
      const int MR = (og1 - og0) * kTileRows;
      for (int rb = 0; rb < MR; rb += kNC) {
        const int CR = MR - rb < kNC ? MR - rb : kNC;
        int T = kNC / CR;
        T = T > S ? S : T;
        if (tid < CR * T) {
          const int row = rb + tid % CR, prt = tid / CR;
          const unsigned long long* pw = part + ((size_t)(og0 + row / kTileRows) * S) * kTileRows + (row % kTileRows);
          float sum = 0.f;
          for (int t0 = prt; t0 < S; t0 += 8 * T) {
            unsigned long long v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = t0 + k * T < S ? ld_relaxed_u64(pw + (size_t)(t0 + k * T) * kTileRows) : 0ull;
            unsigned spins = 0;
            for (;;) {
              bool stale = false;
#pragma unroll
              for (int k = 0; k < 8; ++k) stale |= t0 + k * T < S && (unsigned)(v[k] >> 32) != tag;
              if (!stale) break;
              if (++spins > (1u << 24)) __trap();
              __nanosleep(32);
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (t0 + k * T < S && (unsigned)(v[k] >> 32) != tag) v[k] = ld_relaxed_u64(pw + (size_t)(t0 + k * T) * kTileRows);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (t0 + k * T < S) sum += __uint_as_float((unsigned)v[k]);
          }
          red[tid] = sum;
        }
        consumers_sync();
        if (tid == 0) ptrace(c, pp.ncalls, j, 4);
        if (tid < CR) {
          float sum = red[tid];
          for (int t = 1; t < T; ++t) sum += red[t * CR + tid];
          const int nf = (og0 * kTileRows) + rb + tid;
          const int rgf = nf / kTileRows;
          int g = 0;
          while (g + 1 < cl.nseg && cl.seg[g + 1].rgoff <= rgf) ++g;
          const int nl = nf - cl.seg[g].rgoff * kTileRows;
          if (nl < cl.seg[g].N) cl.seg[g].y[nl] = __float2half_rn(sum);
        }
        if (rb + kNC < MR) consumers_sync();   // red is reused by the next chunk
      }
    }
    // call j complete in this CTA: its y stores (all consumer threads) before the count
    consumers_sync();
    if (tid == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(pp.ctr), "l"(1ull) : "memory");
      ptrace(c, pp.ncalls, j, 5);
    }
  }
  // this launch's adds total exactly 2^32 (see the header comment)
  if (tid == 0 && c == 0) {
    const unsigned long long add = (1ull << 32) - (unsigned long long)pp.ncalls * (unsigned long long)G;
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(pp.ctr), "l"(add) : "memory");
  }
}

#ifdef SHIFTADD_DEV_TRACE
}  // namespace
cudaError_t dev_set_program_trace(void* buf) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(g_ptrace, &p, sizeof p);
}
cudaError_t dev_set_program_variant(int v) { return cudaMemcpyToSymbol(g_pvariant, &v, sizeof v); }
namespace {
#endif

uint64_t fnv1a(const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

}  // namespace

size_t program_bytes(int ncalls) { return sizeof(ProgHeader) + (size_t)ncalls * sizeof(ProgCall); }

// Partial region (bytes) of one call: S x RGtot rows of 16 64-bit words, 0 without split-K.
size_t program_part_bytes(int S, int RGtot) { return S > 1 ? (size_t)S * RGtot * kTileRows * 8 : 0; }

size_t program_workspace_bytes(size_t part_max) { return 256 + 2 * ((part_max + 255) / 256 * 256); }

int program_qmax_stages(int qmax, int* smem) {
  const int slot = 16 * qmax * (kTileBytes + kTileExps);
  const int fixed = kLutBytes + kProgBarBytes + kScratchFloats * 4 + 64 + 2 * (int)sizeof(ProgCall);
  int nst = (227 * 1024 - fixed) / slot;
  nst = nst > 16 ? 16 : nst;
  *smem = fixed + nst * slot;
  return nst;
}

// Host encoding of validated calls (ProgCall array after a header); returns the hash.
uint64_t program_encode(const ProgramCallDesc* calls, int ncalls, void* out) {
  ProgHeader* hdr = static_cast<ProgHeader*>(out);
  ProgCall* pc = reinterpret_cast<ProgCall*>(hdr + 1);
  for (int j = 0; j < ncalls; ++j) {
    const ProgramCallDesc& d = calls[j];
    ProgCall cl = {};
    cl.x = d.x;
    cl.S = d.K / kTileK;
    cl.nseg = d.nseg;
    cl.wait = d.wait;
    int rg = 0, w = 0;
    for (int i = 0; i < d.nseg; ++i) {
      ProgSeg& s = cl.seg[i];
      s.planes = d.seg[i].planes;
      s.exps = d.seg[i].exps;
      s.y = d.seg[i].y;
      s.q = d.seg[i].q;
      s.N = d.seg[i].N;
      s.RG = (s.N + kTileRows - 1) / kTileRows;
      s.rgoff = rg;
      s.woff = w;
      rg += s.RG;
      w += s.q * s.RG;
    }
    cl.RGtot = rg;
    cl.Ws = w;
    pc[j] = cl;
  }
  ProgHeader h = {};
  h.magic = kProgMagic;
  h.ncalls = ncalls;
  h.hash = fnv1a(pc, (size_t)ncalls * sizeof(ProgCall));
  *hdr = h;
  return h.hash;
}

cudaError_t launch_lut_program(const void* program, int ncalls, uint64_t hash, int qmax, size_t part_max,
                               void* workspace, int sms, cudaStream_t stream) {
  int smem = 0;
  const int nst = program_qmax_stages(qmax, &smem);
  // kernel attributes are per device: set them once on each device that launches
  static std::once_flag once[64];
  static cudaError_t attr_err[64];
  int dev = 0;
  const cudaError_t de = cudaGetDevice(&dev);
  if (de != cudaSuccess) return de;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    attr_err[dev] = cudaFuncSetAttribute(lut_program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr_err[dev] != cudaSuccess) return attr_err[dev];
  ProgParams p = {};
  p.hdr = static_cast<const ProgHeader*>(program);
  p.calls = reinterpret_cast<const ProgCall*>(p.hdr + 1);
  p.ncalls = ncalls;
  p.hash = hash;
  char* ws = static_cast<char*>(workspace);
  const size_t region = (part_max + 255) / 256 * 256;
  p.ctr = reinterpret_cast<unsigned long long*>(ws);
  p.part[0] = reinterpret_cast<unsigned long long*>(ws + 256);
  p.part[1] = reinterpret_cast<unsigned long long*>(ws + 256 + region);
  p.part_words = region / sizeof(unsigned long long);
  p.nst = nst;
  p.slot = 16 * qmax * (kTileBytes + kTileExps);
  p.slot_planes = 16 * qmax * kTileBytes;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3((kNWC + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  // every CTA spins on the others: all of them must be co-resident (one per SM)
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lut_program_kernel, p);
}

}  // namespace shiftadd
