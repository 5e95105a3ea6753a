// common.cuh -- shared device helpers and internal launch interfaces of libshiftadd.
// Product code only: nothing here is shared with oracle/ (which is test infrastructure).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "shiftadd.h"

namespace shiftadd {

// Runs f() (kernel-attribute setup: attributes are per device) once on each device that
// launches, thread-safely, and returns its result for the current device.  Every call site
// passes its own lambda, so each gets its own flags.
template <class F>
cudaError_t once_per_device(F f) {
  static std::once_flag once[64];
  static cudaError_t err[64];
  int dev = 0;
  const cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [&] { err[dev] = f(); });
  return err[dev];
}

// Device-tiled layout geometry (include/shiftadd.h, SHIFTADD_LAYOUT_TILED).
constexpr int kTileRows = 16;    // output rows per tile
constexpr int kTileK = 256;      // reduction indices per tile (32 key bytes per row)
constexpr int kTileBytes = 512;  // 16 rows x 32 key bytes
constexpr int kTileExps = 32;    // 16 rows x 2 chunk exponents
// Split-K workspace: a 256 KB region of per-row-group arrival counters at offset 0 (every
// call leaves the counters it used zeroed, so a later call of any shape finds them zero),
// then the fp32 partials [M][S][Npad].
constexpr int kMaxRowGroups = 65536;
constexpr size_t kCounterBytes = (size_t)kMaxRowGroups * sizeof(unsigned);
constexpr int kMaxRows = kMaxRowGroups * kTileRows;

// LUT slab in shared memory for one 256-k slice: 256 keys x 64 words.  Word (key, col):
// cols 0..31 hold the 32 groups of an even slice segment, cols 32..63 of an odd one, so a
// CTA can build the next slice's LUT without waiting for the current one to drain.
constexpr int kLutBytes = 256 * 256;
}  // namespace shiftadd

// Dynamic shared memory as a named PTX symbol.  The kernels that use it declare no static
// shared memory, so their dynamic region starts right after the 1 KB the driver reserves at
// the bottom of every CTA's shared window: kDynBase.  Using that constant as the LUT base
// lets ptxas fold it into the LDS immediate -- LDS [R + 0x400] -- instead of spending an
// IADD per lookup on a base register; the kernels check the assumption once (trap if not).
extern "C" __shared__ __align__(16) unsigned char shiftadd_dyn_smem[];

namespace shiftadd {

constexpr uint32_t kDynBase = 0x400u;

__device__ __forceinline__ uint32_t dyn_smem_base() {
  asm volatile("" ::"l"(shiftadd_dyn_smem));  // reference the symbol so it is declared
  uint32_t b;
  asm("mov.u32 %0, shiftadd_dyn_smem;" : "=r"(b));
  // Bits 24+ of a shared::cta address carry the CTA's rank in its cluster; the kernels are
  // launched without clusters (rank 0), so the base is the constant window offset.
  return b & 0x00ffffffu;
}

__device__ __forceinline__ void check_dyn_base() {
  if (dyn_smem_base() != kDynBase) __trap();
}

// Bounds-checked debug builds (-DSHIFTADD_BOUNDS_CHECK, tools/check_build.sh; this pool has
// compute-sanitizer disabled): every shared-memory access through the wrappers below, every
// bulk-copy destination and DSMEM store, and every split-K partial word store traps if it
// leaves the launch's dynamic shared memory / the partial region.  Cluster-window addresses
// carry the rank in bits 24+, stripped before the check.  Product builds compile it away.
#ifdef SHIFTADD_BOUNDS_CHECK
__device__ __forceinline__ void smem_check(uint32_t addr, uint32_t bytes) {
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  const uint32_t a = addr & 0x00ffffffu;
  if (a < kDynBase || a + bytes > kDynBase + dyn || (a & (bytes >= 16 ? 15u : bytes - 1u))) __trap();
}
#else
__device__ __forceinline__ void smem_check(uint32_t, uint32_t) {}
#endif

// PTX prmt.b32 (default mode).  Unlike __byte_perm, the selector's per-nibble msb is honoured:
// it replicates the sign bit of the selected byte over the target byte.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
  smem_check(addr, 4);
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t addr) {
  smem_check(addr, 16);
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  smem_check(addr, 4);
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_f32x4(uint32_t addr, float4 v) {
  smem_check(addr, 16);
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// a4 -- the "shift" (App. H :974; DenseShift): p * 2^e as an integer add
// on the fp32 exponent field.  Guarded: +-0 stays 0 and Inf/NaN pass through; every other
// p this kernel produces is a normal fp32 (sums of fp16 values are multiples of 2^-24, so
// |p| >= 2^-24, and |p| <= 2^24 for one 128-k chunk) and e in [-100, 100] keeps p * 2^e
// normal, so the add is bit-identical to the multiply.  e == EXP_ZERO contributes 0.
__device__ __forceinline__ float shift_pow2(float p, int e) {
  const uint32_t b = __float_as_uint(p);
  const uint32_t ex = b & 0x7f800000u;
  const uint32_t r = ((ex - 0x00800000u) < 0x7f000000u) ? b + ((uint32_t)e << 23) : b;
  return (e == -128) ? 0.f : __uint_as_float(r);
}

// NEXT-f2 -- the second additive-PoT term (Eq. 2 with K = 2): given
// v1 = p * 2^{e1} and the code c2 = s1*s2*(P1 - P2), returns sign(c2) * v1 * 2^{-|c2|}
// (= s1 s2 p 2^{P2}): an exponent-field subtract.  c2 == 0 -> 0; Inf/NaN pass through; a
// result below the fp32 normal range (|.| < 2^-126) is flushed to 0 (reading R20).
__device__ __forceinline__ float shift_apot2(float v1, int c2) {
  const int d = c2 < 0 ? -c2 : c2;
  const uint32_t b = __float_as_uint(v1);
  const int ex = (int)((b >> 23) & 0xffu);
  float r = (ex == 255) ? v1 : (ex > d ? __uint_as_float(b - ((uint32_t)d << 23)) : 0.f);
  r = c2 < 0 ? -r : r;
  return c2 == 0 ? 0.f : r;
}

// Programmatic dependent launch (sm_90+): wait for the upstream grid before touching
// anything it may produce or consume (x, y, workspace); let dependents start early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// L2 cache policies: streamed weights are read exactly once per call -> evict_first, so
// they do not push x, the split-K partials or the next layer's activations out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streaming 16-byte weight load: read-only path, no L1 allocation, L2 evict-first.
__device__ __forceinline__ uint4 ldg_stream(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ldg_s8_stream(const int8_t* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s8 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// 16-byte load of data other CTAs / the next call will re-read (activations): L2 evict-last.
__device__ __forceinline__ uint4 ldg_keep(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// One unit (slice s, row group rg) of the tiled layout: Q plane tiles of 512 B (lane reads
// its 16 B) and Q x 32 chunk exponents (lane reads its byte).
template <int Q>
__device__ __forceinline__ void load_unit(const uint4* __restrict__ planes, const int8_t* __restrict__ exps,
                                          long long u, int lane, uint64_t pol, uint4 (&w)[Q], int (&e)[Q]) {
#pragma unroll
  for (int i = 0; i < Q; ++i) w[i] = ldg_stream(planes + (u * Q + i) * 32 + lane, pol);
#pragma unroll
  for (int i = 0; i < Q; ++i) e[i] = ldg_s8_stream(exps + (u * Q + i) * 32 + lane, pol);
}

// NEXT-f3 fused all-gather epilogue (P == 0: off).  y_peers: device array of 2P device
// pointers (y_peers[b*P + r] = rank r's gathered buffer b, [P*N], mapped here); flag_peers:
// device array of P pointers (rank r's flag array uint32[P]); epoch: this rank's device call
// counter for the layer (call c = *epoch + 1 writes buffer c & 1 and publishes c).
struct GatherArgs {
  __half* const* y_peers = nullptr;
  uint32_t* const* flag_peers = nullptr;
  const uint32_t* epoch = nullptr;
  unsigned* counter = nullptr;
  int P = 0;
  int rank = 0;
};

// NEXT-f3 completion signal (kernels 3 and 8).  After bar.sync, thread 0 of every CTA adds 1
// to the launch counter with a gpu-scope acq_rel atomic (its release half covers the CTA's
// peer stores, cumulative through the barrier).  The last CTA -- whose acquire observed every
// other CTA's release -- re-arms the counter and publishes the call number into flag[rank] of
// every rank with one release pattern (fence.acq_rel.sys, then relaxed system-scope stores).
__device__ __forceinline__ void gather_signal(const GatherArgs& ga) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ga.counter) : "memory");
    if (prev == gridDim.x - 1) {
      // one release pattern for all P flags: fence.acq_rel.sys + strong relaxed stores
      // (st.release.sys per flag compiles to a MEMBAR.ALL.SYS each)
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(ga.counter) : "memory");
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int r = 0; r < ga.P; ++r)
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(ga.flag_peers[r] + ga.rank), "r"(*ga.epoch + 1u)
                     : "memory");
    }
  }
}

struct GemmArgs {
  const __half* x;
  int ldx;
  const uint8_t* planes;
  const int8_t* exps;
  const int8_t* exps2 = nullptr;   // NEXT-f2 second additive-PoT term codes (same layout as exps)
  GatherArgs gather;               // NEXT-f3
  int M, N, K, q, g;
  __half* y;
  int ldy;
  void* workspace;
  size_t workspace_bytes;
  unsigned flags;
  cudaStream_t stream;
};

// The all-SM streaming LUT-GEMV (lut_stream.cu, kernel id 8): one launch covers one or several
// output segments that share x (fused projections), each with its own packed weights and q.
constexpr int kMaxSegments = 4;
// its workspace region: after the split-K counters and the fused-gather launch counter
constexpr size_t kStreamWsOff = kCounterBytes + 256;
// Workspace map: [0, kCounterBytes) per-row-group arrival counters (kernels 1, 2; left zero);
// kCounterBytes: the fused-gather launch counter (left zero); kStreamWsOff: kernel 8's epoch
// word (never written by anything else); kPartOff: the split-K partials of whichever kernel
// runs (kernels 1, 2: fp32; kernel 8: {epoch, fp32} words).  Partials of different calls may
// overlap -- they are rewritten every call -- but nothing may overwrite the counters or the
// epoch word, whose values carry over from call to call.
constexpr size_t kPartOff = kStreamWsOff + 256;
struct StreamSeg {
  const uint8_t* planes;
  const int8_t* exps;
  __half* y;
  int q, N;
};
struct StreamLaunch {
  const __half* x;
  int M, ldx, ldy;   // M <= 8 rows per launch (M = 1: ldx, ldy unused)
  int K;
  int nseg;
  StreamSeg seg[kMaxSegments];
  void* workspace;
  int grid, nst, su, pdl;
  int half;   // 1: the co-resident variant (<= 113 KB shared memory, two CTAs fit one SM)
  const int8_t* exps_bw;   // non-null: NEXT-f1 block-wise exponents [q][8][K/8] (M = 1, one segment)
  int colwise;             // 1: exps_bw holds NEXT-f1 column-wise exponents [q][K] instead
  GatherArgs gather;       // NEXT-f3 (M = 1, one segment, K >= 512): y into every rank's buffer
  int one_slice;           // M = 1: one slice per CTA (grid = S x floor(#SMs / S)), see abi.cu
  const int8_t* exps2;     // NEXT-f2 second additive-PoT term codes (M = 1, one segment; tiled like exps)
};

// The persistent decode program (lut_program.cu, kernel id 9): ordered calls of the fused form.
struct ProgramCallDesc {
  const __half* x;
  int K, nseg, wait;
  StreamSeg seg[kMaxSegments];
};
size_t program_bytes(int ncalls);
size_t program_part_bytes(int S, int RGtot);
size_t program_workspace_bytes(size_t part_max);
uint64_t program_encode(const ProgramCallDesc* calls, int ncalls, void* out);
cudaError_t launch_lut_program(const void* program, int ncalls, uint64_t hash, int qmax, size_t part_max,
                               void* workspace, int sms, cudaStream_t stream);

struct LaunchPlan {
  int grid;
  int threads;
  int smem;
  int kernel;  // 0 generic, 1 tiled M=1 split-K, 2 tiled small batch, 3 tiled M=1 cluster split-K,
              // 4 tiled M=1 split-K with the TMA weight ring, 5 tiled M=2 cluster TMA ring,
              // 6 tiled M=3..4 cluster TMA ring, 7 tiled M>4 as row chunks through 5/6,
              // 8 tiled all-SM streaming LUT-GEMV (lut_stream.cu)
};

// Implemented in the kernel translation units.
cudaError_t launch_pack(const int8_t* signs, const float* alpha, int q, int N, int K, int g,
                        int layout, uint8_t* planes, int8_t* exps, int32_t* counts,
                        cudaStream_t stream);

cudaError_t launch_pack_apot2(const float* alpha, int q, int N, int K, int g, int layout, int8_t* exps2,
                              cudaStream_t stream);
cudaError_t launch_pack_blockwise(const int8_t* signs, const float* alpha_bw, int q, int N, int K, int layout,
                                  uint8_t* planes, int8_t* exps_bw, int32_t* counts, cudaStream_t stream);
cudaError_t launch_pack_colwise(const int8_t* signs, const float* alpha_col, int q, int N, int K,
                                int layout, uint8_t* planes, int8_t* exps_col, int32_t* counts,
                                cudaStream_t stream);

cudaError_t launch_bcq_quantize(const float* w, int N, int K, int q, int g, int T, int pot, int8_t* signs,
                                float* alpha, cudaStream_t stream);

LaunchPlan plan_generic(int M, int N, int K, int q, int g, int sms);
cudaError_t launch_gemm_generic(const GemmArgs& a, const LaunchPlan& p);

LaunchPlan plan_gemv_tiled(int N, int K, int q, int sms);
bool stream_applicable(int N, int K, int q, int sms);
cudaError_t launch_copy(void* dst, const void* src, size_t bytes, bool pdl, bool src_ready, cudaStream_t stream);
bool cluster_is_4slot(int N, int K, int q);
bool m2_applicable(int N, int K, int q, int sms);
LaunchPlan plan_gemm_m2(int N, int K, int q, int sms);
cudaError_t launch_gemm_m2(const GemmArgs& a, const LaunchPlan& p);
bool m4_applicable(int N, int K, int q, int sms);
LaunchPlan plan_gemm_m4(int N, int K, int q, int sms);
cudaError_t launch_gemm_m4(const GemmArgs& a, const LaunchPlan& p);
LaunchPlan plan_gemv_stream(int N, int K, int q, int sms);
size_t workspace_gemv_tiled(int N, int K);
cudaError_t launch_gemv_tiled(const GemmArgs& a, const LaunchPlan& p);

bool cluster_applicable(int N, int K, int q, int sms);
// NEXT-f1: column-wise scales, M = 1, tiled planes, exps_col [q][K]; K <= 4096.
bool colwise_applicable(int N, int K, int q);
cudaError_t launch_gemv_colwise(const GemmArgs& a);
cudaError_t launch_gather_wait(const uint32_t* flags, int P, uint32_t* epoch, cudaStream_t stream);
LaunchPlan plan_gemv_cluster(int N, int K, int q, int sms);
cudaError_t launch_gemv_cluster(const GemmArgs& a, const LaunchPlan& p);

int stream_lut_bytes(int MW);
int stream_smem_bytes(int qmax, int nst, int su, int MW);
int stream_stages(int qmax, int budget, int su, int MW);
size_t stream_workspace_bytes(int M, int S, int RGtot);
bool stream_shape_ok(int K, int sms);
cudaError_t launch_lut_stream(const StreamLaunch& L, cudaStream_t stream);
// kernel 10: fused segments on the cluster TMA ring (M = 1, K <= 4096)
bool fused_cluster_ok(int K, int RGtot);
cudaError_t launch_gemv_cluster_fused(const StreamLaunch& L, cudaStream_t stream);
#ifdef SHIFTADD_DEV_TRACE
cudaError_t dev_set_trace(void* buf);
cudaError_t dev_set_program_trace(void* buf);
cudaError_t dev_set_program_variant(int v);
extern int g_dev_variant;
void dev_set_variant(int v);
#endif

LaunchPlan plan_gemm_tiled_mb(int M, int N, int K, int q, int sms);
size_t workspace_gemm_tiled_mb(int M, int N, int K);
cudaError_t launch_gemm_tiled_mb(const GemmArgs& a, const LaunchPlan& p);

}  // namespace shiftadd
