// abi.cu -- the extern "C" boundary of libshiftadd (include/shiftadd.h, §8(b)).
//
// Synchronous argument validation (nothing is launched on failure), device checks, the
// mixed-bit dispatch of §8 a6 (q -> template instance, host side, no device cost) and the
// layout/batch dispatch between the kernels.  No exceptions cross the boundary.
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>

#include "common.cuh"

namespace shiftadd {
namespace {

thread_local std::string g_last_error;

shiftadd_status fail(shiftadd_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

shiftadd_status cuda_fail(cudaError_t e, const char* what) {
  return fail(SHIFTADD_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

struct DevInfo {
  cudaError_t err;
  int major, minor, sms;
};

// Immutable per-device facts, computed once per device.
shiftadd_status device_info(DevInfo* out) {
  static std::once_flag once[64];
  static DevInfo info[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(SHIFTADD_ERR_CUDA, "device ordinal %d out of range", dev);
  std::call_once(once[dev], [dev] {
    DevInfo d{cudaSuccess, 0, 0, 0};
    d.err = cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
    if (d.err == cudaSuccess) d.err = cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (d.err == cudaSuccess) d.err = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    info[dev] = d;
  });
  *out = info[dev];
  if (out->err != cudaSuccess) return cuda_fail(out->err, "cudaDeviceGetAttribute");
  if (out->major != 10 || out->minor != 0)
    return fail(SHIFTADD_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a only", dev,
                out->major, out->minor);
  return SHIFTADD_OK;
}

shiftadd_status check_shape(int q, int N, int K, int g, int max_q) {
  if (q < 1 || q > max_q) return fail(SHIFTADD_ERR_INVALID, "q=%d outside [1, %d]", q, max_q);
  if (N < 1 || K < 8) return fail(SHIFTADD_ERR_INVALID, "need N >= 1 and K >= 8 (N=%d, K=%d)", N, K);
  if (N > kMaxRows) return fail(SHIFTADD_ERR_INVALID, "N=%d above %d", N, kMaxRows);
  if (K % 8) return fail(SHIFTADD_ERR_INVALID, "K=%d is not a multiple of 8", K);
  if (g < 8 || g % 8 || K % g) return fail(SHIFTADD_ERR_INVALID, "need 8 | g and g | K (g=%d, K=%d)", g, K);
  return SHIFTADD_OK;
}

shiftadd_status check_layout(int layout, int K, int g) {
  if (layout == SHIFTADD_LAYOUT_CANONICAL) return SHIFTADD_OK;
  if (layout != SHIFTADD_LAYOUT_TILED) return fail(SHIFTADD_ERR_INVALID, "unknown layout %d", layout);
  if (K % kTileK) return fail(SHIFTADD_ERR_INVALID, "tiled layout needs K %% 256 == 0 (K=%d)", K);
  if (g % 128) return fail(SHIFTADD_ERR_INVALID, "tiled layout needs g %% 128 == 0 (g=%d)", g);
  return SHIFTADD_OK;
}

// shared-memory budget of the streaming kernel's CTA (one per SM): LUT slab + weight ring
constexpr int kStreamSmemBudget = 200 * 1024;

size_t tiled_rows(int N) { return (size_t)((N + kTileRows - 1) / kTileRows); }

int mw_of(int M) { return M == 1 ? 1 : M == 2 ? 2 : M <= 4 ? 4 : 8; }

// Kernel 8, M = 1: one slice per CTA (one LUT build, one run per segment) beats the
// weight-balanced split on layers with many slices and little work per CTA (measured:
// LLaMA-2-7B down_proj, S = 43 on 129 SMs, 9.3 vs 9.8 us in the dev build), not on large or
// few-slice layers (70B gate/up S = 32: 27.1 vs 26.0; q/k/v-sized S = 16: 13.2 vs 13.1).
bool stream_one_slice(int S, double plane_bytes, int sms) {
  return S >= 24 && S <= sms && plane_bytes <= 16e6;
}

// Streaming kernel (id 8) geometry for a launch of Mc <= 8 rows (or the first chunk of M).
LaunchPlan plan_stream(int M, int q, int K, int sms) {
  const int MW = mw_of(M > 8 ? 8 : M);
  const int S = K / kTileK;
  const int grid = MW == 8 ? S * (sms / S) : sms;   // MW = 8: one slice per CTA
  const int nst = stream_stages(q, kStreamSmemBudget, 16, MW);
  return LaunchPlan{grid, 17 * 32, stream_smem_bytes(q, nst, 16, MW), 8};
}

LaunchPlan make_plan(int layout, int M, int N, int K, int q, int g, int sms, unsigned flags) {
  if (layout == SHIFTADD_LAYOUT_CANONICAL) return plan_generic(M, N, K, q, g, sms);
  const bool force_stream = flags & SHIFTADD_FLAG_SPLITK, force_cluster = flags & SHIFTADD_FLAG_CLUSTER;
  if (M == 1) {
    // K <= 4096: the cluster kernel (K-split reduced over DSMEM, measured faster at these
    // sizes); larger K (and SHIFTADD_FLAG_SPLITK): the all-SM streaming kernel (id 8), whose
    // split-K goes through the workspace.  The register-ring / TMA-ring split-K kernels (ids
    // 1, 4) remain for K > 256 x #SMs.
    if (!force_stream && (K <= 4096 || force_cluster) && cluster_applicable(N, K, q, sms))
      return plan_gemv_cluster(N, K, q, sms);
    if (stream_shape_ok(K, sms)) return plan_stream(1, q, K, sms);
    if (stream_applicable(N, K, q, sms)) return plan_gemv_stream(N, K, q, sms);
    return plan_gemv_tiled(N, K, q, sms);
  }
  // a7 small batch.  M = 2..4 with K <= 4096: the cluster rings (float2 / float4 fp32 entries,
  // DSMEM reduction; measured faster there).  Otherwise the streaming kernel with M-wide fp16
  // LUT entries: one pass over the weights for up to 8 rows (two for 9..16).
  const bool small_m = M <= 4 && K <= 4096 && !force_stream;
  if (small_m && M == 2 && m2_applicable(N, K, q, sms)) return plan_gemm_m2(N, K, q, sms);
  if (small_m && M >= 3 && m4_applicable(N, K, q, sms)) return plan_gemm_m4(N, K, q, sms);
  if (!force_cluster && stream_shape_ok(K, sms)) return plan_stream(M, q, K, sms);
  if (M == 2 && m2_applicable(N, K, q, sms)) return plan_gemm_m2(N, K, q, sms);
  if ((M == 3 || M == 4) && m4_applicable(N, K, q, sms)) return plan_gemm_m4(N, K, q, sms);
  if (M > 4 && m2_applicable(N, K, q, sms) && m4_applicable(N, K, q, sms)) {
    LaunchPlan p = plan_gemm_m4(N, K, q, sms);   // row chunks of 2..4 through kernels 5/6
    p.kernel = 7;
    return p;
  }
  return plan_gemm_tiled_mb(M, N, K, q, sms);
}

size_t workspace_for(int layout, int M, int N, int K) {
  if (layout == SHIFTADD_LAYOUT_CANONICAL) return 0;
  const int S = K / kTileK, RG = (N + kTileRows - 1) / kTileRows;
  const size_t b = stream_workspace_bytes(M > 8 ? 8 : M, S, RG);   // row chunks of 8 reuse it in order
  const size_t a = M == 1 ? workspace_gemv_tiled(N, K) : workspace_gemm_tiled_mb(M, N, K);
  return a > b ? a : b;
}

}  // namespace
}  // namespace shiftadd

using namespace shiftadd;

extern "C" {

int shiftadd_abi_version(void) { return SHIFTADD_ABI_VERSION; }

const char* shiftadd_status_string(int status) {
  switch (status) {
    case SHIFTADD_OK: return "ok";
    case SHIFTADD_ERR_INVALID: return "invalid argument";
    case SHIFTADD_ERR_UNSUPPORTED: return "unsupported";
    case SHIFTADD_ERR_CUDA: return "cuda error";
    default: return "unknown status";
  }
}

const char* shiftadd_last_error(void) { return g_last_error.c_str(); }

size_t shiftadd_packed_bytes(int layout, int q, int N, int K, int g, size_t* exps_bytes) {
  if (exps_bytes) *exps_bytes = 0;
  if (check_shape(q, N, K, g, 8) != SHIFTADD_OK || check_layout(layout, K, g) != SHIFTADD_OK) return 0;
  if (layout == SHIFTADD_LAYOUT_CANONICAL) {
    if (exps_bytes) *exps_bytes = (size_t)q * N * (K / g);
    return (size_t)q * N * (K / 8);
  }
  const size_t tiles = (size_t)(K / kTileK) * tiled_rows(N) * q;
  if (exps_bytes) *exps_bytes = tiles * kTileExps;
  return tiles * kTileBytes;
}

shiftadd_status shiftadd_pack(const int8_t* signs, const float* alpha, int q, int N, int K, int g,
                              int layout, uint8_t* planes, int8_t* exps, int32_t* counts, void* stream) {
  if (!signs || !alpha || !planes || !exps) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, g, 8);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, g)) != SHIFTADD_OK) return st;
  if (!aligned(signs, 8) || !aligned(alpha, 4) || !aligned(planes, 16) || (counts && !aligned(counts, 4)))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (signs 8 B, alpha 4 B, planes 16 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  cudaError_t e = launch_pack(signs, alpha, q, N, K, g, layout, planes, exps, counts,
                              reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_pack_colwise(const int8_t* signs, const float* alpha_col, int q, int N, int K,
                                      int layout, uint8_t* planes, int8_t* exps_col, int32_t* counts,
                                      void* stream) {
  if (!signs || !alpha_col || !planes || !exps_col) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, 8, 8);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, 128)) != SHIFTADD_OK) return st;
  if (!aligned(signs, 8) || !aligned(alpha_col, 4) || !aligned(planes, 16) || (counts && !aligned(counts, 4)))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (signs 8 B, alpha 4 B, planes 16 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  cudaError_t e = launch_pack_colwise(signs, alpha_col, q, N, K, layout, planes, exps_col, counts,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack_colwise launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_lut_gemv_colwise(const uint16_t* x, const uint8_t* planes, const int8_t* exps_col,
                                          int layout, int N, int K, int q, uint16_t* y, unsigned flags,
                                          void* stream) {
  if (!x || !planes || !exps_col || !y) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, 8, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, 128)) != SHIFTADD_OK) return st;
  if (layout != SHIFTADD_LAYOUT_TILED)
    return fail(SHIFTADD_ERR_UNSUPPORTED, "column-wise GEMV needs the tiled layout");
  if (flags & ~SHIFTADD_FLAG_PDL) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(x, 16) || !aligned(planes, 16) || !aligned(exps_col, 8) || !aligned(y, 2))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (x, planes 16 B; exps_col 8 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  if (!colwise_applicable(N, K, q))
    return fail(SHIFTADD_ERR_UNSUPPORTED, "column-wise GEMV: K=%d N=%d outside K <= 4096 / band limit", K, N);
  GemmArgs a;
  a.x = reinterpret_cast<const __half*>(x);
  a.ldx = K;
  a.planes = planes;
  a.exps = exps_col;
  a.M = 1;
  a.N = N;
  a.K = K;
  a.q = q;
  a.g = K;
  a.y = reinterpret_cast<__half*>(y);
  a.ldy = N;
  a.workspace = nullptr;
  a.workspace_bytes = 0;
  a.flags = flags;
  a.stream = reinterpret_cast<cudaStream_t>(stream);
  const cudaError_t e = launch_gemv_colwise(a);
  if (e == cudaErrorNotSupported) return fail(SHIFTADD_ERR_UNSUPPORTED, "no cluster configuration for this shape");
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_colwise launch");
  return SHIFTADD_OK;
}

size_t shiftadd_workspace_bytes_colwise(int N, int K) {
  if (N < 1 || N > kMaxRows || K < kTileK || K % kTileK) return 0;
  return stream_workspace_bytes(2, K / kTileK, (N + kTileRows - 1) / kTileRows);   // covers M = 1 and pairs
}

shiftadd_status shiftadd_lut_gemm_colwise(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps_col,
                                          int layout, int M, int N, int K, int q, uint16_t* y, int ldy,
                                          void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  if (M == 1)
    return shiftadd_lut_gemv_colwise_ws(x, planes, exps_col, layout, N, K, q, y, workspace, workspace_bytes, flags,
                                        stream);
  if (!x || !planes || !exps_col || !y) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  if (M < 1 || M > 16) return fail(SHIFTADD_ERR_UNSUPPORTED, "M=%d outside [1, 16]", M);
  shiftadd_status st = check_shape(q, N, K, 8, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, 128)) != SHIFTADD_OK) return st;
  if (layout != SHIFTADD_LAYOUT_TILED)
    return fail(SHIFTADD_ERR_UNSUPPORTED, "column-wise GEMM needs the tiled layout");
  if (flags & ~(SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK)) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (ldx < K || ldy < N) return fail(SHIFTADD_ERR_INVALID, "ldx < K or ldy < N");
  if (!aligned(x, 16) || (ldx % 8) || !aligned(planes, 16) || !aligned(exps_col, 8) || !aligned(y, 2))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (x rows, planes 16 B; exps_col 8 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  if (!stream_shape_ok(K, di.sms)) return fail(SHIFTADD_ERR_UNSUPPORTED, "column-wise GEMM: K=%d above 256 x #SMs", K);
  const size_t need = shiftadd_workspace_bytes_colwise(N, K);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned(workspace, 16)))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 16-B aligned (got %zu)", need, workspace_bytes);
  // pairs of rows (fp16-pair LUT entries: one weight pass per 2 rows), stream-ordered
  cudaError_t e = cudaSuccess;
  for (int m0 = 0; m0 < M && e == cudaSuccess; m0 += 2) {
    const int mc = M - m0 < 2 ? M - m0 : 2;
    if (mc == 1) {
      const shiftadd_status s1 = shiftadd_lut_gemv_colwise_ws(x + (size_t)m0 * ldx, planes, exps_col, layout, N, K, q,
                                                              y + (size_t)m0 * ldy, workspace, workspace_bytes,
                                                              flags | SHIFTADD_FLAG_SPLITK, stream);
      if (s1 != SHIFTADD_OK) return s1;
      continue;
    }
    StreamLaunch L = {};
    L.x = reinterpret_cast<const __half*>(x) + (size_t)m0 * ldx;
    L.M = 2;
    L.ldx = ldx;
    L.ldy = ldy;
    L.K = K;
    L.nseg = 1;
    L.seg[0] = StreamSeg{planes, exps_col, reinterpret_cast<__half*>(y) + (size_t)m0 * ldy, q, N};
    L.exps_bw = exps_col;
    L.colwise = 1;
    L.workspace = workspace;
    L.grid = di.sms;
    L.su = 16;
    const int lut = q <= 2 ? 64 * 1024 : 128 * 1024;
    const int slot = L.su * q * (kTileBytes + kTileExps);
    L.nst = (kStreamSmemBudget - lut - 640) / slot;
    L.nst = L.nst > 16 ? 16 : L.nst;
    L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
    e = launch_lut_stream(L, reinterpret_cast<cudaStream_t>(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemm_colwise launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_lut_gemv_colwise_ws(const uint16_t* x, const uint8_t* planes, const int8_t* exps_col,
                                             int layout, int N, int K, int q, uint16_t* y, void* workspace,
                                             size_t workspace_bytes, unsigned flags, void* stream) {
  if (!x || !planes || !exps_col || !y) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, 8, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, 128)) != SHIFTADD_OK) return st;
  if (layout != SHIFTADD_LAYOUT_TILED)
    return fail(SHIFTADD_ERR_UNSUPPORTED, "column-wise GEMV needs the tiled layout");
  if (flags & ~(SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK)) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(x, 16) || !aligned(planes, 16) || !aligned(exps_col, 8) || !aligned(y, 2))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (x, planes 16 B; exps_col 8 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  // K <= 4096: the cluster kernel (no workspace) unless SHIFTADD_FLAG_SPLITK; else the all-SM
  // streaming kernel with per-plane column-scaled LUTs
  if (!(flags & SHIFTADD_FLAG_SPLITK) && colwise_applicable(N, K, q))
    return shiftadd_lut_gemv_colwise(x, planes, exps_col, layout, N, K, q, y, flags & SHIFTADD_FLAG_PDL, stream);
  if (!stream_shape_ok(K, di.sms)) return fail(SHIFTADD_ERR_UNSUPPORTED, "column-wise GEMV: K=%d above 256 x #SMs", K);
  const size_t need = shiftadd_workspace_bytes_colwise(N, K);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned(workspace, 16)))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 16-B aligned (got %zu)", need, workspace_bytes);
  StreamLaunch L = {};
  L.x = reinterpret_cast<const __half*>(x);
  L.M = 1;
  L.ldx = K;
  L.K = K;
  L.nseg = 1;
  L.seg[0] = StreamSeg{planes, exps_col, reinterpret_cast<__half*>(y), q, N};
  L.exps_bw = exps_col;
  L.colwise = 1;
  L.workspace = workspace;
  L.grid = di.sms;
  L.su = 16;
  const int lut = q <= 2 ? 64 * 1024 : 128 * 1024;
  const int slot = L.su * q * (kTileBytes + kTileExps);
  L.nst = (kStreamSmemBudget - lut - 640) / slot;
  L.nst = L.nst > 16 ? 16 : L.nst;
  L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  const cudaError_t e = launch_lut_stream(L, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_colwise_ws launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_pack_blockwise(const int8_t* signs, const float* alpha_bw, int q, int N, int K, int layout,
                                       uint8_t* planes, int8_t* exps_bw, int32_t* counts, void* stream) {
  if (!signs || !alpha_bw || !planes || !exps_bw) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, 8, 8);
  if (st != SHIFTADD_OK) return st;
  if (N % 8) return fail(SHIFTADD_ERR_INVALID, "block-wise scales need 8 | N (N=%d)", N);
  if ((st = check_layout(layout, K, 128)) != SHIFTADD_OK) return st;
  if (!aligned(signs, 8) || !aligned(alpha_bw, 4) || !aligned(planes, 16) || (counts && !aligned(counts, 4)))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (signs 8 B, alpha 4 B, planes 16 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  const cudaError_t e = launch_pack_blockwise(signs, alpha_bw, q, N, K, layout, planes, exps_bw, counts,
                                              reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack_blockwise launch");
  return SHIFTADD_OK;
}

size_t shiftadd_workspace_bytes_blockwise(int N, int K) {
  if (N < 8 || N % 8 || N > kMaxRows || K < kTileK || K % kTileK) return 0;
  return stream_workspace_bytes(1, K / kTileK, (N + kTileRows - 1) / kTileRows);
}

shiftadd_status shiftadd_lut_gemv_blockwise(const uint16_t* x, const uint8_t* planes, const int8_t* exps_bw,
                                            int layout, int N, int K, int q, uint16_t* y, void* workspace,
                                            size_t workspace_bytes, unsigned flags, void* stream) {
  if (!x || !planes || !exps_bw || !y) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, 8, 4);
  if (st != SHIFTADD_OK) return st;
  if (N % 8) return fail(SHIFTADD_ERR_INVALID, "block-wise scales need 8 | N (N=%d)", N);
  if ((st = check_layout(layout, K, 128)) != SHIFTADD_OK) return st;
  if (layout != SHIFTADD_LAYOUT_TILED) return fail(SHIFTADD_ERR_UNSUPPORTED, "block-wise GEMV needs the tiled layout");
  if (flags & ~SHIFTADD_FLAG_PDL) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(x, 16) || !aligned(planes, 16) || !aligned(y, 2))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (x, planes 16 B)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  if (!stream_shape_ok(K, di.sms)) return fail(SHIFTADD_ERR_UNSUPPORTED, "block-wise GEMV: K=%d above 256 x #SMs", K);
  const size_t need = shiftadd_workspace_bytes_blockwise(N, K);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned(workspace, 16)))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 16-B aligned (got %zu)", need, workspace_bytes);
  StreamLaunch L = {};
  L.x = reinterpret_cast<const __half*>(x);
  L.M = 1;
  L.ldx = K;
  L.K = K;
  L.nseg = 1;
  L.seg[0] = StreamSeg{planes, exps_bw, reinterpret_cast<__half*>(y), q, N};
  L.exps_bw = exps_bw;
  L.workspace = workspace;
  L.grid = di.sms;
  if (N % 128 == 0) {   // scaled LUTs: q LUTs of 32 KB (64 KB slab for q <= 2, two slabs else)
    L.su = 16;
    const int lut = q <= 2 ? 64 * 1024 : 128 * 1024;
    const int slot = L.su * q * (kTileBytes + kTileExps);
    L.nst = (kStreamSmemBudget - lut - 640) / slot;
    L.nst = L.nst > 16 ? 16 : L.nst;
  } else {
    L.su = 8;
    L.nst = stream_stages(q, kStreamSmemBudget, L.su, 1);
  }
  L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  const cudaError_t e = launch_lut_stream(L, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_blockwise launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_pack_apot2(const int8_t* signs, const float* alpha, int q, int N, int K, int g,
                                    int layout, uint8_t* planes, int8_t* exps, int8_t* exps2, int32_t* counts,
                                    void* stream) {
  if (!exps2) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  const shiftadd_status st = shiftadd_pack(signs, alpha, q, N, K, g, layout, planes, exps, counts, stream);
  if (st != SHIFTADD_OK) return st;
  const cudaError_t e = launch_pack_apot2(alpha, q, N, K, g, layout, exps2, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack_apot2 launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_lut_gemm_apot2(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                        const int8_t* exps2, int layout, int M, int N, int K, int q, int g,
                                        uint16_t* y, int ldy, unsigned flags, void* stream) {
  return shiftadd_lut_gemm_apot2_ws(x, ldx, planes, exps, exps2, layout, M, N, K, q, g, y, ldy, nullptr, 0, flags,
                                    stream);
}

size_t shiftadd_workspace_bytes_apot2(int N, int K) {
  if (N < 1 || N > kMaxRows || K < kTileK || K % kTileK) return 0;
  return stream_workspace_bytes(1, K / kTileK, (N + kTileRows - 1) / kTileRows);
}

shiftadd_status shiftadd_lut_gemm_apot2_ws(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                           const int8_t* exps2, int layout, int M, int N, int K, int q, int g,
                                           uint16_t* y, int ldy, void* workspace, size_t workspace_bytes,
                                           unsigned flags, void* stream) {
  if (!x || !planes || !exps || !exps2 || !y) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, g, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, g)) != SHIFTADD_OK) return st;
  if (M < 1) return fail(SHIFTADD_ERR_INVALID, "M=%d < 1", M);
  if (M > 16) return fail(SHIFTADD_ERR_UNSUPPORTED, "M=%d > 16", M);
  if (ldx < K || ldy < N) return fail(SHIFTADD_ERR_INVALID, "ldx=%d < K=%d or ldy=%d < N=%d", ldx, K, ldy, N);
  if (flags & ~(SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK)) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(x, 16) || (M > 1 && (ldx % 8)) || !aligned(planes, 16) || !aligned(y, 2))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (x rows and planes need 16 B)");
  if (layout == SHIFTADD_LAYOUT_TILED && M != 1)
    return fail(SHIFTADD_ERR_UNSUPPORTED, "additive-PoT-2 tiled path is batch-1 (use the canonical layout)");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  // the cluster kernel for K <= 4096 (and, without a workspace, wherever it applies)
  const bool cluster = layout == SHIFTADD_LAYOUT_TILED && !(flags & SHIFTADD_FLAG_SPLITK) &&
                       (K <= 4096 || !workspace) && cluster_applicable(N, K, q, di.sms);
  if (layout == SHIFTADD_LAYOUT_TILED && !cluster) {
    // the all-SM streaming kernel (id 8) with the second-term codes as a third ring array
    if (K < 2 * kTileK || !stream_shape_ok(K, di.sms) || !aligned(exps, 16) || !aligned(exps2, 16))
      return fail(SHIFTADD_ERR_UNSUPPORTED, "additive-PoT-2 tiled path: K=%d N=%d q=%d has no kernel", K, N, q);
    const size_t need = shiftadd_workspace_bytes_apot2(N, K);
    if (!workspace || workspace_bytes < need || !aligned(workspace, 16))
      return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 16-B aligned (got %zu)", need, workspace_bytes);
    StreamLaunch L = {};
    L.x = reinterpret_cast<const __half*>(x);
    L.M = 1;
    L.ldx = K;
    L.K = K;
    L.nseg = 1;
    L.seg[0] = StreamSeg{planes, exps, reinterpret_cast<__half*>(y), q, N};
    L.exps2 = exps2;
    L.workspace = workspace;
    L.grid = di.sms;
    L.su = 16;
    const int slot = L.su * q * (kTileBytes + 2 * kTileExps);
    L.nst = (kStreamSmemBudget - 64 * 1024 - 640) / slot;
    L.nst = L.nst > 16 ? 16 : L.nst;
    L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
    const cudaError_t e = launch_lut_stream(L, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "lut_gemm_apot2 (streaming) launch");
    return SHIFTADD_OK;
  }
  GemmArgs a;
  a.x = reinterpret_cast<const __half*>(x);
  a.ldx = ldx;
  a.planes = planes;
  a.exps = exps;
  a.exps2 = exps2;
  a.M = M;
  a.N = N;
  a.K = K;
  a.q = q;
  a.g = g;
  a.y = reinterpret_cast<__half*>(y);
  a.ldy = ldy;
  a.workspace = nullptr;
  a.workspace_bytes = 0;
  a.flags = flags & SHIFTADD_FLAG_PDL;
  a.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (layout == SHIFTADD_LAYOUT_CANONICAL) e = launch_gemm_generic(a, plan_generic(M, N, K, q, g, di.sms));
  else e = launch_gemv_cluster(a, plan_gemv_cluster(N, K, q, di.sms));
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemm_apot2 launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_bcq_quantize(const float* w, int N, int K, int q, int g, int T, unsigned flags,
                                      int8_t* signs, float* alpha, void* stream) {
  if (!w || !signs || !alpha) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  if (q < 1 || q > 4) return fail(SHIFTADD_ERR_INVALID, "q=%d outside [1, 4]", q);
  if (N < 1 || K < 1 || g < 1 || K % g) return fail(SHIFTADD_ERR_INVALID, "need N, K, g >= 1 and g | K");
  if (T < 0 || T > 1000) return fail(SHIFTADD_ERR_INVALID, "T=%d outside [0, 1000]", T);
  if ((long long)N * (K / g) >= 0x7fffffffLL) return fail(SHIFTADD_ERR_INVALID, "too many scale groups");
  if (flags & ~SHIFTADD_BCQ_POT) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(w, 4) || !aligned(alpha, 4)) return fail(SHIFTADD_ERR_INVALID, "misaligned pointer");
  DevInfo di;
  shiftadd_status st;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  const cudaError_t e = launch_bcq_quantize(w, N, K, q, g, T, (flags & SHIFTADD_BCQ_POT) ? 1 : 0, signs, alpha,
                                            reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "bcq_quantize launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_lut_gemm_gather(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                         int layout, int M, int N, int K, int q, int g, uint16_t* const* y_peers,
                                         uint32_t* const* flag_peers, int P, int rank, uint32_t* epoch,
                                         void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  if (M < 1 || M > 8) return fail(SHIFTADD_ERR_UNSUPPORTED, "fused gather: M=%d outside [1, 8]", M);
  if (M > 1 && (ldx < K || ldx % 8)) return fail(SHIFTADD_ERR_INVALID, "ldx must be >= K and a multiple of 8");
  if (!x || !planes || !exps || !y_peers || !flag_peers || !epoch || !workspace)
    return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, g, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, g)) != SHIFTADD_OK) return st;
  if (P < 2 || P > 8 || rank < 0 || rank >= P) return fail(SHIFTADD_ERR_INVALID, "need 2 <= P <= 8, 0 <= rank < P");
  if (flags & ~SHIFTADD_FLAG_PDL) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (layout != SHIFTADD_LAYOUT_TILED) return fail(SHIFTADD_ERR_UNSUPPORTED, "fused gather needs the tiled layout");
  if (workspace_bytes < kCounterBytes + 16 || !aligned(workspace, 16))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs >= %zu bytes, 16-B aligned", kCounterBytes + 16);
  if (!aligned(x, 16) || !aligned(planes, 16)) return fail(SHIFTADD_ERR_INVALID, "misaligned x / planes");
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  if (!cluster_applicable(N, K, q, di.sms) || K > 4096 || M > 1) {
    // K > 4096 (LLaMA-2-70B down_proj, OPT-66B fc2 shards): the all-SM streaming kernel (8),
    // its owner CTAs storing into every rank's buffer
    if (K < 2 * kTileK || !stream_shape_ok(K, di.sms) || !aligned(exps, 16))
      return fail(SHIFTADD_ERR_UNSUPPORTED, "fused gather: K=%d N=%d q=%d has no kernel", K, N, q);
    const size_t need = stream_workspace_bytes(1, K / kTileK, (N + kTileRows - 1) / kTileRows);
    if (workspace_bytes < need)
      return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes (got %zu)", need, workspace_bytes);
    const size_t need_m = stream_workspace_bytes(M, K / kTileK, (N + kTileRows - 1) / kTileRows);
    if (workspace_bytes < need_m)
      return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes (got %zu)", need_m, workspace_bytes);
    StreamLaunch L = {};
    L.x = reinterpret_cast<const __half*>(x);
    L.M = M;
    L.ldx = M > 1 ? ldx : K;
    L.ldy = N;
    L.K = K;
    L.nseg = 1;
    L.seg[0] = StreamSeg{planes, exps, nullptr, q, N};
    L.workspace = workspace;
    const LaunchPlan pc = plan_stream(M, q, K, di.sms);
    L.grid = pc.grid;
    L.su = 16;
    L.nst = stream_stages(q, kStreamSmemBudget, L.su, mw_of(M));
    L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
    L.gather.y_peers = reinterpret_cast<__half* const*>(y_peers);
    L.gather.flag_peers = flag_peers;
    L.gather.counter = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + kCounterBytes);
    L.gather.P = P;
    L.gather.rank = rank;
    L.gather.epoch = epoch;
    const cudaError_t e = launch_lut_stream(L, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_gather (streaming) launch");
    return SHIFTADD_OK;
  }
  GemmArgs a;
  a.x = reinterpret_cast<const __half*>(x);
  a.ldx = K;
  a.planes = planes;
  a.exps = exps;
  a.M = 1;
  a.N = N;
  a.K = K;
  a.q = q;
  a.g = g;
  a.y = nullptr;
  a.ldy = N;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.flags = flags;
  a.stream = reinterpret_cast<cudaStream_t>(stream);
  a.gather.y_peers = reinterpret_cast<__half* const*>(y_peers);
  a.gather.flag_peers = flag_peers;
  a.gather.counter = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + kCounterBytes);
  a.gather.P = P;
  a.gather.rank = rank;
  a.gather.epoch = epoch;
  const cudaError_t e = launch_gemv_cluster(a, plan_gemv_cluster(N, K, q, di.sms));
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_gather launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_lut_gemv_gather(const uint16_t* x, const uint8_t* planes, const int8_t* exps, int layout,
                                         int N, int K, int q, int g, uint16_t* const* y_peers,
                                         uint32_t* const* flag_peers, int P, int rank, uint32_t* epoch,
                                         void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  return shiftadd_lut_gemm_gather(x, K, planes, exps, layout, 1, N, K, q, g, y_peers, flag_peers, P, rank, epoch,
                                  workspace, workspace_bytes, flags, stream);
}

shiftadd_status shiftadd_gather_wait(const uint32_t* flags_local, int P, uint32_t* epoch, void* stream) {
  if (!flags_local || !epoch) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  if (P < 1 || P > 32) return fail(SHIFTADD_ERR_INVALID, "P=%d outside [1, 32]", P);
  DevInfo di;
  shiftadd_status st;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  const cudaError_t e = launch_gather_wait(flags_local, P, epoch, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "gather_wait launch");
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_copy(void* dst, const void* src, size_t bytes, unsigned flags, void* stream) {
  if (!dst || !src) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  if (bytes % 16 || !aligned(dst, 16) || !aligned(src, 16))
    return fail(SHIFTADD_ERR_INVALID, "copy needs 16-B aligned pointers and a multiple of 16 bytes (%zu)", bytes);
  if (flags & ~(SHIFTADD_FLAG_PDL | SHIFTADD_COPY_SRC_READY)) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  DevInfo di;
  shiftadd_status st;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  const cudaError_t e = launch_copy(dst, src, bytes, flags & SHIFTADD_FLAG_PDL, flags & SHIFTADD_COPY_SRC_READY,
                                    reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "copy launch");
  return SHIFTADD_OK;
}

#ifdef SHIFTADD_DEV_TRACE
// development builds only: per-CTA phase timestamps of the streaming kernel into `buf`
// (16 u64 per CTA), NULL to stop
int shiftadd_dev_set_trace(void* buf) { return (int)dev_set_trace(buf); }
int shiftadd_dev_set_program_trace(void* buf) { return (int)dev_set_program_trace(buf); }
int shiftadd_dev_set_program_variant(int v) { return (int)dev_set_program_variant(v); }
void shiftadd_dev_set_variant(int v) { dev_set_variant(v); }
#endif

size_t shiftadd_workspace_bytes(int layout, int M, int N, int K, int q, int g) {
  if (check_shape(q, N, K, g, 4) != SHIFTADD_OK || check_layout(layout, K, g) != SHIFTADD_OK) return 0;
  if (M < 1 || M > 16) return 0;
  return workspace_for(layout, M, N, K);
}

shiftadd_status shiftadd_gemm_plan(int layout, int M, int N, int K, int q, int g, int out[4]) {
  if (!out) return fail(SHIFTADD_ERR_INVALID, "null out");
  shiftadd_status st = check_shape(q, N, K, g, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, g)) != SHIFTADD_OK) return st;
  if (M < 1 || M > 16) return fail(SHIFTADD_ERR_UNSUPPORTED, "M=%d outside [1, 16]", M);
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  const LaunchPlan p = make_plan(layout, M, N, K, q, g, di.sms, 0u);
  out[0] = p.grid;
  out[1] = p.threads;
  out[2] = p.smem;
  out[3] = p.kernel;
  return SHIFTADD_OK;
}

shiftadd_status shiftadd_lut_gemm(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                  int layout, int M, int N, int K, int q, int g, uint16_t* y, int ldy,
                                  void* workspace, size_t workspace_bytes, unsigned flags, void* stream) {
  if (!x || !planes || !exps || !y) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  shiftadd_status st = check_shape(q, N, K, g, 4);
  if (st != SHIFTADD_OK) return st;
  if ((st = check_layout(layout, K, g)) != SHIFTADD_OK) return st;
  if (M < 1) return fail(SHIFTADD_ERR_INVALID, "M=%d < 1", M);
  if (M > 16) return fail(SHIFTADD_ERR_UNSUPPORTED, "M=%d > 16 (small-batch kernels cover M <= 16)", M);
  if (ldx < K || ldy < N) return fail(SHIFTADD_ERR_INVALID, "ldx=%d < K=%d or ldy=%d < N=%d", ldx, K, ldy, N);
  if (flags & ~(SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK | SHIFTADD_FLAG_CLUSTER))
    return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(x, 16) || (M > 1 && (ldx % 8)) || !aligned(planes, 16) || !aligned(y, 2))
    return fail(SHIFTADD_ERR_INVALID, "misaligned pointer (x rows and planes need 16 B)");
  const size_t need = workspace_for(layout, M, N, K);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned(workspace, 16)))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 16-B aligned (got %zu)", need, workspace_bytes);
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;

  GemmArgs a;
  a.x = reinterpret_cast<const __half*>(x);
  a.ldx = ldx;
  a.planes = planes;
  a.exps = exps;
  a.M = M;
  a.N = N;
  a.K = K;
  a.q = q;
  a.g = g;
  a.y = reinterpret_cast<__half*>(y);
  a.ldy = ldy;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.flags = flags;
  a.stream = reinterpret_cast<cudaStream_t>(stream);
  LaunchPlan p = make_plan(layout, M, N, K, q, g, di.sms, flags);
  // the TMA ring copies exponent tiles with 16-B bulk copies
  if ((p.kernel == 4 || p.kernel == 8) && !aligned(exps, 16))
    p = M == 1 ? plan_gemv_tiled(N, K, q, di.sms) : plan_gemm_tiled_mb(M, N, K, q, di.sms);
  if ((p.kernel >= 5 && p.kernel <= 7) && !aligned(exps, 16)) p = plan_gemm_tiled_mb(M, N, K, q, di.sms);
  cudaError_t e;
  if (layout == SHIFTADD_LAYOUT_CANONICAL) e = launch_gemm_generic(a, p);
  else if (p.kernel == 8) {
    // row chunks of <= 8 (one launch for M <= 8), stream-ordered on the same workspace
    e = cudaSuccess;
    for (int m0 = 0; m0 < M && e == cudaSuccess; m0 += 8) {
      const int mc = M - m0 < 8 ? M - m0 : 8;
      StreamLaunch L = {};
      L.x = a.x + (size_t)m0 * ldx;
      L.M = mc;
      L.ldx = ldx;
      L.ldy = ldy;
      L.K = K;
      L.nseg = 1;
      L.seg[0] = StreamSeg{planes, exps, a.y + (size_t)m0 * ldy, q, N};
      L.workspace = workspace;
      const LaunchPlan pc = plan_stream(mc, q, K, di.sms);
      L.grid = pc.grid;
      if (mc == 1 && stream_one_slice(K / kTileK, (double)q * N * K / 8, di.sms)) {
        L.one_slice = 1;
        L.grid = (K / kTileK) * (di.sms / (K / kTileK));
      }
      L.su = 16;
      L.nst = stream_stages(q, kStreamSmemBudget, L.su, mw_of(mc));
      L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
#ifdef SHIFTADD_DEV_TRACE
      if ((g_dev_variant & 1) && mc == 1) {
        L.half = 1;
        L.su = 8;
        L.nst = stream_stages(q, 112 * 1024, L.su, 1);
      }
#endif
      e = launch_lut_stream(L, a.stream);
    }
  }
  else if (p.kernel == 3) e = launch_gemv_cluster(a, p);
  else if (p.kernel == 5) e = launch_gemm_m2(a, p);
  else if (p.kernel == 6) e = launch_gemm_m4(a, p);
  else if (p.kernel == 7) {
    // M > 4: row chunks of 4 (the last two 3 + 2 when M % 4 == 1), each one pass over the
    // weights with 2- or 4-wide LUT entries (measured faster than one 16-row pass re-walking
    // the weights per 4-row chunk on the split-K kernel)
    e = cudaSuccess;
    for (int m0 = 0; m0 < M && e == cudaSuccess;) {
      const int left = M - m0;
      const int mc = left >= 6 || left == 4 ? 4 : (left == 5 ? 3 : left);
      GemmArgs c = a;
      c.x = a.x + (size_t)m0 * ldx;
      c.y = a.y + (size_t)m0 * ldy;
      c.M = mc;
      e = mc == 2 ? launch_gemm_m2(c, plan_gemm_m2(N, K, q, di.sms)) : launch_gemm_m4(c, plan_gemm_m4(N, K, q, di.sms));
      m0 += mc;
    }
  }
  else if (M == 1) e = launch_gemv_tiled(a, p);
  else e = launch_gemm_tiled_mb(a, p);
  if (e == cudaErrorNotSupported) return fail(SHIFTADD_ERR_UNSUPPORTED, "no kernel for this configuration");
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemm launch");
  return SHIFTADD_OK;
}

size_t shiftadd_workspace_bytes_fused(int layout, int M, int K, int g, int nseg, const shiftadd_segment* segs) {
  if (layout != SHIFTADD_LAYOUT_TILED || !segs || nseg < 1 || nseg > kMaxSegments || M < 1 || M > 16) return 0;
  if (K < kTileK || K % kTileK || g < 128 || g % 128 || K % g) return 0;
  int rg = 0;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].N < 1 || segs[i].N > kMaxRows) return 0;
    rg += (segs[i].N + kTileRows - 1) / kTileRows;
  }
  return stream_workspace_bytes(M, K / kTileK, rg);
}

shiftadd_status shiftadd_lut_gemv_fused(const uint16_t* x, int K, int g, int layout, int nseg,
                                        const shiftadd_segment* segs, void* workspace, size_t workspace_bytes,
                                        unsigned flags, void* stream) {
  if (!x || !segs) return fail(SHIFTADD_ERR_INVALID, "null pointer argument");
  if (layout != SHIFTADD_LAYOUT_TILED) return fail(SHIFTADD_ERR_UNSUPPORTED, "fused segments need the tiled layout");
  if (nseg < 1 || nseg > kMaxSegments) return fail(SHIFTADD_ERR_INVALID, "nseg=%d outside [1, %d]", nseg, kMaxSegments);
  if (flags & ~(SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK)) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!aligned(x, 16)) return fail(SHIFTADD_ERR_INVALID, "x must be 16-B aligned");
  shiftadd_status st;
  int rg = 0;
  for (int i = 0; i < nseg; ++i) {
    const shiftadd_segment& sg = segs[i];
    if (!sg.planes || !sg.exps || !sg.y) return fail(SHIFTADD_ERR_INVALID, "segment %d: null pointer", i);
    if ((st = check_shape(sg.q, sg.N, K, g, 4)) != SHIFTADD_OK) return st;
    if (!aligned(sg.planes, 16) || !aligned(sg.exps, 16) || !aligned(sg.y, 2))
      return fail(SHIFTADD_ERR_INVALID, "segment %d: planes / exps must be 16-B aligned", i);
    rg += (sg.N + kTileRows - 1) / kTileRows;
  }
  if ((st = check_layout(layout, K, g)) != SHIFTADD_OK) return st;
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  if (!stream_shape_ok(K, di.sms))
    return fail(SHIFTADD_ERR_UNSUPPORTED, "fused segments: K=%d above 256 x %d SMs", K, di.sms);
  const size_t need = stream_workspace_bytes(1, K / kTileK, rg);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned(workspace, 16)))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 16-B aligned (got %zu)", need, workspace_bytes);
  StreamLaunch L = {};
  L.x = reinterpret_cast<const __half*>(x);
  L.M = 1;
  L.ldx = K;
  L.K = K;
  L.nseg = nseg;
  int qmax = 1;
  for (int i = 0; i < nseg; ++i) {
    L.seg[i] = StreamSeg{segs[i].planes, segs[i].exps, reinterpret_cast<__half*>(segs[i].y), segs[i].q, segs[i].N};
    qmax = segs[i].q > qmax ? segs[i].q : qmax;
  }
  L.workspace = workspace;
  L.grid = di.sms;
  L.su = 16;
  L.nst = stream_stages(qmax, kStreamSmemBudget, L.su, 1);
  L.pdl = (flags & SHIFTADD_FLAG_PDL) ? 1 : 0;
  {
    double pb = 0;
    for (int i = 0; i < nseg; ++i) pb += (double)segs[i].q * segs[i].N * K / 8;
    if (stream_one_slice(K / kTileK, pb, di.sms)) {
      L.one_slice = 1;
      L.grid = (K / kTileK) * (di.sms / (K / kTileK));
    }
  }
  // K <= 4096: the cluster TMA ring (kernel 10, DSMEM reduction, no workspace) unless
  // SHIFTADD_FLAG_SPLITK; otherwise (or if no cluster shape fits) the all-SM streaming kernel
  // (measured on B200: q/k/v 4096 x 3 at 2/3/2 bits 8.2 vs 9.1 us; gate/up 11008 x 2 at 2/3
  // bits 12.0 vs 11.5 us -- the 120 SMs clusters of 8 pack lose to all 148 above ~24 MB)
  double plane_bytes = 0;
  for (int i = 0; i < nseg; ++i) plane_bytes += (double)segs[i].q * segs[i].N * K / 8;
  if (!(flags & SHIFTADD_FLAG_SPLITK) && K <= 4096 && plane_bytes <= 24e6 && fused_cluster_ok(K, rg)) {
    const cudaError_t ec = launch_gemv_cluster_fused(L, reinterpret_cast<cudaStream_t>(stream));
    if (ec != cudaSuccess) return cuda_fail(ec, "lut_gemv_fused (cluster) launch");
    return SHIFTADD_OK;
  }
#ifdef SHIFTADD_DEV_TRACE
  if (g_dev_variant & 1) {
    L.half = 1;
    L.su = 8;
    L.nst = stream_stages(qmax, 112 * 1024, L.su, 1);
  }
#endif
  const cudaError_t e = launch_lut_stream(L, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_fused launch");
  return SHIFTADD_OK;
}

// ------------------------------------------------------------------ decode program (kernel 9)
size_t shiftadd_program_bytes(int ncalls) { return ncalls < 1 ? 0 : program_bytes(ncalls); }

namespace {
shiftadd_status check_program(const shiftadd_call* calls, int ncalls, std::vector<ProgramCallDesc>* out,
                              int* qmax, size_t* part_max) {
  if (!calls || ncalls < 1) return fail(SHIFTADD_ERR_INVALID, "need ncalls >= 1 and a call array");
  out->resize(ncalls);
  *qmax = 1;
  *part_max = 0;
  shiftadd_status st;
  for (int j = 0; j < ncalls; ++j) {
    const shiftadd_call& c = calls[j];
    if (!c.x) return fail(SHIFTADD_ERR_INVALID, "call %d: null x", j);
    if (!aligned(c.x, 16)) return fail(SHIFTADD_ERR_INVALID, "call %d: x must be 16-B aligned", j);
    if (c.nseg < 1 || c.nseg > kMaxSegments)
      return fail(SHIFTADD_ERR_INVALID, "call %d: nseg=%d outside [1, %d]", j, c.nseg, kMaxSegments);
    if (c.flags & ~SHIFTADD_CALL_WAIT) return fail(SHIFTADD_ERR_INVALID, "call %d: unknown flags 0x%x", j, c.flags);
    ProgramCallDesc& d = (*out)[j];
    d.x = reinterpret_cast<const __half*>(c.x);
    d.K = c.K;
    d.nseg = c.nseg;
    d.wait = (c.flags & SHIFTADD_CALL_WAIT) ? 1 : 0;
    int rg = 0;
    for (int i = 0; i < c.nseg; ++i) {
      const shiftadd_segment& sg = c.seg[i];
      if (!sg.planes || !sg.exps || !sg.y) return fail(SHIFTADD_ERR_INVALID, "call %d segment %d: null pointer", j, i);
      if ((st = check_shape(sg.q, sg.N, c.K, c.g, 4)) != SHIFTADD_OK) return st;
      if (!aligned(sg.planes, 16) || !aligned(sg.exps, 16) || !aligned(sg.y, 2))
        return fail(SHIFTADD_ERR_INVALID, "call %d segment %d: planes / exps must be 16-B aligned", j, i);
      d.seg[i] = StreamSeg{sg.planes, sg.exps, reinterpret_cast<__half*>(sg.y), sg.q, sg.N};
      *qmax = sg.q > *qmax ? sg.q : *qmax;
      rg += (sg.N + kTileRows - 1) / kTileRows;
    }
    if ((st = check_layout(SHIFTADD_LAYOUT_TILED, c.K, c.g)) != SHIFTADD_OK) return st;
    const size_t pb = program_part_bytes(c.K / kTileK, rg);
    *part_max = pb > *part_max ? pb : *part_max;
  }
  return SHIFTADD_OK;
}
}  // namespace

shiftadd_status shiftadd_program_encode(const shiftadd_call* calls, int ncalls, void* out, size_t out_bytes) {
  std::vector<ProgramCallDesc> d;
  int qmax;
  size_t part_max;
  const shiftadd_status st = check_program(calls, ncalls, &d, &qmax, &part_max);
  if (st != SHIFTADD_OK) return st;
  if (!out || out_bytes < program_bytes(ncalls) || !aligned(out, 8))
    return fail(SHIFTADD_ERR_INVALID, "program buffer needs %zu bytes, 8-B aligned", program_bytes(ncalls));
  program_encode(d.data(), ncalls, out);
  return SHIFTADD_OK;
}

size_t shiftadd_workspace_bytes_program(const shiftadd_call* calls, int ncalls) {
  std::vector<ProgramCallDesc> d;
  int qmax;
  size_t part_max;
  if (check_program(calls, ncalls, &d, &qmax, &part_max) != SHIFTADD_OK) return 0;
  return program_workspace_bytes(part_max);
}

shiftadd_status shiftadd_lut_gemv_program(const shiftadd_call* calls, int ncalls, const void* program,
                                          size_t program_bytes_, void* workspace, size_t workspace_bytes,
                                          unsigned flags, void* stream) {
  std::vector<ProgramCallDesc> d;
  int qmax;
  size_t part_max;
  shiftadd_status st = check_program(calls, ncalls, &d, &qmax, &part_max);
  if (st != SHIFTADD_OK) return st;
  if (flags) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  if (!program || program_bytes_ < program_bytes(ncalls) || !aligned(program, 16))
    return fail(SHIFTADD_ERR_INVALID, "program needs %zu device bytes, 16-B aligned", program_bytes(ncalls));
  const size_t need = program_workspace_bytes(part_max);
  if (!workspace || workspace_bytes < need || !aligned(workspace, 256))
    return fail(SHIFTADD_ERR_INVALID, "workspace needs %zu bytes, 256-B aligned (got %zu)", need, workspace_bytes);
  DevInfo di;
  if ((st = device_info(&di)) != SHIFTADD_OK) return st;
  for (int j = 0; j < ncalls; ++j)
    if (!stream_shape_ok(d[j].K, di.sms))
      return fail(SHIFTADD_ERR_UNSUPPORTED, "call %d: K=%d above 256 x %d SMs", j, d[j].K, di.sms);
  thread_local std::vector<unsigned char> enc;
  enc.resize(program_bytes(ncalls));
  const uint64_t hash = program_encode(d.data(), ncalls, enc.data());
  const cudaError_t e = launch_lut_program(program, ncalls, hash, qmax, part_max, workspace, di.sms,
                                           reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "lut_gemv_program launch");
  return SHIFTADD_OK;
}

// ------------------------------------------------------------------ host-side chain of calls
shiftadd_status shiftadd_lut_gemv_chain(const shiftadd_call* calls, int ncalls, void* workspace,
                                        size_t workspace_bytes, unsigned flags, void* stream) {
  if (!calls || ncalls < 1) return fail(SHIFTADD_ERR_INVALID, "need ncalls >= 1 and a call array");
  if (flags & ~SHIFTADD_FLAG_PDL) return fail(SHIFTADD_ERR_INVALID, "unknown flags 0x%x", flags);
  for (int j = 0; j < ncalls; ++j) {
    const shiftadd_call& c = calls[j];
    shiftadd_status st;
    if (c.nseg == 1) {
      const shiftadd_segment& sg = c.seg[0];
      st = shiftadd_lut_gemm(c.x, c.K, sg.planes, sg.exps, SHIFTADD_LAYOUT_TILED, 1, sg.N, c.K, sg.q, c.g, sg.y, sg.N,
                             workspace, workspace_bytes, flags, stream);
    } else {
      st = shiftadd_lut_gemv_fused(c.x, c.K, c.g, SHIFTADD_LAYOUT_TILED, c.nseg, c.seg, workspace, workspace_bytes,
                                   flags, stream);
    }
    if (st != SHIFTADD_OK) {
      const std::string detail = g_last_error;
      return fail(st, "chain call %d: %s", j, detail.c_str());
    }
  }
  return SHIFTADD_OK;
}

size_t shiftadd_workspace_bytes_chain(const shiftadd_call* calls, int ncalls) {
  if (!calls || ncalls < 1) return 0;
  size_t need = 0;
  for (int j = 0; j < ncalls; ++j) {
    const shiftadd_call& c = calls[j];
    size_t b = 0;
    if (c.nseg == 1)
      b = shiftadd_workspace_bytes(SHIFTADD_LAYOUT_TILED, 1, c.seg[0].N, c.K, c.seg[0].q, c.g);
    else
      b = shiftadd_workspace_bytes_fused(SHIFTADD_LAYOUT_TILED, 1, c.K, c.g, c.nseg, c.seg);
    need = b > need ? b : need;
  }
  return need;
}

shiftadd_status shiftadd_lut_gemv(const uint16_t* x, const uint8_t* planes, const int8_t* exps, int layout,
                                  int N, int K, int q, int g, uint16_t* y, void* workspace,
                                  size_t workspace_bytes, unsigned flags, void* stream) {
  return shiftadd_lut_gemm(x, K, planes, exps, layout, 1, N, K, q, g, y, N, workspace, workspace_bytes, flags,
                           stream);
}

}  // extern "C"
