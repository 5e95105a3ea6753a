/*
 * shiftadd.h -- C ABI of the B200 (sm_100a) ShiftAddLLM LUT-GEMV hot path.
 *
 * The operation (arxiv 2406.05981, §4.1):
 *   y = sum_i alpha_i (.) (B_i x)    -- BCQ weights w_q = sum_i alpha_i b_i,
 *   alpha_i = sign * 2^P, P = round(log2|alpha|)  (Eq. 2),
 *   x * 2^P done as an integer add on the float exponent field,
 *   B_i x done by building 256 partial sums per 8 activations and querying them with
 *   8-bit keys formed by 8 grouped binary weights, output FP16 (:186).
 *
 * Conventions (all functions):
 *   - Every pointer argument is a caller-owned CUDA DEVICE pointer unless stated otherwise.
 *     The library never allocates, frees or synchronises; every launch is stream-ordered
 *     on `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - Arguments are validated synchronously before anything is launched; a validation
 *     failure returns SHIFTADD_ERR_INVALID / _UNSUPPORTED and launches nothing.
 *   - Launch failures return SHIFTADD_ERR_CUDA; asynchronous device faults surface at the
 *     caller's next synchronisation.  shiftadd_last_error() returns a thread-local detail.
 *   - No C++ exception crosses the ABI.  No global mutable state beyond per-device
 *     immutable caches (SM count, kernel attributes), so calls are thread-safe per stream.
 *   - fp16 tensors are passed as uint16_t IEEE binary16 bit patterns.
 *
 * Notation: x[M][K] activations (K = reduction dim), N outputs, q bit-planes, scale group
 * g along K.  A key byte holds 8 consecutive k of one output row n of one plane i:
 * bit (k & 7) of byte k >> 3 is 1 <=> the weight sign is +1 (LSB = lowest k).
 */
#ifndef SHIFTADD_H
#define SHIFTADD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHIFTADD_ABI_VERSION 1

typedef enum {
  SHIFTADD_OK = 0,
  SHIFTADD_ERR_INVALID = 2,      /* bad argument (null pointer, shape, alignment, range)   */
  SHIFTADD_ERR_UNSUPPORTED = 6,  /* valid request this build has no kernel for (e.g. M>16) */
  SHIFTADD_ERR_CUDA = 7          /* CUDA runtime error (no device, not sm_100, launch)     */
} shiftadd_status;

/* Exponent encoding of a PoT scale (reading R5 in DESIGN.md). */
#define SHIFTADD_EXP_ZERO ((int8_t)-128) /* alpha == 0: the group contributes nothing */
#define SHIFTADD_EXP_MIN (-100)          /* finite exponents are clamped to [MIN, MAX]  */
#define SHIFTADD_EXP_MAX (100)

/* Weight layouts.  Both hold the same bytes (one a permutation of the other).
 *  CANONICAL: planes u8 [q][N][K/8], exps i8 [q][N][K/g]  (the north_star layout).
 *  TILED    : device-tiled, for the fast kernels.  Tiles of 16 rows x
 *             256 k per plane, stored in (slice s, row-group rg, plane i) order, 512 B each:
 *               byte ((s*RG + rg)*q + i)*512 + r*32 + h*16 + j
 *                 = canonical planes[i][16rg + r][32s + 16h + ((j + r) & 15)]   (0 if n >= N)
 *             and one exponent per 128-k chunk:
 *               exps ((s*RG + rg)*q + i)*32 + r*2 + h
 *                 = canonical exps[i][16rg + r][(256s + 128h) / g]            (EXP_ZERO if n >= N)
 *             with RG = ceil(N/16).  Requires K % 256 == 0 and g % 128 == 0. */
typedef enum { SHIFTADD_LAYOUT_CANONICAL = 0, SHIFTADD_LAYOUT_TILED = 1 } shiftadd_layout;

/* Flags for shiftadd_lut_gemm. */
#define SHIFTADD_FLAG_PDL 1u /* launch with programmatic dependent launch: the kernel's weight
                                prefetch may overlap the previous kernel on the stream; x,
                                y and the workspace are touched only after it completes. */
#define SHIFTADD_FLAG_SPLITK 2u /* tiled layout: always use the grid-wide split-K
                                   decompositions (K-slices per CTA, partials in the
                                   workspace) -- for M = 1 the all-SM streaming kernel (id 8)
                                   where K <= 256 x #SMs; for M >= 2 the small-batch split-K
                                   kernel -- instead of the cluster kernels (K-split reduced
                                   over distributed shared memory).  For testing and
                                   measurement; results agree within rounding order. */

#define SHIFTADD_FLAG_CLUSTER 4u /* tiled layout: use the thread-block-cluster kernels (K-split
                                    reduced over distributed shared memory; ids 3, 5, 6, 7) where
                                    they apply, instead of the all-SM streaming kernel.  For
                                    testing and measurement; results agree within rounding order. */

int shiftadd_abi_version(void);
const char* shiftadd_status_string(int status);
const char* shiftadd_last_error(void);

/* Bytes of the packed planes for a layout (returned) and of its exponents (*exps_bytes if
 * non-NULL).  Returns 0 (and sets last_error) for shapes the layout cannot hold. */
size_t shiftadd_packed_bytes(int layout, int q, int N, int K, int g, size_t* exps_bytes);

/* a1 -- bit-plane packing and PoT exponent encoding.
 *   signs : i8  [q][N][K], each -1 or +1                 (b_i)
 *   alpha : f32 [q][N][K/g]                              (group scales alpha_i)
 *   planes: out, shiftadd_packed_bytes(layout,...) bytes, 16-byte aligned
 *   exps  : out, *exps_bytes bytes
 *   counts: out, optional (may be NULL) i32[2] device scalars, ACCUMULATED into (caller
 *           zeroes them): counts[0] += clamped exponents, counts[1] += invalid inputs
 *           (non-finite alpha or a sign not in {-1,+1}; their exponent is EXP_ZERO).
 * Steps: a group with alpha < 0 has its signs negated and keeps |alpha| (exact, reading R3);
 * e = round(log2|alpha|) (exact integer mantissa rule), EXP_ZERO for alpha = +-0, clamped to
 * [EXP_MIN, EXP_MAX].  Constraints: 1 <= q <= 8, N >= 1, K % 8 == 0, g % 8 == 0, K % g == 0;
 * TILED additionally K % 256 == 0 and g % 128 == 0. */
shiftadd_status shiftadd_pack(const int8_t* signs, const float* alpha, int q, int N, int K,
                              int g, int layout, uint8_t* planes, int8_t* exps,
                              int32_t* counts, void* stream);

/* Workspace bytes a shiftadd_lut_gemm call with these arguments needs (0 if none).  The
 * caller zeroes a fresh workspace once (cudaMemsetAsync).  Layout: 256 KB of split-K
 * per-row-group arrival counters at offset 0, then fp32 partials [M][K/256][N padded to 16];
 * every call leaves the counters zeroed again, so one workspace can be reused by calls of
 * any shape without clearing.  One workspace must not be used by two calls that can run
 * concurrently.  N <= 1,048,576.  The tiled kernels size their grid to the SM count and need
 * all their CTAs co-resident; do not co-schedule kernels that pin SMs for the whole call. */
size_t shiftadd_workspace_bytes(int layout, int M, int N, int K, int q, int g);

/* a2-a7 -- shift-and-add LUT-GEMM, M in [1, 16] (App. D :804-817):
 *   y[m][n] = fp16_rne( sum_i sum_G 2^{e[i][n][G]} sum_{k in G} s(i,n,k) x[m][k] )
 *   x    : fp16 [M][ldx], ldx >= K, rows 16-byte aligned
 *   planes, exps : packed by shiftadd_pack in `layout`, with the same q, N, K, g
 *   y    : fp16 [M][ldy], ldy >= N (a shard may write into a wider buffer)
 *   workspace: shiftadd_workspace_bytes(...) bytes, 16-byte aligned (NULL if 0)
 *   q    : 1..4 bits per weight of THIS layer (mixed-bit dispatch)
 *   flags: 0 or a combination of SHIFTADD_FLAG_PDL, SHIFTADD_FLAG_SPLITK
 * Accumulation is fp32 in a fixed order per launch shape: results are bit-identical run to
 * run on one device.  Exponents outside [EXP_MIN, EXP_MAX] (other than EXP_ZERO) are
 * undefined behaviour (pack never emits them).  NaN/Inf in x propagate to the outputs
 * whose dot product they enter. */
shiftadd_status shiftadd_lut_gemm(const uint16_t* x, int ldx, const uint8_t* planes,
                                  const int8_t* exps, int layout, int M, int N, int K, int q,
                                  int g, uint16_t* y, int ldy, void* workspace,
                                  size_t workspace_bytes, unsigned flags, void* stream);

/* Fused projections (§8 a3/a6; BASELINE north_star "mixed 2/3/4-bit per-layer dispatch"):
 * several output segments that read the same activations x -- LLaMA q/k/v, or gate/up --
 * in ONE launch, each with its own packed weights and bit width (PAPER.md:286-292 allocates
 * q per layer, so the k_proj of a block may carry 3 bits while q/v carry 2).  Segment i:
 *   y_i[n] = fp16_rne( sum_j sum_G 2^{e_i[j][n][G]} sum_{k in G} s_i(j,n,k) x[k] ), n < N_i.
 * Equivalent to nseg shiftadd_lut_gemv calls; the one launch builds each K-slice's LUT once
 * for all segments and streams their weights: K <= 4096 with <= 24 MB of planes on the
 * thread-block-cluster TMA ring (kernel id 10, K-split reduced over DSMEM, workspace unused),
 * otherwise -- or with SHIFTADD_FLAG_SPLITK -- as one byte range per slice on the all-SM
 * streaming kernel (id 8).  Batch 1 (M = 1), tiled layout only, K % 256 == 0, K <= 256 x #SMs,
 * 1 <= nseg <= 4, each segment 1 <= q <= 4 with planes / exps 16-B aligned (packed by
 * shiftadd_pack with the same K and g), y_i fp16 [N_i].  Workspace: shiftadd_workspace_bytes_fused
 * bytes (same zero-once contract as shiftadd_lut_gemm; calls of either kind may share it, not
 * concurrently).  flags: 0 or SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK. */
typedef struct {
  const uint8_t* planes; /* tiled planes of segment i            */
  const int8_t* exps;    /* tiled exponents of segment i         */
  int N;                 /* output rows of segment i             */
  int q;                 /* bit width of segment i (1..4)        */
  uint16_t* y;           /* fp16 [N] output of segment i         */
} shiftadd_segment;
size_t shiftadd_workspace_bytes_fused(int layout, int M, int K, int g, int nseg, const shiftadd_segment* segs);
shiftadd_status shiftadd_lut_gemv_fused(const uint16_t* x, int K, int g, int layout, int nseg,
                                        const shiftadd_segment* segs, void* workspace, size_t workspace_bytes,
                                        unsigned flags, void* stream);

/* A decode step as ONE persistent launch (§8 a2-a6 over a whole model; kernel id 9): an
 * ordered "program" of batch-1 calls of the shiftadd_lut_gemv_fused form -- in a decoder,
 * per block q/k/v, o, gate/up, down (PAPER.md:286-292 gives each layer its own q).  One CTA
 * per SM runs the calls in order; its producer warp streams the weights of call after call
 * into shared memory (weights never depend on activations), so HBM stays busy across call
 * boundaries, and the consumer warps build each call's LUTs, query, reduce and store y.
 * Call j computes, for every segment i, exactly what shiftadd_lut_gemv_fused computes:
 *   y_i[n] = fp16_rne( sum_j sum_G 2^{e_i[j][n][G]} sum_{k in G} s_i(j,n,k) x[k] ).
 * SHIFTADD_CALL_WAIT in a call's flags: x is read only after every earlier call of the
 * program has stored all of its y (the call consumes earlier outputs -- e.g. x of call j is
 * y of call j-1); without it, x must not be written by the program.  Outputs of different
 * calls must not overlap.
 * Usage: shiftadd_program_encode(calls) writes shiftadd_program_bytes(ncalls) bytes into a
 * caller HOST buffer; the caller copies them to DEVICE memory once (they hold the device
 * pointers of the calls, not the data); shiftadd_lut_gemv_program(calls, program, ...) then
 * launches with the same calls (validated again on the host; the kernel traps if the device
 * copy is not the encoding of these calls).
 * Per call: x fp16 [K] 16-B aligned, K % 256 == 0, 256 <= K <= 256 x #SMs, g % 128 == 0,
 * g | K, 1 <= nseg <= 4, each segment as in shiftadd_lut_gemv_fused (tiled layout).
 * Workspace: shiftadd_workspace_bytes_program(calls) bytes, zeroed once before first use,
 * used by program launches only (not shared with other entry points), one launch at a time.
 * flags: 0.  The launch is cooperative (one CTA per SM, all co-resident). */
#define SHIFTADD_CALL_WAIT 1u
typedef struct {
  const uint16_t* x;     /* fp16 [K] activations of this call                 */
  int K;                 /* reduction length                                   */
  int g;                 /* scale group of every segment (multiple of 128)     */
  int nseg;              /* output segments sharing x (1..4)                   */
  unsigned flags;        /* 0 or SHIFTADD_CALL_WAIT                            */
  shiftadd_segment seg[4];
} shiftadd_call;
size_t shiftadd_program_bytes(int ncalls);
shiftadd_status shiftadd_program_encode(const shiftadd_call* calls, int ncalls, void* out, size_t out_bytes);
size_t shiftadd_workspace_bytes_program(const shiftadd_call* calls, int ncalls);
shiftadd_status shiftadd_lut_gemv_program(const shiftadd_call* calls, int ncalls, const void* program,
                                          size_t program_bytes, void* workspace, size_t workspace_bytes,
                                          unsigned flags, void* stream);

/* The same ordered calls issued from the host as one kernel per call (no persistent kernel;
 * each call is the shift-and-LUT linear layer of PAPER.md:182-187):
 * each call goes through shiftadd_lut_gemm (one segment) or shiftadd_lut_gemv_fused, all on
 * `stream`, so a decode step costs one C call instead of one per projection.  With
 * SHIFTADD_FLAG_PDL every launch is a programmatic dependent of the previous one (x read after
 * the previous call completed: the decoder's dependency, as SHIFTADD_CALL_WAIT).  Workspace:
 * shiftadd_workspace_bytes_chain(calls) bytes (the calls share it in order).  Errors name the
 * failing call; calls before it have been enqueued. */
size_t shiftadd_workspace_bytes_chain(const shiftadd_call* calls, int ncalls);
shiftadd_status shiftadd_lut_gemv_chain(const shiftadd_call* calls, int ncalls, void* workspace,
                                        size_t workspace_bytes, unsigned flags, void* stream);

/* Batch-1 convenience: shiftadd_lut_gemm with M = 1, ldx = K, ldy = N. */
shiftadd_status shiftadd_lut_gemv(const uint16_t* x, const uint8_t* planes, const int8_t* exps,
                                  int layout, int N, int K, int q, int g, uint16_t* y,
                                  void* workspace, size_t workspace_bytes, unsigned flags,
                                  void* stream);

/* NEXT-f1 -- column-wise scales, "Ours (Acc.)" (Fig. 3(c); the paper's
 * open gap "we lack the fast CUDA kernel", :545).  Plane i has one PoT scale per input
 * column k, shared by all output rows:  W_hat[n][k] = sum_i 2^{e_i[k]} s_i(n, k).
 *
 * shiftadd_pack_colwise: signs int8 [q][N][K] (+-1), alpha_col fp32 [q][K] ->
 *   planes (same byte format and layouts as shiftadd_pack, with each column's sign folded
 *   into that column's bits of every row) and exps_col int8 [q][K] (same P rule, zero
 *   sentinel and clamp counting as shiftadd_pack; no layout permutation).  1 <= q <= 8,
 *   K % 8 == 0 (tiled: K % 256 == 0), N <= 1,048,576.  Errors as shiftadd_pack.
 *
 * shiftadd_lut_gemv_colwise: y[n] = fp16_rne( sum_i sum_k s_i(n,k) 2^{e_i[k]} x[k] ), M = 1,
 *   tiled layout.  The kernel follows SPEC.md:375 (ColumnWisePerPlane): per 256-k slice it
 *   builds one LUT bank per plane from x[k] * 2^{e_i[k]} (an exact fp32 shift), queries it
 *   with that plane's key bytes and accumulates unscaled; the K-split is reduced inside a
 *   thread-block cluster of K/256 CTAs.  Supported: layout TILED, K % 256 == 0,
 *   K <= 4096, N such that a cluster band holds <= 512 row groups (N <= ~57 K rows on
 *   B200); otherwise SHIFTADD_ERR_UNSUPPORTED.  1 <= q <= 4.  flags: 0 or SHIFTADD_FLAG_PDL.  No
 *   workspace.  x 16-byte aligned, planes 16-byte aligned, exps_col 8-byte aligned. */
shiftadd_status shiftadd_pack_colwise(const int8_t* signs, const float* alpha_col, int q, int N, int K,
                                      int layout, uint8_t* planes, int8_t* exps_col, int32_t* counts,
                                      void* stream);
shiftadd_status shiftadd_lut_gemv_colwise(const uint16_t* x, const uint8_t* planes, const int8_t* exps_col,
                                          int layout, int N, int K, int q, uint16_t* y, unsigned flags,
                                          void* stream);
/* shiftadd_lut_gemv_colwise_ws: the same result for any K % 256 == 0 up to 256 x #SMs (the
 *   LLaMA-2-70B / OPT-66B shapes the cluster kernel cannot hold).  K <= 4096 shapes the
 *   cluster kernel takes go there (no workspace touched) unless flags has
 *   SHIFTADD_FLAG_SPLITK; otherwise the all-SM streaming kernel (id 8) builds, per 256-k slice,
 *   plane i's LUT from x[k] 2^{e_i[k]} and reduces the K-split through `workspace`
 *   (shiftadd_workspace_bytes_colwise(N, K) bytes, same zero-once contract as
 *   shiftadd_lut_gemm).  flags: 0 or SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK. */
/* shiftadd_lut_gemm_colwise: the same for M <= 16 batch rows x [M][K] (row stride ldx, a
 *   multiple of 8), y [M][N] (row stride ldy) -- a7 with column-wise scales: pairs of rows
 *   share one weight pass (plane LUT entries hold the fp16 pair of both rows' sums, built in
 *   fp32 and rounded once, PAPER.md:186's FP16 LUT); M = 1 is shiftadd_lut_gemv_colwise_ws. */
size_t shiftadd_workspace_bytes_colwise(int N, int K);
shiftadd_status shiftadd_lut_gemv_colwise_ws(const uint16_t* x, const uint8_t* planes, const int8_t* exps_col,
                                             int layout, int N, int K, int q, uint16_t* y, void* workspace,
                                             size_t workspace_bytes, unsigned flags, void* stream);
shiftadd_status shiftadd_lut_gemm_colwise(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps_col,
                                          int layout, int M, int N, int K, int q, uint16_t* y, int ldy,
                                          void* workspace, size_t workspace_bytes, unsigned flags, void* stream);

/* NEXT-f1 -- block-wise scales, "Ours (Lat.)" (Fig. 4(a)): "a block-wise
 * scaling factor design that groups 8 columns and 1/8 of the original rows to share a scaling
 * factor, ensuring compatibility with the BCQ kernel".  Plane i has one PoT scale per (row
 * block b = n / (N/8), column group c = k / 8) -- the 8 weights of a key byte share it:
 *   W_hat[n][k] = sum_i 2^{e_i[n / (N/8)][k / 8]} s_i(n, k)       (reading R24)
 *
 * shiftadd_pack_blockwise: signs int8 [q][N][K] (+-1), alpha_bw fp32 [q][8][K/8] -> planes
 *   (same byte format and layouts as shiftadd_pack, each block's sign folded into its 8-bit
 *   groups) and exps_bw int8 [q][8][K/8] (the compact layout: q K bytes; same P rule, zero
 *   sentinel and clamp counting as shiftadd_pack).  8 | N, K % 8 == 0 (tiled: K % 256 == 0).
 *
 * shiftadd_lut_gemv_blockwise: y[n] = fp16_rne( sum_i sum_c 2^{e_i[b(n)][c]} T_c[key_i(n, c)] ),
 *   M = 1, tiled planes: every LUT query is scaled by its block's 2^e (one FFMA per query; the
 *   lane keeps its 16 q scale factors in registers, the exponent array is read once per CTA,
 *   never streamed).  K % 256 == 0, K <= 256 x #SMs, 8 | N, 1 <= q <= 4.  Workspace:
 *   shiftadd_workspace_bytes_blockwise(N, K) bytes (shiftadd_lut_gemm's zero-once contract).
 *   flags: 0 or SHIFTADD_FLAG_PDL.  planes 16-B aligned, x 16-B aligned. */
shiftadd_status shiftadd_pack_blockwise(const int8_t* signs, const float* alpha_bw, int q, int N, int K, int layout,
                                       uint8_t* planes, int8_t* exps_bw, int32_t* counts, void* stream);
size_t shiftadd_workspace_bytes_blockwise(int N, int K);
shiftadd_status shiftadd_lut_gemv_blockwise(const uint16_t* x, const uint8_t* planes, const int8_t* exps_bw,
                                            int layout, int N, int K, int q, uint16_t* y, void* workspace,
                                            size_t workspace_bytes, unsigned flags, void* stream);

/* NEXT-f2 -- additive PoT with K = 2 terms per scale (Eq. 2: "the k-th
 * PoT minimizes the residual of the (k-1)-th").
 *
 * shiftadd_pack_apot2: as shiftadd_pack (same planes and exps: term 1, P1 = round(log2|a|),
 *   its sign folded into the bits) plus exps2 (int8, same size and layout permutation as
 *   exps): the second term relative to the first, c2 = s1*s2*(P1 - P2) with
 *   P2 = round(log2|a - s1 2^P1|), so a group's folded scale is 2^P1 (1 + sign(c2) 2^-|c2|).
 *   c2 = 0 when a is 0, P1 was clamped, the residual is 0, P2 < EXP_MIN or P1 - P2 > 127.
 *
 * shiftadd_lut_gemm_apot2: y[m][n] = fp16_rne( sum_i sum_G 2^{e_i} (1 + sign(c2) 2^-|c2|)
 *   sum_{k in G} s(i,n,k) x[m][k] ): each 128-k chunk (tiled) or lookup (canonical) sum p
 *   adds v1 = p 2^{e1} and sign(c2) v1 2^-|c2| (two exponent adds).  Supported: canonical
 *   layout, any shape shiftadd_lut_gemm accepts (M <= 16); tiled layout, M = 1, K <= 4096
 *   (and K <= 8192 up to 12 MB of planes) -- otherwise SHIFTADD_ERR_UNSUPPORTED.  No
 *   workspace.  flags: 0 or SHIFTADD_FLAG_PDL.  Terms below 2^-126 are flushed to 0. */
shiftadd_status shiftadd_pack_apot2(const int8_t* signs, const float* alpha, int q, int N, int K, int g,
                                    int layout, uint8_t* planes, int8_t* exps, int8_t* exps2, int32_t* counts,
                                    void* stream);
shiftadd_status shiftadd_lut_gemm_apot2(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                        const int8_t* exps2, int layout, int M, int N, int K, int q, int g,
                                        uint16_t* y, int ldy, unsigned flags, void* stream);
/* shiftadd_lut_gemm_apot2_ws: the same with a workspace, which lets tiled batch-1 layers the
 *   cluster kernel cannot take (K > 4096: the LLaMA-2-70B / OPT-66B shapes; or with
 *   SHIFTADD_FLAG_SPLITK) run on the all-SM streaming kernel (id 8) with the second-term codes
 *   streamed beside the exponents (exps, exps2 16-B aligned; workspace
 *   shiftadd_workspace_bytes_apot2(N, K) bytes, same zero-once contract as shiftadd_lut_gemm).
 *   flags: 0 or SHIFTADD_FLAG_PDL | SHIFTADD_FLAG_SPLITK. */
size_t shiftadd_workspace_bytes_apot2(int N, int K);
shiftadd_status shiftadd_lut_gemm_apot2_ws(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                           const int8_t* exps2, int layout, int M, int N, int K, int q, int g,
                                           uint16_t* y, int ldy, void* workspace, size_t workspace_bytes,
                                           unsigned flags, void* stream);

/* NEXT-f4 -- Alg. 1 alternating multi-bit BCQ quantiser, the step before
 * shiftadd_pack.  Per scale group (g consecutive k of one output row of w fp32 [N][K]):
 * greedy init (Eq. 1: b_i = sign(r_{i-1}), sign(0) = +1; alpha_i = mean|r_{i-1}|), then T
 * cycles of least-squares scale refit alpha = (B^T B + 1e-8 g I)^-1 B^T w (Line 6) -- with
 * SHIFTADD_BCQ_POT each alpha_i is then projected to sign * 2^round(log2|alpha_i|) (Eq. 2,
 * K = 1) -- and code refit to the nearest representable level sum_i +-alpha_i (Line 7; ties
 * -> smaller |level|, then the negative level).  fp64 throughout.
 *   w     : fp32 [N][K] device, 4-byte aligned;  1 <= q <= 4;  g | K, 1 <= g;  0 <= T <= 1000
 *   signs : int8 [q][N][K] device (output, +-1; the codes of the final alphas)
 *   alpha : fp32 [q][N][K/g] device (output; feed both to shiftadd_pack)
 * One CTA per group; N*K/g < 2^31.  Errors: SHIFTADD_ERR_INVALID on bad sizes/pointers. */
#define SHIFTADD_BCQ_POT 1u
shiftadd_status shiftadd_bcq_quantize(const float* w, int N, int K, int q, int g, int T, unsigned flags,
                                      int8_t* signs, float* alpha, void* stream);

/* NEXT-f3 -- batch-1 LUT-GEMV with the all-gather fused into its epilogue (§8(e) rows are
 * independent per rank; BASELINE.json north_star's all-gather of y).  Rank `rank` of P owns
 * N rows (its packed shard).  Call c = *epoch + 1 stores each output element directly into
 * every rank's gathered buffer c % 2, y_peers[(c%2)*P + r][rank*N + n] (peer memory over
 * NVLink / CUDA IPC); the last CTA of the launch then publishes c into flag_peers[r][rank]
 * of every rank (one system-scope release pattern).  shiftadd_gather_wait(flags_local, P,
 * epoch) enqueues a wait (acquire, system scope) until all P ranks have published
 * *epoch + 1 and then advances *epoch; after it the local buffer c % 2 holds the whole y
 * [P*N].  The call counter lives on the device, so both calls may be captured in a CUDA graph
 * and replayed.  Double buffering is safe: a rank reaches call c + 2 only after every rank
 * finished call c + 1, which consumed buffer c % 2.
 *   y_peers: device array of 2P device pointers; flag_peers: device array of P device
 *   pointers (flag arrays uint32[P], zero-initialised); epoch: device uint32, starts at 0,
 *   one per (rank, layer).  2 <= P <= 8.
 *   workspace: shiftadd_workspace_bytes(...) and >= 256 KB + 16 B (a launch counter at
 *   byte 256 KB, left zero).  Supported: tiled layout; K <= 4096 shapes the cluster kernel
 *   takes (kernel id 3), and 512 <= K <= 256 x #SMs with 16-B aligned exps on the all-SM
 *   streaming kernel (id 8, whose owner CTAs store into the peers); otherwise
 *   SHIFTADD_ERR_UNSUPPORTED.
 *   The wait traps (CUDA error) after ~5 s without progress instead of hanging. */
shiftadd_status shiftadd_lut_gemv_gather(const uint16_t* x, const uint8_t* planes, const int8_t* exps, int layout,
                                         int N, int K, int q, int g, uint16_t* const* y_peers,
                                         uint32_t* const* flag_peers, int P, int rank, uint32_t* epoch,
                                         void* workspace, size_t workspace_bytes, unsigned flags, void* stream);
/* shiftadd_lut_gemm_gather: the same for M <= 8 batch rows (x [M][K], row stride ldx): every
 *   rank's gathered buffer holds y [M][P*N] (row m at m*P*N, this rank's rows at rank*N);
 *   M > 1 runs on the all-SM streaming kernel (one weight pass, M-wide fp16 LUT entries).
 *   shiftadd_lut_gemv_gather is the M = 1 form. */
shiftadd_status shiftadd_lut_gemm_gather(const uint16_t* x, int ldx, const uint8_t* planes, const int8_t* exps,
                                         int layout, int M, int N, int K, int q, int g, uint16_t* const* y_peers,
                                         uint32_t* const* flag_peers, int P, int rank, uint32_t* epoch,
                                         void* workspace, size_t workspace_bytes, unsigned flags, void* stream);
shiftadd_status shiftadd_gather_wait(const uint32_t* flags_local, int P, uint32_t* epoch, void* stream);

/* §8(d) e2e -- stream-ordered copy between device memory and pinned (page-locked, UVA-mapped)
 * host memory done by a small kernel instead of the copy engine: a decode step's inputs
 * host->device and its outputs device->host are kilobytes, where a copy-engine memcpy node
 * costs ~10 us of latency; the kernel reads or writes the host buffer over PCIe directly and
 * joins the PDL chain of the step's GEMV launches.
 *   dst, src: device or pinned host pointers (either direction, or device to device),
 *   16-B aligned; bytes: any multiple of 16 (INVALID otherwise).
 *   flags: SHIFTADD_FLAG_PDL launches with programmatic dependent launch: the copy writes dst
 *   only after griddepcontrol.wait (the preceding kernel has finished reading dst);
 *   SHIFTADD_COPY_SRC_READY additionally lets it read src before that wait (src is not
 *   written by the preceding kernel, e.g. host inputs), so the PCIe read overlaps it.
 * No allocation; asynchronous faults surface at the next sync. */
#define SHIFTADD_COPY_SRC_READY 4u
shiftadd_status shiftadd_copy(void* dst, const void* src, size_t bytes, unsigned flags, void* stream);

/* Launch geometry the gemm call would use (for measurement/reporting; host only):
 * out[0] = grid CTAs, out[1] = threads per CTA, out[2] = dynamic smem bytes,
 * out[3] = kernel id (0 generic, 1 tiled M=1 split-K, 2 tiled small-batch, 3 tiled M=1
 * cluster split-K (TMA weight ring), 4 tiled M=1 split-K with the TMA weight ring, 5 tiled M=2
 * cluster TMA ring, 6 tiled M=3..4 cluster TMA ring, 7 tiled M>4 as row chunks of <= 4
 * through 5/6, 8 tiled all-SM streaming LUT-GEMV), for flags = 0.  Needs a device. */
shiftadd_status shiftadd_gemm_plan(int layout, int M, int N, int K, int q, int g, int out[4]);

#ifdef __cplusplus
}
#endif
#endif /* SHIFTADD_H */
