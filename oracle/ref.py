"""fp64 CPU oracle for the ShiftAddLLM shift-and-add LUT-GEMV (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  It never imports the product package and shares no code with it.

What the hot path computes (PAPER.md, arxiv 2406.05981):
  * BCQ weights  w_q = sum_i alpha_i b_i,  b_i in {-1,+1}            (§3)
  * PoT scales   POT(alpha) = sign(alpha) 2^P,  P = round(log2|alpha|) (Eq. 2)
  * shift        x * 2^P is an add on the float exponent field        (§4.1)
  * LUT          256 partial sums per 8 activations, n/8 LUTs, every
                 8 grouped binary weights form an 8-bit key           (§4.1)
  * output       "add all the partial sums ... in FP16 format"

Since the LUT method reaches exactly (up to summation order and the final fp16 rounding)
the BCQ product, the oracle is that definition written out: dequantise
W_hat = sum_i 2^{e_i} s_i from the packed bytes and do a naive fp64 matvec (``gemm``).
``lut_gemm`` follows the paper's LUT route step by step as a second route, and
``gemm_scalar`` is a pure-Python loop for small shapes.  Readings of points where the paper
is silent are DESIGN.md §Readings R1..R15 (same numbering as SURVEY.md §8(c) C1..C15).
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

# Exponent encoding (reading R5 / SURVEY C5): alpha == 0 -> sentinel, finite
# exponents clamped into [EXP_MIN, EXP_MAX] and counted.  Defined here independently of
# include/shiftadd.h (the oracle shares no constants with the product).
EXP_ZERO = -128
EXP_MIN = -100
EXP_MAX = 100

# Device-tiled layout geometry: a tile is 16 output rows x 256
# reduction indices (32 key bytes per row) of one plane.
TILE_ROWS = 16
TILE_K = 256

__all__ = [
    "EXP_ZERO", "EXP_MIN", "EXP_MAX", "TILE_ROWS", "TILE_K",
    "pot_exponent", "pack_canonical", "unpack_signs", "to_tiled", "from_tiled",
    "tiled_sizes", "dequant", "gemm", "gemm_scalar", "lut_direct", "lut_incremental",
    "lut_gemm", "to_fp16", "err_floor", "err_normwise", "packed_bytes",
    "algorithmic_bytes", "tile_planes", "pack_colwise", "dequant_colwise", "gemm_colwise",
    "lut_gemm_colwise", "algorithmic_bytes_colwise", "additive_pot", "pack_apot2",
    "dequant_apot2", "gemm_apot2", "pot_round_exact", "bcq_greedy", "bcq_ls", "bcq_bs_codes",
    "bcq_quantize", "pack_blockwise", "dequant_blockwise", "gemm_blockwise", "lut_gemm_blockwise",
    "blockwise_row_exps", "algorithmic_bytes_blockwise",
]


# ----------------------------------------------------------------------------- a1: pack
def pot_exponent(alpha):
    """P = round(log2 |alpha|) for every alpha (Eq. 2), fp64.

    Returns (exps int8 array, n_clamped).  alpha == +-0 -> EXP_ZERO (reading R5); a finite
    P outside [EXP_MIN, EXP_MAX] is clamped and counted (R5); non-finite alpha raises
    ValueError.  Ties are impossible: log2|alpha| = k + 1/2 needs alpha = 2^(k+1/2), which is
    irrational, and an fp32 alpha is at least 2^-24 relative away from it, far beyond fp64's
    log2 error, so fp64 ``rint(log2)`` is the exact rounding for every fp32 input.
    """
    a = np.asarray(alpha, dtype=np.float32)
    if not np.all(np.isfinite(a)):
        raise ValueError("non-finite scale factor")
    mag = np.abs(a.astype(np.float64))
    zero = mag == 0.0
    with np.errstate(divide="ignore"):
        p = np.rint(np.log2(np.where(zero, 1.0, mag)))
    clamped = (~zero) & ((p < EXP_MIN) | (p > EXP_MAX))
    p = np.clip(p, EXP_MIN, EXP_MAX)
    out = np.where(zero, EXP_ZERO, p).astype(np.int8)
    return out, int(np.count_nonzero(clamped))


def pack_canonical(signs, alpha, g):
    """Pack q sign planes + scales into key bytes and PoT exponents (§8(a1), canonical layout).

    signs : int8 [q][N][K], every entry -1 or +1      (b_i in {-1,1}^{m x n})
    alpha : float32 [q][N][K/g]                        (group-wise scale alpha_i)
    g     : scale-group length along K (8 | g, g | K)  (reading R6)

    Steps, in order:
      1. sign fold (R3): alpha*b = (-alpha)(-b), so a group whose alpha < 0 gets its signs
         negated and keeps |alpha|; Eq. 2's sign(alpha) then lives in the bits.
      2. exponent: P = round(log2|alpha|)  (pot_exponent).
      3. bits: key byte planes[i][n][k>>3] bit (k&7) = 1  <=>  folded sign = +1
         (R1: LSB = lowest k of the 8 grouped weights, 1 <-> +1; R2: the 8
         weights of a key are 8 consecutive reduction indices of one output row).
    Returns planes uint8 [q][N][K/8], exps int8 [q][N][K/g], n_clamped.
    """
    s = np.asarray(signs)
    a = np.asarray(alpha, dtype=np.float32)
    if s.ndim != 3:
        raise ValueError("signs must be [q][N][K]")
    q, n, k = s.shape
    if g <= 0 or g % 8 or k % 8 or k % g:
        raise ValueError("need 8 | g, g | K and 8 | K")
    if a.shape != (q, n, k // g):
        raise ValueError("alpha must be [q][N][K/g]")
    if not np.all((s == 1) | (s == -1)):
        raise ValueError("signs must be -1 or +1")
    exps, n_clamped = pot_exponent(a)
    flip = np.repeat(a < 0, g, axis=2)                      # step 1, per element of the group
    folded = np.where(flip, -s.astype(np.int16), s.astype(np.int16))
    bits = (folded == 1).astype(np.uint8).reshape(q, n, k // 8, 8)
    weights = (1 << np.arange(8, dtype=np.uint16)).astype(np.uint16)   # bit b <-> k = 8t+b
    planes = (bits.astype(np.uint16) * weights).sum(axis=3).astype(np.uint8)
    return planes, exps, n_clamped


def unpack_signs(planes, K):
    """Inverse of step 3: key bytes -> {-1,+1} int8 [q][N][K] (reading R1)."""
    p = np.asarray(planes, dtype=np.uint8)
    bits = (p[..., :, None] >> np.arange(8, dtype=np.uint8)) & 1
    bits = bits.reshape(p.shape[:-1] + (p.shape[-1] * 8,))[..., :K]
    return np.where(bits == 1, 1, -1).astype(np.int8)


# ------------------------------------------------------------------- a1: tiled layout
def tiled_sizes(q, N, K):
    """Byte sizes (planes, exps) of the device-tiled layout."""
    rg = -(-N // TILE_ROWS)
    s = K // TILE_K
    return s * rg * q * TILE_ROWS * (TILE_K // 8), s * rg * q * TILE_ROWS * 2


def to_tiled(planes, exps, g):
    """Permute canonical bytes into the device-tiled layout.

    A tile is (slice s of 256 k, row-group rg of 16 rows, plane i); tiles are stored in
    (s, rg, i) order, 512 plane bytes each:
        off = ((s*RG + rg)*q + i)*512 + r*32 + h*16 + j
        val = planes[i][16 rg + r][32 s + 16 h + ((j + r) mod 16)]   (0 for rows >= N)
    and one exponent per 128-k chunk (h) of each row:
        off = ((s*RG + rg)*q + i)*32 + r*2 + h
        val = exps[i][16 rg + r][(256 s + 128 h) // g]               (EXP_ZERO for rows >= N)
    The (j + r) mod 16 rotation is a pure byte permutation; it is what lets 16 rows read 16
    different LUTs in the same step.  Requires 256 | K and 128 | g.
    """
    p = np.asarray(planes, dtype=np.uint8)
    e = np.asarray(exps, dtype=np.int8)
    q, n, kb = p.shape
    K = kb * 8
    if K % TILE_K or g % 128 or K % g:
        raise ValueError("tiled layout needs 256 | K and 128 | g")
    RG = -(-n // TILE_ROWS)
    S = K // TILE_K
    npad = RG * TILE_ROWS
    pp = np.zeros((q, npad, kb), dtype=np.uint8)
    pp[:, :n] = p
    ep = np.full((q, npad, K // g), EXP_ZERO, dtype=np.int8)
    ep[:, :n] = e
    out_p = np.zeros(S * RG * q * 512, dtype=np.uint8)
    out_e = np.zeros(S * RG * q * 32, dtype=np.int8)
    # Walk the definition element by element (vectorised over r, h, j only).
    r = np.arange(16)[:, None, None]
    h = np.arange(2)[None, :, None]
    j = np.arange(16)[None, None, :]
    for s in range(S):
        for rg in range(RG):
            rows = TILE_ROWS * rg + r
            cols = 32 * s + 16 * h + (j + r) % 16
            erow = TILE_ROWS * rg + np.arange(16)[:, None]
            ecol = (256 * s + 128 * np.arange(2)[None, :]) // g
            for i in range(q):
                base = ((s * RG + rg) * q + i)
                out_p[base * 512:(base + 1) * 512] = pp[i, rows, cols].reshape(-1)
                out_e[base * 32:(base + 1) * 32] = ep[i, erow, ecol].reshape(-1)
    return out_p, out_e


def from_tiled(planes_t, exps_t, q, N, K, g):
    """Inverse permutation of ``to_tiled`` (for g == 128 the exps map back one-to-one)."""
    pt = np.asarray(planes_t, dtype=np.uint8)
    et = np.asarray(exps_t, dtype=np.int8)
    RG = -(-N // TILE_ROWS)
    S = K // TILE_K
    planes = np.zeros((q, RG * TILE_ROWS, K // 8), dtype=np.uint8)
    exps = np.full((q, RG * TILE_ROWS, K // g), EXP_ZERO, dtype=np.int8)
    for s in range(S):
        for rg in range(RG):
            for i in range(q):
                base = ((s * RG + rg) * q + i)
                tile = pt[base * 512:(base + 1) * 512].reshape(16, 2, 16)
                etile = et[base * 32:(base + 1) * 32].reshape(16, 2)
                for r in range(16):
                    n = TILE_ROWS * rg + r
                    for h in range(2):
                        for j in range(16):
                            planes[i, n, 32 * s + 16 * h + (j + r) % 16] = tile[r, h, j]
                        exps[i, n, (256 * s + 128 * h) // g] = etile[r, h]
    return planes[:, :N], exps[:, :N]


# --------------------------------------------------------------- definition: dequant + gemm
def dequant(planes, exps, g, K):
    """W_hat[n][k] = sum_i 2^{e_i[n][k//g]} * s_i[n][k]  (PAPER.md:120 with Eq. 2), fp64.

    EXP_ZERO groups contribute 0.  Each term is +-2^e; the sum of the q terms is exact in
    fp64 whenever the exponents of one element span < 53 binades (always true for the
    synthetic and test inputs, whose exponents span < 20).
    """
    p = np.asarray(planes, dtype=np.uint8)
    e = np.asarray(exps, dtype=np.int8).astype(np.int64)
    q, n, _ = p.shape
    s = unpack_signs(p, K).astype(np.float64)                        # [q][N][K]
    scale = np.where(e == EXP_ZERO, 0.0, np.ldexp(1.0, np.where(e == EXP_ZERO, 0, e)))
    scale = np.repeat(scale, g, axis=2)                              # [q][N][K]
    return (s * scale).sum(axis=0)


def gemm(x, planes, exps, g, row_chunk=2048):
    """y = x W_hat^T in fp64 (the plain definition; §8(c)).  x: [M][K] (any float dtype).

    Row-chunked over N only to bound memory; each output is a plain fp64 dot product.
    """
    xf = np.asarray(x, dtype=np.float64)
    if xf.ndim == 1:
        xf = xf[None, :]
    p = np.asarray(planes, dtype=np.uint8)
    e = np.asarray(exps, dtype=np.int8)
    q, n, kb = p.shape
    K = kb * 8
    if xf.shape[1] != K:
        raise ValueError("x must be [M][K]")
    y = np.empty((xf.shape[0], n), dtype=np.float64)
    for n0 in range(0, n, row_chunk):
        n1 = min(n, n0 + row_chunk)
        w = dequant(p[:, n0:n1], e[:, n0:n1], g, K)
        y[:, n0:n1] = xf @ w.T
    return y


def gemm_scalar(x, planes, exps, g):
    """Pure-Python triple loop over the packed bytes (Python floats are fp64).

    y[m][n] = sum_i sum_k s_i(n,k) 2^{e_i(n, k//g)} x[m][k], s = +1 iff bit (k&7) of byte
    planes[i][n][k>>3] is set.  For small shapes and config 1 only.
    """
    xs = [[float(v) for v in row] for row in np.atleast_2d(np.asarray(x, dtype=np.float64))]
    p = np.asarray(planes, dtype=np.uint8).tolist()
    e = np.asarray(exps, dtype=np.int8).tolist()
    q = len(p)
    n = len(p[0])
    K = len(p[0][0]) * 8
    out = []
    for xm in xs:
        row = []
        for nn in range(n):
            acc = 0.0
            for i in range(q):
                bytes_ = p[i][nn]
                ex = e[i][nn]
                for k in range(K):
                    ei = ex[k // g]
                    if ei == EXP_ZERO:
                        continue
                    bit = (bytes_[k >> 3] >> (k & 7)) & 1
                    term = math.ldexp(xm[k], ei)
                    acc += term if bit else -term
            row.append(acc)
        out.append(row)
    return np.asarray(out, dtype=np.float64)


# ------------------------------------------------------------------- the paper's LUT route
def lut_direct(x8):
    """T[key] = sum_{b<8} (bit_b(key) ? +1 : -1) * x_b for key = 0..255.

    fp64; exact for any 8 fp16 inputs (40-bit fp16 span + 3 carry bits < 53).
    """
    xv = np.asarray(x8, dtype=np.float64).reshape(-1)
    if xv.shape[0] != 8:
        raise ValueError("x8 must have 8 entries")
    keys = np.arange(256)
    signs = np.where(((keys[:, None] >> np.arange(8)[None, :]) & 1) == 1, 1.0, -1.0)
    return (signs * xv[None, :]).sum(axis=1)


def lut_incremental(x8):
    """Same table by the lowest-set-bit recursion: T[0] = -sum x,
    T[key] = T[key & (key-1)] + 2 x_{lowest set bit of key}."""
    xv = [float(v) for v in np.asarray(x8, dtype=np.float64).reshape(-1)]
    t = [0.0] * 256
    t[0] = -sum(xv)
    for key in range(1, 256):
        low = (key & -key).bit_length() - 1
        t[key] = t[key & (key - 1)] + 2.0 * xv[low]
    return np.asarray(t, dtype=np.float64)


def lut_gemm(x, planes, exps, g):
    """The paper's route (§4.1, Fig. 2(c,d)) in fp64, step by step:

      1. build n/8 LUTs per activation row (lut_direct on each 8-activation group);
      2. query: each key byte planes[i][n][t] selects T_t[key];
      3. add the queried partial sums over a scale group G;
      4. shift: multiply the group sum by 2^{e_i[n][G]} (EXP_ZERO -> 0);
      5. add over groups and planes.
    """
    xf = np.atleast_2d(np.asarray(x, dtype=np.float64))
    p = np.asarray(planes, dtype=np.uint8)
    e = np.asarray(exps, dtype=np.int8).astype(np.int64)
    q, n, kb = p.shape
    K = kb * 8
    gb = g // 8
    y = np.zeros((xf.shape[0], n), dtype=np.float64)
    t_idx = np.arange(kb)[None, :]
    for m in range(xf.shape[0]):
        luts = np.stack([lut_direct(xf[m, 8 * t:8 * t + 8]) for t in range(kb)])  # [K/8][256]
        for i in range(q):
            looked = luts[t_idx, p[i].astype(np.int64)]                  # [N][K/8]
            grp = looked.reshape(n, K // g, gb).sum(axis=2)               # [N][K/g]
            ei = e[i]
            scale = np.where(ei == EXP_ZERO, 0.0, np.ldexp(1.0, np.where(ei == EXP_ZERO, 0, ei)))
            y[m] += (grp * scale).sum(axis=1)
    return y


# ------------------------------------- NEXT-f1: column-wise scales ("Ours (Acc.)", §4.2)
# PAPER.md:223-228 (Fig. 3(c)): "column-wise scaling factors ... Each scaling factor
# corresponds to a constant activation value": plane i has one scale alpha_i[k] per input
# column k, shared by every output row.  The LUT realisation is SPEC.md:375
# (ColumnWisePerPlane): "for each plane i, activations are pre-shifted per column by that
# plane's column PotScale, one LUT bank per plane built from shifted x; queries then
# accumulate unscaled".  Readings R17-R18.
def tile_planes(planes):
    """The device-tiled permutation of plane bytes alone (same tiles as ``to_tiled``)."""
    p = np.asarray(planes, dtype=np.uint8)
    q, n, kb = p.shape
    zeros = np.zeros((q, n, 1), dtype=np.int8)
    return to_tiled(p, zeros, kb * 8)[0]


def pack_colwise(signs, alpha_col):
    """signs int8 [q][N][K] (+-1), alpha_col float32 [q][K] -> planes, exps_col, n_clamped.

      1. sign fold per column (R3 applied to a column group, R17): alpha_i[k] < 0 negates
         s_i[n][k] for every row n and keeps |alpha_i[k]|;
      2. exponent: P = round(log2|alpha_i[k]|) (pot_exponent: same zero/clamp rules);
      3. bits exactly as pack_canonical step 3 (R1, R2).
    Returns planes uint8 [q][N][K/8], exps_col int8 [q][K], n_clamped.
    """
    s = np.asarray(signs)
    a = np.asarray(alpha_col, dtype=np.float32)
    if s.ndim != 3:
        raise ValueError("signs must be [q][N][K]")
    q, n, k = s.shape
    if k % 8:
        raise ValueError("need 8 | K")
    if a.shape != (q, k):
        raise ValueError("alpha_col must be [q][K]")
    if not np.all((s == 1) | (s == -1)):
        raise ValueError("signs must be -1 or +1")
    exps, n_clamped = pot_exponent(a)
    flip = (a < 0)[:, None, :]
    folded = np.where(flip, -s.astype(np.int16), s.astype(np.int16))
    bits = (folded == 1).astype(np.uint8).reshape(q, n, k // 8, 8)
    weights = (1 << np.arange(8, dtype=np.uint16)).astype(np.uint16)
    planes = (bits.astype(np.uint16) * weights).sum(axis=3).astype(np.uint8)
    return planes, exps, n_clamped


def _pow2(e):
    e = np.asarray(e, dtype=np.int64)
    return np.where(e == EXP_ZERO, 0.0, np.ldexp(1.0, np.where(e == EXP_ZERO, 0, e)))


def dequant_colwise(planes, exps_col, K):
    """W_hat[n][k] = sum_i 2^{e_i[k]} s_i[n][k] (column-wise PoT scales), fp64."""
    p = np.asarray(planes, dtype=np.uint8)
    s = unpack_signs(p, K).astype(np.float64)                  # [q][N][K]
    scale = _pow2(exps_col)[:, None, :]                         # [q][1][K]
    return (s * scale).sum(axis=0)


def gemm_colwise(x, planes, exps_col, row_chunk=2048):
    """y = x W_hat^T in fp64 with column-wise scales (the plain definition)."""
    xf = np.atleast_2d(np.asarray(x, dtype=np.float64))
    p = np.asarray(planes, dtype=np.uint8)
    q, n, kb = p.shape
    K = kb * 8
    if xf.shape[1] != K or np.asarray(exps_col).shape != (q, K):
        raise ValueError("x must be [M][K] and exps_col [q][K]")
    y = np.empty((xf.shape[0], n), dtype=np.float64)
    for n0 in range(0, n, row_chunk):
        n1 = min(n, n0 + row_chunk)
        y[:, n0:n1] = xf @ dequant_colwise(p[:, n0:n1], exps_col, K).T
    return y


def lut_gemm_colwise(x, planes, exps_col):
    """SPEC.md:375 ColumnWisePerPlane, step by step, fp64:

      1. pre-shift: x_i[k] = 2^{e_i[k]} * x[k]  (EXP_ZERO -> 0)     (the paper's step (1),
         "bitwise shifts between activations and scaling factors");
      2. one LUT bank per plane: lut_direct on each 8-group of x_i;
      3. query: plane i's key byte planes[i][n][t] selects bank_i T_t[key];
      4. add all queried partial sums (no per-group shift).
    """
    xf = np.atleast_2d(np.asarray(x, dtype=np.float64))
    p = np.asarray(planes, dtype=np.uint8)
    q, n, kb = p.shape
    sc = _pow2(exps_col)
    y = np.zeros((xf.shape[0], n), dtype=np.float64)
    t_idx = np.arange(kb)[None, :]
    for m in range(xf.shape[0]):
        for i in range(q):
            xi = xf[m] * sc[i]
            bank = np.stack([lut_direct(xi[8 * t:8 * t + 8]) for t in range(kb)])   # [K/8][256]
            y[m] += bank[t_idx, p[i].astype(np.int64)].sum(axis=1)
    return y


# ------------------------------------------------ NEXT-f1: block-wise scales, "Ours (Lat.)"
# PAPER.md:239-244 (§4.2, Fig. 4(a)): "a block-wise scaling factor design that groups 8
# columns and 1/8 of the original rows to share a scaling factor, ensuring compatibility with
# the BCQ kernel".  In the OPTQ orientation of that section rows are outputs and columns are
# inputs, so (reading R24) plane i has one PoT scale per (row block
# b = n // (N/8), column group c = k // 8): the 8 weights of a key byte share it.
def _block_rows(N):
    if N % 8:
        raise ValueError("block-wise scales need 8 | N (1/8 of the rows per block)")
    return N // 8


def pack_blockwise(signs, alpha_bw):
    """signs int8 [q][N][K] (+-1), alpha_bw float32 [q][8][K/8] -> planes, exps_bw, n_clamped.

      1. sign fold per block (R3): alpha_i[b][c] < 0 negates s_i[n][k] for the rows n of
         block b and the 8 columns k of group c, and keeps |alpha_i[b][c]|;
      2. exponent: P = round(log2|alpha|) (pot_exponent: same zero / clamp rules);
      3. bits exactly as pack_canonical step 3 (R1, R2).
    Returns planes uint8 [q][N][K/8], exps_bw int8 [q][8][K/8], n_clamped.
    """
    s = np.asarray(signs)
    a = np.asarray(alpha_bw, dtype=np.float32)
    if s.ndim != 3:
        raise ValueError("signs must be [q][N][K]")
    q, n, k = s.shape
    nb = _block_rows(n)
    if k % 8:
        raise ValueError("need 8 | K")
    if a.shape != (q, 8, k // 8):
        raise ValueError("alpha_bw must be [q][8][K/8]")
    if not np.all((s == 1) | (s == -1)):
        raise ValueError("signs must be -1 or +1")
    exps, n_clamped = pot_exponent(a)
    flip = np.repeat(np.repeat(a < 0, nb, axis=1), 8, axis=2)   # [q][N][K]
    folded = np.where(flip, -s.astype(np.int16), s.astype(np.int16))
    bits = (folded == 1).astype(np.uint8).reshape(q, n, k // 8, 8)
    weights = (1 << np.arange(8, dtype=np.uint16)).astype(np.uint16)
    planes = (bits.astype(np.uint16) * weights).sum(axis=3).astype(np.uint8)
    return planes, exps, n_clamped


def dequant_blockwise(planes, exps_bw, K):
    """W_hat[n][k] = sum_i 2^{e_i[n // (N/8)][k // 8]} s_i[n][k], fp64."""
    p = np.asarray(planes, dtype=np.uint8)
    q, n, _ = p.shape
    nb = _block_rows(n)
    s = unpack_signs(p, K).astype(np.float64)                              # [q][N][K]
    scale = np.repeat(np.repeat(_pow2(exps_bw), nb, axis=1), 8, axis=2)    # [q][N][K]
    return (s * scale).sum(axis=0)


def gemm_blockwise(x, planes, exps_bw, row_chunk=2048):
    """y = x W_hat^T in fp64 with block-wise scales (the plain definition)."""
    xf = np.atleast_2d(np.asarray(x, dtype=np.float64))
    p = np.asarray(planes, dtype=np.uint8)
    q, n, kb = p.shape
    K = kb * 8
    nb = _block_rows(n)
    e = np.asarray(exps_bw)
    if xf.shape[1] != K or e.shape != (q, 8, kb):
        raise ValueError("x must be [M][K] and exps_bw [q][8][K/8]")
    y = np.empty((xf.shape[0], n), dtype=np.float64)
    rows = np.arange(n) // nb
    for n0 in range(0, n, row_chunk):
        n1 = min(n, n0 + row_chunk)
        s = unpack_signs(p[:, n0:n1], K).astype(np.float64)
        scale = np.repeat(_pow2(e)[:, rows[n0:n1], :], 8, axis=2)
        y[:, n0:n1] = xf @ (s * scale).sum(axis=0).T
    return y


def lut_gemm_blockwise(x, planes, exps_bw):
    """The LUT route with block-wise scales, step by step, fp64: one LUT per 8 activations
    (lut_direct), the key byte of plane i selects T_t[key], and since the
    8 weights of the key share one scale, that query is shifted by 2^{e_i[b][t]}
    before it is added."""
    xf = np.atleast_2d(np.asarray(x, dtype=np.float64))
    p = np.asarray(planes, dtype=np.uint8)
    q, n, kb = p.shape
    nb = _block_rows(n)
    sc = _pow2(exps_bw)                                       # [q][8][K/8]
    y = np.zeros((xf.shape[0], n), dtype=np.float64)
    t_idx = np.arange(kb)[None, :]
    rows = np.arange(n) // nb
    for m in range(xf.shape[0]):
        bank = np.stack([lut_direct(xf[m, 8 * t:8 * t + 8]) for t in range(kb)])   # [K/8][256]
        for i in range(q):
            queried = bank[t_idx, p[i].astype(np.int64)]                            # [N][K/8]
            y[m] += (queried * sc[i][rows]).sum(axis=1)
    return y


def blockwise_row_exps(exps_bw, N):
    """The block-wise exponents replicated into the row-wise layout with g = 8: [q][N][K/8]
    (SURVEY C6's "block-wise = g = 8 with exponents replicated over N/8-row blocks")."""
    return np.repeat(np.asarray(exps_bw), _block_rows(N), axis=1)


def algorithmic_bytes_blockwise(M, q, N, K):
    """HBM bytes of one block-wise GEMV call: planes + int8 exps [q][8][K/8] + fp16 x + y."""
    return q * N * K // 8 + q * K + 2 * M * K + 2 * M * N


def algorithmic_bytes_colwise(M, q, N, K):
    """HBM bytes of one column-wise GEMV call: planes + int8 exps [q][K] + fp16 x + fp16 y."""
    return q * N * K // 8 + q * K + 2 * M * K + 2 * M * N


# --------------------------------------------- NEXT-f2: additive PoT with K = 2 terms
# Eq. 2: alpha_k = POT(r_{k-1}), r_{k-1} = alpha - sum_{j<k} alpha_j,
# POT(a) = sign(a) 2^round(log2|a|), K terms "adopt a greedy strategy".  Readings R19-R20.
def additive_pot(alpha, K):
    """Greedy K-term PoT of one scalar (Python floats, exact): [(sign, P), ...] of length
    <= K (a zero residual ends the expansion early).  Term 1 uses pot_exponent's clamp."""
    terms = []
    r = float(np.float32(alpha))
    for k in range(K):
        if r == 0.0:
            break
        p = int(pot_exponent(np.float32(r))[0])
        sgn = 1 if r > 0 else -1
        terms.append((sgn, p))
        r = r - sgn * math.ldexp(1.0, p)
    return terms


def pack_apot2(signs, alpha, g):
    """K = 2 additive PoT pack: planes and exps exactly as pack_canonical (term 1, its sign
    folded into the bits), plus exps2 int8 [q][N][K/g]: the second term relative to the
    first, c2 = s1*s2*(P1 - P2), so a group's folded scale is 2^P1 (1 + sign(c2) 2^-|c2|).
    c2 = 0 (no second term) when alpha == 0, the residual is 0, P1 was clamped, or
    P2 < EXP_MIN or P1 - P2 > 127 (reading R19).  P2 <= P1 - 1 always (|r1| <= (sqrt2-1) 2^P1),
    and r1 = alpha - s1 2^P1 is exact in fp32 (Sterbenz), so c2 is a pure function of alpha.
    Returns planes, exps, exps2, n_clamped."""
    planes, exps, n_clamped = pack_canonical(signs, alpha, g)
    a = np.asarray(alpha, dtype=np.float32)
    e1 = exps.astype(np.int64)
    mag = np.abs(a.astype(np.float64))
    zero = mag == 0.0
    with np.errstate(divide="ignore"):
        p_raw = np.rint(np.log2(np.where(zero, 1.0, mag)))
    clamped = (~zero) & ((p_raw < EXP_MIN) | (p_raw > EXP_MAX))
    s1 = np.where(a < 0, -1.0, 1.0)
    r1 = a.astype(np.float64) - s1 * np.ldexp(1.0, np.where(zero, 0, e1))
    rz = (r1 == 0.0) | zero | clamped
    with np.errstate(divide="ignore"):
        p2 = np.rint(np.log2(np.where(rz, 1.0, np.abs(r1))))
    d = e1 - p2
    ok = (~rz) & (p2 >= EXP_MIN) & (d <= 127)
    sign = s1 * np.where(r1 < 0, -1.0, 1.0)
    exps2 = np.where(ok, sign * d, 0).astype(np.int8)
    return planes, exps, exps2, n_clamped


def dequant_apot2(planes, exps, exps2, g, K):
    """W_hat[n][k] = sum_i 2^{e_i} (1 + sign(c2) 2^{-|c2|}) s_i[n][k] (folded bits), fp64."""
    p = np.asarray(planes, dtype=np.uint8)
    e = np.asarray(exps, dtype=np.int8).astype(np.int64)
    c2 = np.asarray(exps2, dtype=np.int8).astype(np.int64)
    s = unpack_signs(p, K).astype(np.float64)
    one = np.where(e == EXP_ZERO, 0.0, np.ldexp(1.0, np.where(e == EXP_ZERO, 0, e)))
    two = np.where(c2 == 0, 0.0, np.sign(c2) * np.ldexp(one, -np.abs(c2)))
    return (s * np.repeat(one + two, g, axis=2)).sum(axis=0)


def gemm_apot2(x, planes, exps, exps2, g, row_chunk=2048):
    """y = x W_hat^T in fp64 with K = 2 additive PoT scales (the plain definition)."""
    xf = np.atleast_2d(np.asarray(x, dtype=np.float64))
    p = np.asarray(planes, dtype=np.uint8)
    q, n, kb = p.shape
    K = kb * 8
    y = np.empty((xf.shape[0], n), dtype=np.float64)
    for n0 in range(0, n, row_chunk):
        n1 = min(n, n0 + row_chunk)
        y[:, n0:n1] = xf @ dequant_apot2(p[:, n0:n1], exps[:, n0:n1], exps2[:, n0:n1], g, K).T
    return y


# ------------------------------------------- NEXT-f4: Alg. 1 alternating multi-bit BCQ
# greedy init (Eq. 1, Line 4), then T cycles of least-squares scale refit
# (Line 6) and binary-search code refit (Line 7); scales projected to PoT "during the
# alternating optimization cycles".  Per scale group (a row's g
# consecutive weights), fp64.  Readings R21-R23.
def pot_round_exact(a):
    """sign(a) 2^round(log2|a|) for an fp64 scalar, by exact rational comparison (no log):
    P = floor(log2|a|) + (|a|^2 >= 2^(2 floor + 1)).  0 -> 0."""
    a = float(a)
    if a == 0.0:
        return 0.0
    m, e = math.frexp(abs(a))            # |a| = m 2^e, m in [0.5, 1)
    p = e - 1                             # floor(log2|a|)
    if Fraction(abs(a)) ** 2 >= Fraction(2) ** (2 * p + 1):
        p += 1
    return math.copysign(math.ldexp(1.0, p), a)


def bcq_greedy(w, q):
    """Eq. 1 on one group vector w (fp64): r_0 = w; b_i = sign(r_{i-1}) (sign(0) = +1, R21),
    alpha_i = r_{i-1}^T b_i / n; r_i = r_{i-1} - alpha_i b_i.  Returns (alpha [q], B [q][n])."""
    r = np.asarray(w, dtype=np.float64).copy()
    n = r.size
    alpha = np.zeros(q)
    B = np.zeros((q, n))
    for i in range(q):
        b = np.where(r >= 0, 1.0, -1.0)
        alpha[i] = float(np.dot(r, b)) / n
        B[i] = b
        r = r - alpha[i] * b
    return alpha, B


def bcq_ls(B, w):
    """Line 6: alpha = (B^T B)^-1 B^T w with B = [b_1..b_q] as columns; the Gram matrix gets
    1e-8 * n on its diagonal (reading R22).  numpy.linalg.solve (LAPACK)."""
    B = np.asarray(B, dtype=np.float64)
    n = B.shape[1]
    G = B @ B.T + 1e-8 * n * np.eye(B.shape[0])
    return np.linalg.solve(G, B @ np.asarray(w, dtype=np.float64))


def bcq_bs_codes(alpha, w):
    """Line 7: each w_j takes the representable level sum_i c_i alpha_i (c in {-1,1}^q)
    nearest to it; ties -> smaller |level|, then the negative level (R23).
    Exhaustive over the 2^q levels (the binary search of the paper finds the same level).
    Returns B [q][n]."""
    a = np.asarray(alpha, dtype=np.float64)
    q = a.size
    codes = np.array([[1.0 if (c >> i) & 1 else -1.0 for i in range(q)] for c in range(1 << q)])  # [2^q][q]
    levels = codes @ a
    wv = np.asarray(w, dtype=np.float64)
    dist = np.abs(wv[:, None] - levels[None, :])                    # [n][2^q]
    key = np.stack([dist, np.abs(levels)[None, :].repeat(wv.size, 0), levels[None, :].repeat(wv.size, 0)])
    # lexicographic argmin over (distance, |level|, level)
    order = np.lexsort((key[2], key[1], key[0]), axis=1)
    best = order[:, 0]
    return codes[best].T.copy()


def bcq_quantize(w, q, g, T, pot=False):
    """Alg. 1 per scale group of a weight matrix w [N][K] (groups: g consecutive k of a row).

    For each group: greedy (Eq. 1); then T times: LS (Line 6), optional PoT projection of
    every alpha_i (pot_round_exact, Eq. 2 with K = 1), BS (Line 7).  Returns signs int8
    [q][N][K] and alpha fp64 [q][N][K/g] (the codes are BS of the returned alphas when T >= 1,
    the greedy codes when T == 0)."""
    W = np.asarray(w, dtype=np.float64)
    N, K = W.shape
    if K % g:
        raise ValueError("g must divide K")
    signs = np.empty((q, N, K), dtype=np.int8)
    alphas = np.empty((q, N, K // g))
    for n in range(N):
        for G in range(K // g):
            wg = W[n, G * g:(G + 1) * g]
            alpha, B = bcq_greedy(wg, q)
            for _ in range(T):
                alpha = bcq_ls(B, wg)
                if pot:
                    alpha = np.array([pot_round_exact(v) for v in alpha])
                B = bcq_bs_codes(alpha, wg)
            signs[:, n, G * g:(G + 1) * g] = B.astype(np.int8)
            alphas[:, n, G] = alpha
    return signs, alphas


# ----------------------------------------------------------------------- output + metrics
def to_fp16(y):
    """fp16 round-to-nearest-even of an fp64 result (PAPER.md:186 'in FP16 format'; R11)."""
    return np.asarray(y, dtype=np.float64).astype(np.float16)


def err_floor(y_test, y_ref):
    """Per batch row m: max_n |y_test - y_ref| / max(|y_ref|, rms_n(y_ref[m])) (reading R10).

    Returns the max over rows.  The 2e-3 bar of BASELINE.json north_star applies to this.
    """
    yt = np.atleast_2d(np.asarray(y_test, dtype=np.float64))
    yr = np.atleast_2d(np.asarray(y_ref, dtype=np.float64))
    rms = np.sqrt(np.mean(yr * yr, axis=1, keepdims=True))
    den = np.maximum(np.abs(yr), rms)
    den = np.where(den == 0.0, 1.0, den)
    return float(np.max(np.abs(yt - yr) / den)) if yr.size else 0.0


def err_normwise(y_test, y_ref):
    """max |y_test - y_ref| / ||y_ref||_inf (reported beside err_floor)."""
    yt = np.asarray(y_test, dtype=np.float64)
    yr = np.asarray(y_ref, dtype=np.float64)
    den = np.max(np.abs(yr)) if yr.size else 1.0
    return float(np.max(np.abs(yt - yr)) / (den if den else 1.0)) if yr.size else 0.0


# ----------------------------------------------------------------------- byte accounting
def packed_bytes(q, N, K, g):
    """Canonical packed bytes of one layer: planes q*N*K/8 + int8 exps q*N*K/g."""
    return q * N * K // 8, q * N * (K // g)


def algorithmic_bytes(M, q, N, K, g):
    """HBM bytes one GEMV call must move (§8(d)): planes + exps + fp16 x + fp16 y."""
    planes, exps = packed_bytes(q, N, K, g)
    return planes + exps + 2 * M * K + 2 * M * N
