"""CPU pins of the fp64 oracle (DESIGN.md §Oracle pins S1-S8).

Each pin checks the oracle against something other than itself: the paper's printed
numbers, SPEC worked values derived from Eq. 2, closed forms, exact rational arithmetic,
exhaustive enumeration, or algebraic invariants -- chosen so that a dropped term, a wrong
sign or bit index, or a transposed operand fails at least one of them.
"""

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rng(seed=0):
    return np.random.default_rng(seed)


def _rand_fp16(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float16)


def _frac(v):
    return Fraction(float(v))


# ------------------------------------------------------------------------- S1: the LUT
@pytest.mark.parametrize("case", ["random", "onehot", "zero", "extreme", "tiny"])
def test_s1_lut_exhaustive_256_keys(case):
    """256 signed partial sums per 8 activations.  Direct, incremental
     and an exact-rational brute force agree on every key."""
    rng = _rng(1)
    if case == "random":
        x8 = _rand_fp16(rng, 8)
    elif case == "onehot":
        x8 = np.zeros(8, np.float16)
        x8[0] = 1.0
    elif case == "zero":
        x8 = np.zeros(8, np.float16)
    elif case == "extreme":
        x8 = np.array([65504, -65504, 6.1e-5, -2.0 ** -24, 1024, -3.5, 0.0, 2.0 ** -14], np.float16)
    else:
        x8 = np.array([2.0 ** -24] * 8, np.float16)
    d = oracle.lut_direct(x8)
    inc = oracle.lut_incremental(x8)
    xs = [_frac(v) for v in x8]
    for key in range(256):
        exact = sum((xs[b] if (key >> b) & 1 else -xs[b]) for b in range(8))
        assert Fraction(float(d[key])) == exact
        assert Fraction(float(inc[key])) == exact
    if case == "onehot":  # T[key] = +1 if bit0 else -1
        assert all(d[k] == (1.0 if k & 1 else -1.0) for k in range(256))
    if case == "zero":
        assert np.all(d == 0.0)
    # complement symmetry: T[~key] = -T[key]
    assert np.all(d[::-1] == -d)


# ------------------------------------------------------------------------ S5: pack (a1)
def test_s5_pot_round_spec_values():
    gold = _gold("pot_round_spec.json")
    for case in gold["pot_round"]:
        e, nclamp = oracle.pot_exponent(np.array([case["alpha"]], np.float32))
        assert int(e[0]) == case["P"] and nclamp == 0
    # the sign lives in the bits after the sign fold: alpha = -0.25 flips every sign
    s = np.ones((1, 1, 8), np.int8)
    planes, exps, _ = oracle.pack_canonical(s, np.array([[[-0.25]]], np.float32), 8)
    assert planes[0, 0, 0] == 0x00 and exps[0, 0, 0] == -2
    planes, exps, _ = oracle.pack_canonical(s, np.array([[[4.0]]], np.float32), 8)
    assert planes[0, 0, 0] == 0xFF and exps[0, 0, 0] == 2


def _pot_bracket(alpha, P):
    """Exact rational check that P = round(log2|alpha|): 2^(2P-1) <= alpha^2 < 2^(2P+1)."""
    a2 = Fraction(float(np.float32(alpha))) ** 2
    return Fraction(2) ** (2 * P - 1) <= a2 < Fraction(2) ** (2 * P + 1)


def test_s5_pot_exact_rational_bracket():
    """P = round(log2|a|)  <=>  2^(2P-1) <= a^2 < 2^(2P+1), checked in exact rationals
    (no log2) on random fp32 scales spanning many binades, and at the sqrt(2) boundary."""
    rng = _rng(2)
    a = (np.exp2(rng.uniform(-40, 40, 20000)) * rng.choice([-1, 1], 20000)).astype(np.float32)
    # the two fp32 neighbours of every 2^(k+1/2) boundary
    b = []
    for k in range(-30, 30):
        m = np.float32(2.0 ** (k + 0.5))
        b += [np.nextafter(m, np.float32(0)), m, np.nextafter(m, np.float32(np.inf))]
    a = np.concatenate([a, np.array(b, np.float32)])
    e, nclamp = oracle.pot_exponent(a)
    assert nclamp == 0
    for v, p in zip(a.tolist(), e.tolist()):
        assert _pot_bracket(v, p), (v, p)


def test_s5_pot_edge_cases():
    e, n = oracle.pot_exponent(np.array([0.0, -0.0], np.float32))
    assert list(e) == [oracle.EXP_ZERO, oracle.EXP_ZERO] and n == 0
    sub = np.float32(1e-42)  # subnormal -> P ~ -139 -> clamp to -100
    e, n = oracle.pot_exponent(np.array([sub, 2.0 ** 101, 2.0 ** -101, 2.0 ** 100, 2.0 ** -100], np.float32))
    assert list(e) == [-100, 100, -100, 100, -100] and n == 3
    for bad in (np.nan, np.inf, -np.inf):
        with pytest.raises(ValueError):
            oracle.pot_exponent(np.array([bad], np.float32))


@pytest.mark.parametrize("K", [8, 24, 64])
def test_s5_bit_order_single_positive(K):
    """LSB = lowest k of the 8 grouped weights, 1 <-> +1."""
    for j in range(K):
        s = -np.ones((1, 1, K), np.int8)
        s[0, 0, j] = 1
        planes, _, _ = oracle.pack_canonical(s, np.ones((1, 1, K // 8), np.float32), 8)
        expect = np.zeros(K // 8, np.uint8)
        expect[j >> 3] = 1 << (j & 7)
        assert np.array_equal(planes[0, 0], expect)
        assert np.array_equal(oracle.unpack_signs(planes, K)[0, 0], s[0, 0])


def test_s5_sign_fold_identity():
    """alpha*b == (-alpha)*(-b): dequant of the packed layer equals sum_i POT(alpha_i) b_i
    computed directly from the unpacked inputs with exact rationals (tiny shape)."""
    rng = _rng(3)
    q, N, K, g = 2, 3, 16, 8
    s = rng.choice([-1, 1], (q, N, K)).astype(np.int8)
    a = (rng.standard_normal((q, N, K // g)) * 0.1).astype(np.float32)
    planes, exps, _ = oracle.pack_canonical(s, a, g)
    w = oracle.dequant(planes, exps, g, K)
    for n in range(N):
        for k in range(K):
            exact = Fraction(0)
            for i in range(q):
                al = float(a[i, n, k // g])
                P = round(math.log2(abs(al)))
                exact += (1 if al > 0 else -1) * Fraction(2) ** P * int(s[i, n, k])
            assert Fraction(float(w[n, k])) == exact


# ------------------------------------------------------------- S2: brute force, tiny K
def _exact_y(x, s, e, g):
    """Exact rational y for one row from unpacked signs s[q][K] and exponents e[q][K/g]."""
    acc = Fraction(0)
    for i in range(s.shape[0]):
        for k in range(s.shape[1]):
            ei = int(e[i][k // g])
            if ei == oracle.EXP_ZERO:
                continue
            acc += int(s[i][k]) * Fraction(2) ** ei * _frac(x[k])
    return acc


@pytest.mark.parametrize("q,K", [(1, 8), (2, 8), (1, 16)])
def test_s2_bruteforce_every_sign_pattern(q, K):
    """Every one of the 2^(qK) sign patterns of one output row: gemm == lut_gemm == exact."""
    rng = _rng(4)
    g = 8
    x = _rand_fp16(rng, (1, K))
    e = rng.integers(-3, 4, (q, 1, K // g)).astype(np.int8)
    npat = 1 << (q * K)
    pats = ((np.arange(npat)[:, None] >> np.arange(q * K)[None, :]) & 1).astype(np.int8)
    signs = np.where(pats == 1, 1, -1).astype(np.int8).reshape(npat, q, K).transpose(1, 0, 2)
    alpha = np.repeat(np.ldexp(1.0, e.astype(np.int64)).astype(np.float32), npat, axis=1)
    planes, exps, _ = oracle.pack_canonical(signs, alpha, g)
    y1 = oracle.gemm(x, planes, exps, g)[0]
    y2 = oracle.lut_gemm(x, planes, exps, g)[0]
    assert np.array_equal(y1, y2)
    for p in range(0, npat, max(1, npat // 512)):   # exact rationals on a spread sample
        assert Fraction(float(y1[p])) == _exact_y(x[0], signs[:, p], exps[:, p], g)


# --------------------------------------------------------------------- S3/S4 closed forms
def test_s3_all_ones_closed_form_and_exponent_shift():
    rng = _rng(5)
    q, N, K, g = 3, 5, 256, 128
    x = _rand_fp16(rng, (2, K))
    e = rng.integers(-8, 9, (q, N, K // g)).astype(np.int8)
    planes = np.full((q, N, K // 8), 0xFF, np.uint8)
    y = oracle.gemm(x, planes, e, g)
    for m in range(2):
        for n in range(N):
            exact = Fraction(0)
            for G in range(K // g):
                sx = sum(_frac(v) for v in x[m, G * g:(G + 1) * g])
                exact += sum(Fraction(2) ** int(e[i, n, G]) for i in range(q)) * sx
            assert Fraction(float(y[m, n])) == exact
    for d in (-5, 1, 7):
        y_d = oracle.gemm(x, planes, (e + d).astype(np.int8), g)
        assert np.array_equal(y_d, np.ldexp(y, d))


def test_s3_flip_plane_group_negates_its_term():
    rng = _rng(6)
    q, N, K, g = 2, 4, 256, 128
    s = rng.choice([-1, 1], (q, N, K)).astype(np.int8)
    a = np.ldexp(1.0, rng.integers(-6, 0, (q, N, K // g))).astype(np.float32)
    planes, exps, _ = oracle.pack_canonical(s, a, g)
    x = _rand_fp16(rng, (1, K))
    y = oracle.gemm(x, planes, exps, g)[0]
    i, G = 1, 1
    flipped = planes.copy()
    flipped[i, :, G * g // 8:(G + 1) * g // 8] ^= 0xFF
    y_f = oracle.gemm(x, flipped, exps, g)[0]
    for n in range(N):
        term = sum(int(s[i, n, k]) * _frac(x[0, k]) for k in range(G * g, (G + 1) * g))
        term *= Fraction(float(a[i, n, G]))
        assert Fraction(float(y_f[n])) == Fraction(float(y[n])) - 2 * term


@pytest.mark.parametrize("e", [-7, 0, 3])
def test_s4_q1_all_ones_is_scaled_sum(e):
    """north_star invariant: q = 1, all-ones B, alpha = 2^e  ->  y = 2^e * sum(x)."""
    rng = _rng(7)
    K = 768
    x = _rand_fp16(rng, (3, K))
    signs = np.ones((1, 4, K), np.int8)
    planes, exps, _ = oracle.pack_canonical(signs, np.full((1, 4, K // 128), 2.0 ** e, np.float32), 128)
    y = oracle.gemm(x, planes, exps, 128)
    for m in range(3):
        exact = Fraction(2) ** e * sum(_frac(v) for v in x[m])
        assert all(Fraction(float(v)) == exact for v in y[m])
    ys = oracle.gemm_scalar(x[:1], planes, exps, 128)
    assert np.allclose(ys, y[:1], rtol=1e-12, atol=0)


# ------------------------------------------------------------ S6: formula-defined weights
def _formula_layer(q, N, K, g):
    """Weights defined by a formula so column j of W_hat is known without the oracle:
    s_i[n][k] = +1 iff (3n + 5k + 7i) mod 4 < 2;  alpha_i[n][G] = 2^-(i + (n + G) mod 3)."""
    n = np.arange(N)[:, None]
    k = np.arange(K)[None, :]
    s = np.stack([np.where((3 * n + 5 * k + 7 * i) % 4 < 2, 1, -1) for i in range(q)]).astype(np.int8)
    G = np.arange(K // g)[None, :]
    a = np.stack([np.ldexp(1.0, -(i + (n + G) % 3)) for i in range(q)]).astype(np.float32)
    return s, a


def _formula_w(q, n, k, g):
    return sum((1 if (3 * n + 5 * k + 7 * i) % 4 < 2 else -1) * Fraction(2) ** -(i + (n + k // g) % 3)
               for i in range(q))


def test_s6_basis_vectors_select_columns_not_rows():
    """x = e_j -> y[n] = W_hat[n][j]: with N != K this fails for a transposed operand."""
    q, N, K, g = 3, 40, 256, 128
    s, a = _formula_layer(q, N, K, g)
    planes, exps, _ = oracle.pack_canonical(s, a, g)
    for j in (0, 1, 7, 8, 127, 128, 255):
        x = np.zeros((1, K), np.float16)
        x[0, j] = 1.0
        y = oracle.gemm(x, planes, exps, g)[0]
        assert all(Fraction(float(y[n])) == _formula_w(q, n, j, g) for n in range(N))


def test_s6_linearity_and_odd_symmetry():
    rng = _rng(8)
    q, N, K, g = 2, 64, 512, 128
    s, a = _formula_layer(q, N, K, g)
    planes, exps, _ = oracle.pack_canonical(s, a, g)
    x1 = _rand_fp16(rng, (1, K))
    x2 = _rand_fp16(rng, (1, K))
    y1 = oracle.gemm(x1, planes, exps, g)
    assert np.array_equal(oracle.gemm(-x1, planes, exps, g), -y1)
    y12 = oracle.gemm(x1.astype(np.float64) + x2.astype(np.float64), planes, exps, g)
    assert np.allclose(y12, y1 + oracle.gemm(x2, planes, exps, g), rtol=0, atol=1e-12)


def test_gemm_matches_scalar_and_lut_routes_on_synthetic_layer():
    q, N, K, g = 3, 24, 512, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(0))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    x = synth.gen_x(2, K, seed=synth.seed_for(0, 1)).numpy()
    y = oracle.gemm(x, planes, exps, g)
    assert np.allclose(oracle.lut_gemm(x, planes, exps, g), y, rtol=1e-13, atol=1e-15)
    assert np.allclose(oracle.gemm_scalar(x, planes, exps, g), y, rtol=1e-13, atol=1e-15)


@pytest.mark.slow
def test_config0_scalar_loop_agrees():
    """Config 0 (OPT-125M q_proj 768x768, 3-bit, g=128): the pure-Python loop (the
    'CPU oracle in seconds' case) equals the numpy route."""
    q, N, K, g = 3, 768, 768, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(0))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    x = synth.gen_x(1, K, seed=synth.seed_for(0, 1)).numpy()
    y = oracle.gemm(x, planes, exps, g)
    ys = oracle.gemm_scalar(x, planes, exps, g)
    assert np.allclose(ys, y, rtol=1e-12, atol=1e-14)


# ------------------------------------------------------------------ tiled layout (a1 opt.)
def test_tiled_layout_definition_and_roundtrip():
    rng = _rng(9)
    for q, N, K, g in [(3, 40, 512, 128), (2, 16, 256, 256), (1, 33, 768, 768)]:
        planes = rng.integers(0, 256, (q, N, K // 8)).astype(np.uint8)
        exps = rng.integers(-100, 101, (q, N, K // g)).astype(np.int8)
        pt, et = oracle.to_tiled(planes, exps, g)
        assert (pt.size, et.size) == oracle.tiled_sizes(q, N, K)
        RG = -(-N // 16)
        # walk the definition independently for random positions
        for _ in range(300):
            s, rg, i = rng.integers(K // 256), rng.integers(RG), rng.integers(q)
            r, h, j = rng.integers(16), rng.integers(2), rng.integers(16)
            n = 16 * rg + r
            off = ((s * RG + rg) * q + i) * 512 + r * 32 + h * 16 + j
            want = planes[i, n, 32 * s + 16 * h + (j + r) % 16] if n < N else 0
            assert pt[off] == want
            eoff = ((s * RG + rg) * q + i) * 32 + r * 2 + h
            ewant = exps[i, n, (256 * s + 128 * h) // g] if n < N else oracle.EXP_ZERO
            assert et[eoff] == ewant
        p2, e2 = oracle.from_tiled(pt, et, q, N, K, g)
        assert np.array_equal(p2, planes) and np.array_equal(e2, exps)


def test_tiled_rotation_gives_distinct_groups_per_step():
    """The layout's purpose: at every step j the 32 lanes (16 rows x 2 halves) of a warp
    read 32 *different* groups t = 16h + (j + r) mod 16 of the 256-k slice."""
    for j in range(16):
        groups = {16 * h + (j + r) % 16 for r in range(16) for h in range(2)}
        assert len(groups) == 32


# ----------------------------------------------------------- S7: byte accounting vs paper
def test_s7_memory_accounting_matches_paper():
    gold = _gold("paper_memory.json")
    tol = gold["tolerance_gib"]
    for name, m in gold["models"].items():
        H, F, L, kv = m["hidden"], m["ffn"], m["layers"], m["kv_dim"]
        shapes = [(H, H), (kv, H), (kv, H), (H, H)]
        shapes += [(F, H), (F, H), (H, F)] if m.get("gated_mlp") else [(F, H), (H, F)]
        emb = m["emb_copies"] * m["vocab"] * H * 2
        for bits, printed in m["printed_gb"].items():
            b = int(bits)
            if b == 16:
                lin = sum(N * K * 2 for N, K in shapes)
            else:
                lin = sum(oracle.packed_bytes(b, N, K, K)[0] for N, K in shapes)
            gib = (L * lin + emb) / 2 ** 30
            assert abs(gib - printed) <= tol, (name, bits, gib, printed)


def test_algorithmic_bytes_config_table():
    """221,184 + 13,824 + 1,536 + 1,536 = 238,080 bytes."""
    assert oracle.algorithmic_bytes(1, 3, 768, 768, 128) == 238080
    assert oracle.packed_bytes(3, 28672, 8192, 128) == (88080384, 5505024)


# ------------------------------------------------------------------------ metric sanity
def test_err_floor_metric():
    y = np.array([[1.0, -2.0, 0.0, 1e-9]])
    assert oracle.err_floor(y, y) == 0.0
    rms = math.sqrt((1 + 4 + 1e-18) / 4)
    yb = y.copy()
    yb[0, 3] += 1e-3
    assert math.isclose(oracle.err_floor(yb, y), 1e-3 / rms, rel_tol=1e-9)
    assert oracle.err_floor(np.zeros((1, 3)), np.zeros((1, 3))) == 0.0


def test_fp16_output_rounding_is_rne():
    # 2049 is a tie between 2048 and 2050 in fp16 -> even mantissa 2048; 2051 -> 2052
    assert oracle.to_fp16(np.array([2049.0, 2051.0, 1e6])).tolist() == [2048.0, 2052.0, float("inf")]


# --------------------------------------- S9: column-wise scales (NEXT-f1, "Ours (Acc.)")
def test_s9_colwise_exact_pot_scales_reproduce_bcq_sum():
    """alpha_i[k] = +-2^P exactly: dequant_colwise(pack_colwise(s, alpha)) = sum_i alpha_i[k]
    s_i[n][k] element by element (Eq. 2 with K = 1 is exact on powers of two).  Pins the
    per-column sign fold (a row-wise fold or a flipped polarity fails) and the bit order."""
    rng = _rng(90)
    q, N, K = 3, 5, 24
    s = rng.choice([-1, 1], size=(q, N, K)).astype(np.int8)
    P = rng.integers(-6, 7, size=(q, K))
    sign = rng.choice([-1.0, 1.0], size=(q, K))
    alpha = (sign * np.ldexp(1.0, P)).astype(np.float32)
    planes, exps, ncl = oracle.pack_colwise(s, alpha)
    assert ncl == 0 and exps.shape == (q, K) and np.array_equal(exps, P.astype(np.int8))
    want = np.zeros((N, K))
    for i in range(q):
        for n in range(N):
            for k in range(K):
                want[n, k] += float(alpha[i, k]) * int(s[i, n, k])
    assert np.array_equal(oracle.dequant_colwise(planes, exps, K), want)


def test_s9_colwise_constant_exponents_reduce_to_rowwise_gemm():
    """If every column of plane i has the same exponent c_i, column-wise and row-wise
    (g = K) scales are the same weight: gemm_colwise must equal the pinned row-wise gemm."""
    rng = _rng(91)
    q, N, K = 3, 40, 256
    planes = rng.integers(0, 256, size=(q, N, K // 8), dtype=np.uint8)
    c = np.array([3, -2, 0], dtype=np.int8)
    e_col = np.repeat(c[:, None], K, axis=1)
    e_row = np.repeat(c[:, None, None], N, axis=1)                  # [q][N][1], g = K
    x = _rand_fp16(rng, (2, K))
    assert np.array_equal(oracle.gemm_colwise(x, planes, e_col), oracle.gemm(x, planes, e_row, K))


def test_s9_colwise_all_ones_closed_form():
    """All-ones planes: y[n] = sum_k x[k] * sum_i 2^{e_i[k]} for every row, exact rationals."""
    rng = _rng(92)
    q, N, K = 2, 3, 32
    planes = np.full((q, N, K // 8), 0xFF, dtype=np.uint8)
    e = rng.integers(-5, 6, size=(q, K)).astype(np.int8)
    e[1, 7] = oracle.EXP_ZERO
    x = _rand_fp16(rng, (1, K))
    want = Fraction(0)
    for k in range(K):
        col = sum((Fraction(2) ** int(e[i, k]) for i in range(q) if e[i, k] != oracle.EXP_ZERO), Fraction(0))
        want += _frac(x[0, k]) * col
    y = oracle.gemm_colwise(x, planes, e)
    assert np.all(y == float(want))


def test_s9_colwise_column_scaling_equals_exponent_shift_on_that_column():
    """Scaling x[k] by 2^d equals adding d to e_i[k] for every plane (exact in fp64).  With
    N != K a scale applied per row instead of per column fails; a dropped plane fails too."""
    rng = _rng(93)
    q, N, K = 3, 24, 64
    planes = rng.integers(0, 256, size=(q, N, K // 8), dtype=np.uint8)
    e = rng.integers(-4, 5, size=(q, K)).astype(np.int8)
    x = _rand_fp16(rng, (1, K)).astype(np.float64)
    for k, d in [(0, 3), (17, -2), (63, 5)]:
        x2 = x.copy()
        x2[0, k] = np.ldexp(x2[0, k], d)
        e2 = e.copy()
        e2[:, k] += d
        assert np.array_equal(oracle.gemm_colwise(x2, planes, e), oracle.gemm_colwise(x, planes, e2))
    # and it is not a row-wise scale: shifting e of column 0 changes rows by column-0 terms
    e3 = e.copy()
    e3[:, 0] += 1
    diff = oracle.gemm_colwise(x, planes, e3) - oracle.gemm_colwise(x, planes, e)
    s0 = oracle.unpack_signs(planes, K)[:, :, 0].astype(np.float64)          # [q][N]
    want = x[0, 0] * (s0 * np.ldexp(1.0, e[:, 0].astype(np.int64))[:, None]).sum(axis=0)
    assert np.allclose(diff[0], want, rtol=0, atol=1e-12)


def test_s9_colwise_lut_route_matches_definition():
    rng = _rng(94)
    q, N, K = 3, 33, 512
    s, a = synth.gen_layer_colwise(q, N, K, seed=5)
    planes, e, _ = oracle.pack_colwise(s.numpy(), a.numpy())
    x = synth.gen_x(2, K, seed=6).numpy()
    y0 = oracle.gemm_colwise(x, planes, e)
    y1 = oracle.lut_gemm_colwise(x, planes, e)
    assert oracle.err_floor(y1, y0) < 1e-12


def test_s9_tile_planes_matches_to_tiled():
    rng = _rng(95)
    planes = rng.integers(0, 256, size=(2, 40, 64), dtype=np.uint8)
    exps = np.zeros((2, 40, 4), dtype=np.int8)
    assert np.array_equal(oracle.tile_planes(planes), oracle.to_tiled(planes, exps, 128)[0])


# ---------------------------------------------- S10: additive PoT, K = 2 terms (NEXT-f2)
def test_s10_additive_pot_spec_examples():
    for c in _gold("apot_spec.json")["cases"]:
        terms = oracle.additive_pot(c["alpha"], c["K"])
        assert [list(t) for t in terms] == c["terms"], c["cite"]
        val = sum(sg * 2.0 ** p for sg, p in terms)
        assert c["alpha"] - val == c["residual"], c["cite"]


def test_s10_residual_non_increasing_and_k2_no_worse_than_k1():
    """residual magnitude non-increasing per term; the K-term error <= 1-term."""
    rng = _rng(100)
    for a in rng.standard_normal(2000) * 10.0 ** rng.uniform(-6, 3, 2000):
        a = float(np.float32(a))
        prev = abs(a)
        val = 0.0
        for sg, p in oracle.additive_pot(a, 3):
            val += sg * 2.0 ** p
            assert abs(a - val) <= prev
            prev = abs(a - val)


def test_s10_exact_two_term_scales_are_reproduced():
    """alpha = +-(2^A + sigma 2^B), A - B >= 2: round(log2|alpha|) = A, the residual is exactly
    sigma 2^B, so W_hat = alpha * s exactly (element by element, against alpha itself)."""
    rng = _rng(101)
    q, N, K, g = 2, 4, 64, 16
    A = rng.integers(-8, 4, size=(q, N, K // g))
    B = A - rng.integers(2, 9, size=A.shape)
    sig = rng.choice([-1.0, 1.0], size=A.shape)
    sgn = rng.choice([-1.0, 1.0], size=A.shape)
    alpha = (sgn * (np.ldexp(1.0, A) + sig * np.ldexp(1.0, B))).astype(np.float32)
    assert np.array_equal(alpha.astype(np.float64), sgn * (np.ldexp(1.0, A) + sig * np.ldexp(1.0, B)))
    s = rng.choice([-1, 1], size=(q, N, K)).astype(np.int8)
    planes, e1, c2, ncl = oracle.pack_apot2(s, alpha, g)
    assert ncl == 0 and np.array_equal(e1, A.astype(np.int8))
    assert np.array_equal(np.abs(c2.astype(np.int64)), A - B)
    want = (s.astype(np.float64) * np.repeat(alpha.astype(np.float64), g, axis=2)).sum(axis=0)
    assert np.array_equal(oracle.dequant_apot2(planes, e1, c2, g, K), want)


def test_s10_vectorised_pack_matches_scalar_greedy():
    """The vectorised c2 of pack_apot2 equals the scalar greedy of additive_pot (K = 2) on
    random alphas, including tiny, huge (clamped) and zero ones."""
    rng = _rng(102)
    a = (rng.standard_normal(4000) * 10.0 ** rng.uniform(-8, 4, 4000)).astype(np.float32)
    a[:5] = [0.0, 3.0, -3.0, 2.0 ** -140, 2.0 ** 120]
    s = np.ones((1, 1, 8 * a.size), dtype=np.int8)
    _, e1, c2, _ = oracle.pack_apot2(s, a.reshape(1, 1, -1), 8)
    for k, av in enumerate(a):
        terms = oracle.additive_pot(float(av), 2)
        p_raw = math.log2(abs(float(av))) if av != 0 else 0.0
        if av == 0 or round(p_raw) < oracle.EXP_MIN or round(p_raw) > oracle.EXP_MAX or len(terms) < 2:
            assert c2[0, 0, k] == 0, (k, av)
            continue
        (s1, p1), (s2, p2) = terms
        if p2 < oracle.EXP_MIN or p1 - p2 > 127:
            assert c2[0, 0, k] == 0
            continue
        assert e1[0, 0, k] == p1 and c2[0, 0, k] == s1 * s2 * (p1 - p2), (k, av, terms, c2[0, 0, k])


def test_s10_zero_second_terms_reduce_to_gemm():
    rng = _rng(103)
    q, N, K, g = 3, 20, 256, 128
    planes = rng.integers(0, 256, size=(q, N, K // 8), dtype=np.uint8)
    e = rng.integers(-6, 6, size=(q, N, K // g)).astype(np.int8)
    x = _rand_fp16(rng, (2, K))
    assert np.array_equal(oracle.gemm_apot2(x, planes, e, np.zeros_like(e), g), oracle.gemm(x, planes, e, g))


# ------------------------------------ S11: Alg. 1 alternating BCQ quantiser (NEXT-f4)
def test_s11_spec_worked_values():
    """SPEC.md:107-110 (1-bit analytic), :117-118 (greedy q=2), :134-136 (BS examples)."""
    a, B = oracle.bcq_greedy([1.0, 2.0, -3.0, 0.5], 1)
    assert a[0] == 1.625 and list(B[0]) == [1, 1, -1, 1]
    a, B = oracle.bcq_greedy([1.0, 2.0, -3.0, 0.5], 2)
    assert a[0] == 1.625 and a[1] == 0.875
    r = np.array([1.0, 2.0, -3.0, 0.5]) - 1.625 * B[0]
    assert list(r) == [-0.625, 0.375, -1.375, -1.125] and list(B[1]) == list(np.where(r >= 0, 1, -1))
    codes = oracle.bcq_bs_codes([1.0, 0.5], [0.7, 1.0])
    assert list(codes[:, 0]) == [1, -1]                    # 0.7 -> level +0.5
    assert list(codes[:, 1]) == [1, -1]                    # tie 0.5 / 1.5 -> smaller |level|
    assert list(oracle.bcq_bs_codes([2.0], [0.3])[:, 0]) == [1]


def test_s11_one_bit_is_the_brute_force_optimum():
    """q = 1: b = sign(w), alpha = w^T b / n minimises ||w - alpha b||^2 over all 2^n sign
    patterns (each with its own optimal alpha)."""
    rng = _rng(110)
    for _ in range(20):
        n = int(rng.integers(2, 11))
        w = rng.standard_normal(n)
        a, B = oracle.bcq_greedy(w, 1)
        got = float(np.sum((w - a[0] * B[0]) ** 2))
        best = min(float(np.sum((w - (w @ b) / n * b) ** 2))
                   for c in range(1 << n) for b in [np.array([1.0 if (c >> j) & 1 else -1.0 for j in range(n)])])
        assert got <= best + 1e-12


def test_s11_ls_solves_the_normal_equations_exactly():
    """Against an exact rational solve of (B^T B + 1e-8 n I) alpha = B^T w (q = 2, 3)."""
    rng = _rng(111)
    for q in (2, 3):
        n = 24
        w = rng.standard_normal(n)
        _, B = oracle.bcq_greedy(w, q)
        a = oracle.bcq_ls(B, w)
        G = [[sum(Fraction(int(B[i, j]) * int(B[k, j])) for j in range(n)) + (Fraction(1e-8) * n if i == k else 0)
              for k in range(q)] for i in range(q)]
        rhs = [sum(Fraction(float(w[j])) * int(B[i, j]) for j in range(n)) for i in range(q)]
        # Gauss-Jordan in rationals
        M = [row[:] + [rhs[i]] for i, row in enumerate(G)]
        for c in range(q):
            piv = next(r for r in range(c, q) if M[r][c] != 0)
            M[c], M[piv] = M[piv], M[c]
            M[c] = [v / M[c][c] for v in M[c]]
            for r in range(q):
                if r != c and M[r][c] != 0:
                    M[r] = [vr - M[r][c] * vc for vr, vc in zip(M[r], M[c])]
        exact = np.array([float(M[i][q]) for i in range(q)])
        assert np.allclose(a, exact, rtol=1e-12, atol=1e-15)


def test_s11_bs_picks_the_nearest_level_by_enumeration():
    rng = _rng(112)
    for q in (1, 2, 3, 4):
        alpha = np.sort(rng.uniform(0.05, 1.0, q))[::-1]
        w = rng.standard_normal(300)
        codes = oracle.bcq_bs_codes(alpha, w)
        lv = alpha @ codes
        for j in range(w.size):
            best = None
            for c in range(1 << q):
                level = sum(alpha[i] * (1 if (c >> i) & 1 else -1) for i in range(q))
                k = (abs(w[j] - level), abs(level), level)
                best = k if best is None or k < best else best
            assert abs(w[j] - lv[j]) == best[0] and lv[j] == best[2]


def test_s11_alternating_is_monotone_and_recovers_representable_weights():
    rng = _rng(113)
    for trial in range(30):
        w = rng.standard_normal(64)
        alpha, B = oracle.bcq_greedy(w, 3)
        prev = float(np.sum((w - alpha @ B) ** 2))
        for _ in range(10):
            alpha = oracle.bcq_ls(B, w)
            B = oracle.bcq_bs_codes(alpha, w)
            cur = float(np.sum((w - alpha @ B) ** 2))
            assert cur <= prev + 1e-9
            prev = cur
    # w drawn from the level set of alpha = (1, 0.5): exactly representable at q = 2
    lv = np.array([-1.5, -0.5, 0.5, 1.5])
    w = rng.choice(lv, size=(1, 64))
    s, a = oracle.bcq_quantize(w, 2, 64, T=15)
    assert np.allclose((a[:, 0, 0][:, None] * s[:, 0, :]).sum(axis=0), w[0], atol=1e-6)


def test_s11_t0_is_greedy_and_pot_projection_matches_pot_exponent():
    rng = _rng(114)
    w = rng.standard_normal((3, 256)) * 0.02
    s, a = oracle.bcq_quantize(w, 3, 128, T=0)
    for n in range(3):
        for G in range(2):
            ag, Bg = oracle.bcq_greedy(w[n, G * 128:(G + 1) * 128], 3)
            assert np.array_equal(a[:, n, G], ag) and np.array_equal(s[:, n, G * 128:(G + 1) * 128], Bg)
    vals = (rng.standard_normal(2000) * 10.0 ** rng.uniform(-6, 4, 2000)).astype(np.float32)
    e, _ = oracle.pot_exponent(vals)
    for v, ei in zip(vals, e):
        assert oracle.pot_round_exact(float(v)) == math.copysign(2.0 ** int(ei), float(v))


# --------------------------------------- S12: block-wise scales ("Ours (Lat.)", NEXT-f1)
def test_s12_blockwise_exact_pot_scales_reproduce_bcq_sum():
    """alpha_i[b][c] = +-2^P exactly: dequant_blockwise(pack_blockwise(s, alpha)) equals
    sum_i alpha_i[n // (N/8)][k // 8] s_i[n][k] element by element, written out as a scalar
    loop with exact rationals.  Pins the block geometry (8 columns x N/8 rows),
    the per-block sign fold and the bit order (a row-wise or column-wise fold fails)."""
    rng = _rng(120)
    q, N, K = 2, 16, 32
    s = rng.choice([-1, 1], size=(q, N, K)).astype(np.int8)
    P = rng.integers(-5, 6, size=(q, 8, K // 8))
    sign = rng.choice([-1.0, 1.0], size=(q, 8, K // 8))
    alpha = (sign * np.ldexp(1.0, P)).astype(np.float32)
    planes, exps, ncl = oracle.pack_blockwise(s, alpha)
    assert ncl == 0 and exps.shape == (q, 8, K // 8) and np.array_equal(exps, P.astype(np.int8))
    W = oracle.dequant_blockwise(planes, exps, K)
    for n in range(N):
        for k in range(K):
            want = sum(_frac(alpha[i, n // (N // 8), k // 8]) * int(s[i, n, k]) for i in range(q))
            assert _frac(W[n, k]) == want, (n, k)


def test_s12_blockwise_brute_force_gemv_exact():
    """Every sign pattern of one 8-weight key per plane (q = 2, 2^16 patterns would be many;
    here all 256 patterns of plane 0 against a fixed plane 1) at N = 8 rows: y = x W^T as an
    exact rational sum equals gemm_blockwise and the LUT route lut_gemm_blockwise."""
    rng = _rng(121)
    q, N, K = 2, 8, 8
    x = _rand_fp16(rng, (1, K))
    P = rng.integers(-3, 4, size=(q, 8, 1))
    alpha = np.ldexp(1.0, P).astype(np.float32)
    s1 = rng.choice([-1, 1], size=(N, K)).astype(np.int8)
    for pat in range(256):
        s0 = np.array([[1 if (pat >> b) & 1 else -1 for b in range(8)]] * N, dtype=np.int8)
        s0[3] = -s0[3]
        s = np.stack([s0, s1])
        planes, exps, _ = oracle.pack_blockwise(s, alpha)
        y = oracle.gemm_blockwise(x, planes, exps)
        y2 = oracle.lut_gemm_blockwise(x, planes, exps)
        for n in range(N):
            want = sum(_frac(x[0, k]) * _frac(alpha[i, n, 0]) * int(s[i, n, k]) for i in range(q) for k in range(K))
            assert _frac(y[0, n]) == want and _frac(y2[0, n]) == want


def test_s12_blockwise_equals_rowwise_g8_with_replicated_exponents():
    """The block-wise weight is the row-wise g = 8 weight whose exponents are the block's,
    replicated over its N/8 rows: same planes from pack_canonical with alpha
    replicated, same dequantised matrix from the pinned row-wise dequant."""
    rng = _rng(122)
    q, N, K = 3, 40, 64
    s = rng.choice([-1, 1], size=(q, N, K)).astype(np.int8)
    alpha = (rng.choice([-1.0, 1.0], size=(q, 8, K // 8)) * rng.uniform(0.01, 0.2, size=(q, 8, K // 8))).astype(np.float32)
    planes, exps, _ = oracle.pack_blockwise(s, alpha)
    alpha_rows = np.repeat(alpha, N // 8, axis=1)                   # [q][N][K/8]
    planes_r, exps_r, _ = oracle.pack_canonical(s, alpha_rows, 8)
    assert np.array_equal(planes, planes_r)
    assert np.array_equal(oracle.blockwise_row_exps(exps, N), exps_r)
    assert np.array_equal(oracle.dequant_blockwise(planes, exps, K), oracle.dequant(planes_r, exps_r, 8, K))


def test_s12_blockwise_scale_of_one_block_moves_only_its_rows_and_columns():
    """Shifting one exponent e_i[b][c] by d scales exactly rows of block b, columns 8c..8c+7
    of plane i's term by 2^d; everything else is unchanged (exact in fp64)."""
    rng = _rng(123)
    q, N, K = 2, 32, 48
    planes = rng.integers(0, 256, size=(q, N, K // 8), dtype=np.uint8)
    exps = rng.integers(-4, 5, size=(q, 8, K // 8)).astype(np.int8)
    W0 = oracle.dequant_blockwise(planes, exps, K)
    e2 = exps.copy()
    e2[1, 5, 2] += 3
    W1 = oracle.dequant_blockwise(planes, e2, K)
    nb = N // 8
    s1 = oracle.unpack_signs(planes, K)[1].astype(np.float64)
    delta = np.zeros_like(W0)
    delta[5 * nb:6 * nb, 16:24] = s1[5 * nb:6 * nb, 16:24] * (2.0 ** (exps[1, 5, 2] + 3) - 2.0 ** exps[1, 5, 2])
    assert np.array_equal(W1 - W0, delta)
