"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  Bars: pack bit-exact; GEMM floor-normalised relative error
<= 2e-3 (BASELINE.json north_star, reading R10); listed invariants bit-exact."""

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 2e-3
DEV = "cuda:0"


@pytest.fixture(scope="module")
def sa():
    import paper_2406_05981_b200 as m
    m.lib()
    return m


def _layer(q, N, K, g, seed):
    signs, alpha = synth.gen_layer(q, N, K, g, seed=seed)
    planes, exps, ncl = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    return signs, alpha, planes, exps


def _gpu(sa, signs, alpha, g, layout):
    return sa.pack(signs.to(DEV), alpha.to(DEV), g, layout=layout)


def _run(sa, x, layer, **kw):
    y = sa.lut_gemm(x.to(DEV), layer, **kw)
    torch.cuda.synchronize()
    return y


# ----------------------------------------------------------------------------- a1: pack
@pytest.mark.parametrize("q,N,K,g", [(3, 768, 768, 128), (1, 40, 512, 256), (4, 17, 1024, 1024),
                                     (2, 100, 4096, 128), (8, 9, 256, 128)])
def test_pack_bit_exact_both_layouts(sa, q, N, K, g):
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(9, q))
    canon = _gpu(sa, signs, alpha, g, sa.LAYOUT_CANONICAL)
    torch.cuda.synchronize()
    assert np.array_equal(canon.planes.cpu().numpy(), planes.reshape(-1))
    assert np.array_equal(canon.exps.cpu().numpy(), exps.reshape(-1))
    pt, et = oracle.to_tiled(planes, exps, g)
    tiled = _gpu(sa, signs, alpha, g, sa.LAYOUT_TILED)
    torch.cuda.synchronize()
    assert np.array_equal(tiled.planes.cpu().numpy(), pt)
    assert np.array_equal(tiled.exps.cpu().numpy(), et)
    assert canon.counts.cpu().tolist() == [0, 0]


def test_pack_canonical_small_groups_and_edge_scales(sa):
    q, N, K, g = 2, 8, 64, 8
    rng = np.random.default_rng(11)
    signs = torch.from_numpy(rng.choice([-1, 1], (q, N, K)).astype(np.int8))
    a = (rng.standard_normal((q, N, K // g)) * 0.05).astype(np.float32)
    a[0, 0, 0] = 0.0
    a[0, 0, 1] = -0.0
    a[0, 1, 0] = 1e-42          # subnormal -> clamp to -100
    a[0, 1, 1] = 2.0 ** 110     # -> clamp to 100
    a[1, 2, 3] = -2.0 ** -101   # -> clamp to -100, signs flipped
    a[1, 3, 0] = np.float32(2 ** 0.5)                                   # just above sqrt(2) in fp32
    a[1, 3, 1] = np.nextafter(np.float32(2 ** 0.5), np.float32(0))      # just below
    alpha = torch.from_numpy(a)
    planes, exps, ncl = oracle.pack_canonical(signs.numpy(), a, g)
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_CANONICAL)
    torch.cuda.synchronize()
    assert np.array_equal(layer.planes.cpu().numpy(), planes.reshape(-1))
    assert np.array_equal(layer.exps.cpu().numpy(), exps.reshape(-1))
    assert layer.counts.cpu().tolist() == [ncl, 0] and ncl == 3


def test_pack_counts_invalid_inputs(sa):
    q, N, K, g = 1, 4, 256, 128
    signs = torch.ones((q, N, K), dtype=torch.int8)
    signs[0, 1, 5] = 0
    signs[0, 2, 7] = 3
    alpha = torch.full((q, N, K // g), 0.01)
    alpha[0, 3, 1] = float("nan")
    alpha[0, 0, 0] = float("inf")
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_CANONICAL)
    torch.cuda.synchronize()
    assert layer.counts.cpu().tolist() == [0, 4]
    e = layer.exps.cpu().numpy().reshape(q, N, K // g)
    assert e[0, 3, 1] == oracle.EXP_ZERO and e[0, 0, 0] == oracle.EXP_ZERO


# ------------------------------------------------------------------- a2-a7: GEMM parity
SHAPES = [
    (3, 768, 768, 128),    # config 0: OPT-125M q_proj
    (1, 40, 512, 128),     # ragged row group (40 = 2.5 x 16)
    (2, 1000, 1280, 256),  # ragged rows, 5 slices, g = 256
    (4, 256, 256, 256),    # single slice (no split-K), q = 4
    (3, 64, 2048, 2048),   # row-wise scales (g = K)
    (2, 4096, 4096, 128),  # OPT-6.7B / LLaMA-2-7B attention at 2 bits
    (2, 23700, 512, 128),  # cluster kernel, C = 1, ragged band of ~10 row groups
    (1, 4000, 3072, 128),  # cluster kernel, C = 3 (12 slices)
    (1, 12000, 4096, 128), # cluster kernel, C = 4, 23 row groups per band
    (3, 1000, 11008, 128), # cluster kernel, 43 slices over clusters of 11 (uneven split)
    (3, 4736, 8192, 128),  # TMA-ring kernel: 64 units per CTA, chunks straddle slices
    (2, 4700, 8448, 128),  # TMA-ring kernel, ragged rows, 33 slices
    (4, 2400, 16384, 128), # TMA-ring kernel, q = 4 (4-stage ring)
    (1, 9500, 4096, 128),  # cluster kernel; forced split-K -> TMA ring, q = 1 (8 stages)
]
# (layout, force split-K): the tiled M = 1 path has two decompositions
KERNELS = [(1, False), (1, True), (0, False)]


@pytest.mark.parametrize("q,N,K,g", SHAPES)
@pytest.mark.parametrize("layout,splitk", KERNELS)
def test_gemv_parity(sa, q, N, K, g, layout, splitk):
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(1, q, N % 7))
    layer = _gpu(sa, signs, alpha, g, layout)
    x = synth.gen_x(1, K, seed=synth.seed_for(1, 99))
    y = _run(sa, x, layer, splitk=splitk)
    y_ref = oracle.gemm(x.numpy(), planes, exps, g)
    assert y.shape == (1, N)
    err = oracle.err_floor(y.float().cpu().numpy(), y_ref)
    assert err <= TOL, err


@pytest.mark.parametrize("M", [2, 3, 4, 5, 8, 16])
@pytest.mark.parametrize("layout", [1, 0])
def test_small_batch_parity(sa, M, layout):
    q, N, K, g = 3, 272, 1024, 128
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(2, M))
    layer = _gpu(sa, signs, alpha, g, layout)
    x = synth.gen_x(M, K, seed=synth.seed_for(2, M, 1))
    y = _run(sa, x, layer)
    y_ref = oracle.gemm(x.numpy(), planes, exps, g)
    err = oracle.err_floor(y.float().cpu().numpy(), y_ref)
    assert err <= TOL, err


@pytest.mark.parametrize("q,N,K", [(2, 4096, 4096), (3, 16384, 4096), (1, 1000, 3072), (3, 40, 512),
                                   (2, 23700, 512)])
@pytest.mark.parametrize("splitk", [False, True])
def test_m2_cluster_ring_parity(sa, q, N, K, splitk):
    """a7 at M = 2 on the cluster TMA ring (kernel 5; splitk forces the small-batch split-K
    kernel), full-size and ragged shapes, output written into a wider buffer (ldy > N)."""
    g = 128
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(2, q, N % 11))
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_TILED)
    assert sa.gemm_plan(layer, 2)[3] == 5
    x = synth.gen_x(2, K, seed=synth.seed_for(2, 5))
    ybuf = torch.full((2, N + 24), 7.0, dtype=torch.float16, device=DEV)
    y = sa.lut_gemm(x.to(DEV), layer, out=ybuf[:, :N], pdl=True, splitk=splitk)
    torch.cuda.synchronize()
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g))
    assert err <= TOL, err
    assert bool((ybuf[:, N:] == 7.0).all())


@pytest.mark.parametrize("M,q,N,K", [(4, 2, 4096, 4096), (3, 3, 11008, 4096), (4, 1, 1000, 3072),
                                     (3, 3, 40, 512), (4, 3, 768, 768)])
@pytest.mark.parametrize("splitk", [False, True])
def test_m4_cluster_ring_parity(sa, M, q, N, K, splitk):
    """a7 at M = 3..4 on the cluster TMA ring (kernel 6, float4 entries; splitk forces the
    small-batch split-K kernel), output written into a wider buffer (ldy > N)."""
    g = 128
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(2, 40 + q, N % 13))
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_TILED)
    assert sa.gemm_plan(layer, M)[3] == 6
    x = synth.gen_x(M, K, seed=synth.seed_for(2, 6, M))
    ybuf = torch.full((M, N + 40), 7.0, dtype=torch.float16, device=DEV)
    y = sa.lut_gemm(x.to(DEV), layer, out=ybuf[:, :N], pdl=True, splitk=splitk)
    torch.cuda.synchronize()
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g))
    assert err <= TOL, err
    assert bool((ybuf[:, N:] == 7.0).all())


@pytest.mark.parametrize("g", [8, 32, 64])
def test_canonical_small_scale_groups(sa, g):
    q, N, K = 2, 70, 576
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(3, g))
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_CANONICAL)
    x = synth.gen_x(3, K, seed=synth.seed_for(3, g, 1))
    y = _run(sa, x, layer)
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g))
    assert err <= TOL, err


def test_mixed_bit_dispatch_interleaved(sa):
    """a6: layers of different q called back to back on one stream each dispatch their own
    instance and stay correct (LLaMA-2-7B-like 2/3-bit mix)."""
    K, g = 1024, 128
    layers = []
    for li, q in enumerate([2, 3, 2, 4, 1, 3]):
        N = 96 + 32 * li
        signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(4, li))
        layers.append((_gpu(sa, signs, alpha, g, sa.LAYOUT_TILED), planes, exps))
    x = synth.gen_x(1, K, seed=synth.seed_for(4, 50))
    outs = [sa.lut_gemm(x.to(DEV), L) for L, _, _ in layers]
    torch.cuda.synchronize()
    for (L, planes, exps), y in zip(layers, outs):
        err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g))
        assert err <= TOL, (L.q, err)


# ------------------------------------------------------------ full-size config parity
def test_m1_kernel_choice(sa):
    """Batch 1: the cluster kernel (K-split over DSMEM) for K <= 4096 where a band holds <= 128
    row groups; otherwise the all-SM streaming kernel (id 8) for K <= 256 x #SMs; the
    register-ring split-K beyond.  Small batch as before."""
    def kid(N, K, M=1, q=1):
        signs, alpha = synth.gen_layer(q, N, K, 128, seed=1, device=DEV)
        return sa.gemm_plan(sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED), M)[3]
    assert kid(4096, 4096) == 3 and kid(16384, 4096) == 3 and kid(256, 256) == 3 and kid(768, 768) == 3
    assert kid(2048, 8192) == 8 and kid(28672, 8192, q=3) == 8 and kid(8192, 28672, q=3) == 8
    assert kid(4096, 11008, q=2) == 8 and kid(80000, 4096) == 8
    assert kid(8192, 2048 * 20) == 1                      # S = 160 > #SMs: register ring
    # small batch: cluster rings for M = 2..4 at K <= 4096 (M = 2 ring: q <= 3); the streaming
    # kernel with M-wide fp16 LUT entries elsewhere (one weight pass per 8 rows)
    assert kid(4096, 4096, M=2, q=3) == 5 and kid(4096, 4096, M=2, q=4) == 8
    assert kid(4096, 8192, M=2) == 8 and kid(4096, 4096, M=3) == 6 and kid(4096, 4096, M=4, q=4) == 8
    assert kid(4096, 4096, M=5) == 8 and kid(4096, 4096, M=16, q=4) == 8 and kid(4096, 11008, M=8) == 8


@pytest.mark.parametrize("splitk", [False, True])
@pytest.mark.parametrize("name,N,K,q", [("fc1", 16384, 4096, 3), ("attn", 4096, 4096, 3),
                                        ("llama7b_down", 4096, 11008, 2)])
def test_config_size_parity_full(sa, name, N, K, q, splitk):
    """Configs 1-2 at full size, in the launch configuration bench.py times (tiled, PDL)."""
    g = 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(1, 7))
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_TILED)
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    x = synth.gen_x(1, K, seed=synth.seed_for(1, 8))
    y = _run(sa, x, layer, pdl=True, splitk=splitk)
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g))
    assert err <= TOL, err


@pytest.mark.parametrize("splitk", [False, True])
def test_llama70b_mlp_sampled_rows(sa, splitk):
    """Config 3 shape (28672 x 8192, 3-bit) on the device; the oracle computes a sample of
    rows one by one from the canonical bytes of just those rows."""
    q, N, K, g = 3, 28672, 8192, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(3, 0), device=DEV)
    layer = sa.pack(signs, alpha, g, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(1, K, seed=synth.seed_for(3, 1))
    y = _run(sa, x, layer, pdl=True, splitk=splitk).float().cpu().numpy()
    rows = np.random.default_rng(3).choice(N, 96, replace=False)
    rows = np.concatenate([rows, [0, 15, 16, N - 1]])
    s_rows = signs[:, rows].cpu().numpy()
    a_rows = alpha[:, rows].cpu().numpy()
    planes, exps, _ = oracle.pack_canonical(s_rows, a_rows, g)
    y_ref = oracle.gemm(x.numpy(), planes, exps, g)
    # floor with the rms of the full output (the sample stands for the whole row)
    full_rms = float(np.sqrt(np.mean(y.astype(np.float64) ** 2)))
    den = np.maximum(np.abs(y_ref[0]), full_rms)
    assert np.max(np.abs(y[0, rows] - y_ref[0]) / den) <= TOL


# --------------------------------------------------------------- exact GPU invariants
def _exact_layer(sa, layout, q=3, N=80, K=512, g=128, seed=5):
    signs, alpha, planes, exps = _layer(q, N, K, g, synth.seed_for(5, seed))
    return _gpu(sa, signs, alpha, g, layout), planes, exps, (q, N, K, g)


@pytest.mark.parametrize("layout,splitk", KERNELS)
def test_basis_vector_gives_rounded_column_exactly(sa, layout, splitk):
    layer, planes, exps, (q, N, K, g) = _exact_layer(sa, layout)
    W = oracle.dequant(planes, exps, g, K)
    for j in (0, 7, 8, 255, 256, 300, K - 1):
        x = synth.gen_special_x("basis", 1, K, j=j)
        y = _run(sa, x, layer, splitk=splitk).cpu().numpy()
        assert np.array_equal(y[0], oracle.to_fp16(W[:, j]))


@pytest.mark.parametrize("layout", [1, 0])
def test_odd_symmetry_bit_exact(sa, layout):
    layer, *_ = _exact_layer(sa, layout)
    x = synth.gen_x(1, 512, seed=7)
    y1 = _run(sa, x, layer).cpu()
    y2 = _run(sa, -x, layer).cpu()
    assert torch.equal(y2, -y1) or torch.equal(y2.float(), -y1.float())


@pytest.mark.parametrize("layout", [1, 0])
@pytest.mark.parametrize("d", [-3, 2])
def test_exponent_shift_scales_exactly(sa, layout, d):
    q, N, K, g = 3, 80, 512, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(5, 1))
    x = synth.gen_x(1, K, seed=8)
    y0 = _run(sa, x, _gpu(sa, signs, alpha, g, layout)).float().cpu().numpy()
    y1 = _run(sa, x, _gpu(sa, signs, alpha * (2.0 ** d), g, layout)).float().cpu().numpy()
    ok = (np.abs(y0) >= 2.0 ** -10) & (np.abs(y0) <= 2.0 ** 10)
    assert ok.mean() > 0.9
    assert np.array_equal(y1[ok], np.ldexp(y0[ok], d))


@pytest.mark.parametrize("layout", [1, 0])
def test_all_zero_scales_give_zero(sa, layout):
    q, N, K, g = 2, 48, 512, 128
    signs = torch.ones((q, N, K), dtype=torch.int8)
    alpha = torch.zeros((q, N, K // g))
    layer = _gpu(sa, signs, alpha, g, layout)
    y = _run(sa, synth.gen_x(2, K, seed=1), layer).float().cpu()
    assert torch.count_nonzero(y) == 0


def test_nan_input_propagates(sa):
    layer, *_ = _exact_layer(sa, 1)
    x = synth.gen_x(1, 512, seed=9)
    x[0, 3] = float("nan")
    y = _run(sa, x, layer).float().cpu()
    assert torch.isnan(y).all()


@pytest.mark.parametrize("splitk", [False, True])
def test_deterministic_and_workspace_left_zeroed(sa, splitk):
    q, N, K, g = 3, 2000, 4096, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(6, 0))
    layer = _gpu(sa, signs, alpha, g, sa.LAYOUT_TILED)
    ws = sa.Workspace(DEV)
    x = synth.gen_x(1, K, seed=3).to(DEV)
    ys = [sa.lut_gemm(x, layer, workspace=ws, pdl=bool(i & 1), splitk=splitk).clone() for i in range(4)]
    torch.cuda.synchronize()
    for y in ys[1:]:
        assert torch.equal(y, ys[0])
    assert int(ws.buf[:65536 * 4].count_nonzero()) == 0   # the per-row-group counters


def test_workspace_reuse_across_shapes(sa):
    """One workspace serves calls of different shapes back to back (counters at a fixed
    region; partial regions of one shape overlap counters of none)."""
    ws = sa.Workspace(DEV)
    cases = []
    for i, (q, N, K) in enumerate([(3, 768, 768), (1, 40, 512), (2, 4000, 4096), (3, 64, 8192), (2, 500, 1024)]):
        signs, alpha, planes, exps = _layer(q, N, K, 128, synth.seed_for(6, 10 + i))
        cases.append((_gpu(sa, signs, alpha, 128, sa.LAYOUT_TILED), planes, exps, K))
    for rep in range(2):
        for L, planes, exps, K in cases:
            for M in (1, 3):
                x = synth.gen_x(M, K, seed=rep * 10 + M)
                y = sa.lut_gemm(x.to(DEV), L, workspace=ws)
                torch.cuda.synchronize()
                err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, 128))
                assert err <= TOL, (L.N, L.K, M, err)


def test_writes_into_wider_output_buffer(sa):
    layer, planes, exps, (q, N, K, g) = _exact_layer(sa, 1)
    x = synth.gen_x(2, K, seed=10)
    out = torch.full((2, N + 24), 7.0, dtype=torch.float16, device=DEV)
    sa.lut_gemm(x.to(DEV), layer, out=out[:, :N])
    torch.cuda.synchronize()
    assert torch.all(out[:, N:] == 7.0)
    err = oracle.err_floor(out[:, :N].float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g))
    assert err <= TOL


def test_gpu_rejects_bad_arguments(sa):
    layer, *_ = _exact_layer(sa, 1)
    x = synth.gen_x(17, 512, seed=1).to(DEV)
    with pytest.raises(sa.ShiftAddError, match="unsupported"):
        sa.lut_gemm(x, layer)
    with pytest.raises(ValueError):
        sa.lut_gemm(x[:1, :256], layer)


def test_stream_kernel_exact_invariants(sa):
    """Kernel 8 (all-SM streaming, chunks straddling two slices, epoch-tagged split-K):
    y(-x) = -y(x) bit-exactly, run-to-run bit-identical with and without PDL, the older
    kernels' counter region untouched."""
    q, N, K, g = 3, 4736, 8192, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(6, 4), device=DEV)
    layer = sa.pack(signs, alpha, g, layout=sa.LAYOUT_TILED)
    assert sa.gemm_plan(layer, 1)[3] == 8
    ws = sa.Workspace(DEV)
    x = synth.gen_x(1, K, seed=11).to(DEV)
    ys = [sa.lut_gemm(x, layer, workspace=ws, pdl=bool(i & 1)).clone() for i in range(4)]
    yn = sa.lut_gemm(-x, layer, workspace=ws)
    torch.cuda.synchronize()
    for y in ys[1:]:
        assert torch.equal(y, ys[0])
    assert torch.equal(yn.float(), -ys[0].float())
    assert int(ws.buf[:65536 * 4].count_nonzero()) == 0


@pytest.mark.parametrize("q,N,K", [(3, 4096, 4096), (2, 4736, 8192)])
def test_misaligned_exponents_use_register_ring(sa, q, N, K):
    """The TMA rings copy exponent tiles with 16-B bulk copies; an exponent array that is not
    16-B aligned takes the register-ring kernels (own launch shape) and gives the same y."""
    g = 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(6, 7, q), device=DEV)
    layer = sa.pack(signs, alpha, g, layout=sa.LAYOUT_TILED)
    buf = torch.empty(layer.exps.numel() + 16, dtype=torch.int8, device=DEV)
    ex = buf[3:3 + layer.exps.numel()]
    ex.copy_(layer.exps)
    assert ex.data_ptr() % 16 != 0
    moved = sa.PackedLayer(layer.planes, ex, q, N, K, g, layer.layout, layer.counts)
    x = synth.gen_x(1, K, seed=12).to(DEV)
    y0 = sa.lut_gemm(x, layer)
    y1 = sa.lut_gemm(x, moved, pdl=True)
    torch.cuda.synchronize()
    planes, exps, _ = oracle.pack_canonical(signs.cpu().numpy(), alpha.cpu().numpy(), g)
    y_ref = oracle.gemm(x.cpu().numpy(), planes, exps, g)
    for y in (y0, y1):
        assert oracle.err_floor(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("q,N,K,M", [(4, 1024, 1024, 5), (2, 4096, 11008, 8), (3, 272, 1024, 16), (4, 300, 4096, 12)])
def test_misaligned_exponents_small_batch_split_k_kernel(sa, q, N, K, M):
    """An exponent array that is not 16-B aligned sends M > 1 to the small-batch split-K kernel
    (gemm_tiled_mb.cu, kernel 2): its row-chunk loop for M > 4 (chunks of 4 rows re-walking the
    CTA's units, S * ceil(M/4) arrivals per row group) at q = 4 and at the LLaMA-2-7B down_proj
    shape; the same y as the oracle, and the counter region is left zeroed."""
    g = 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(6, 8, q + M), device=DEV)
    layer = sa.pack(signs, alpha, g, layout=sa.LAYOUT_TILED)
    buf = torch.empty(layer.exps.numel() + 16, dtype=torch.int8, device=DEV)
    ex = buf[5:5 + layer.exps.numel()]
    ex.copy_(layer.exps)
    assert ex.data_ptr() % 16 != 0
    moved = sa.PackedLayer(layer.planes, ex, q, N, K, g, layer.layout, layer.counts)
    x = synth.gen_x(M, K, seed=13 + M)
    ws = sa.Workspace(DEV)
    y = sa.lut_gemm(x.to(DEV), moved, workspace=ws, pdl=True)
    torch.cuda.synchronize()
    planes, exps, _ = oracle.pack_canonical(signs.cpu().numpy(), alpha.cpu().numpy(), g)
    assert oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, g)) <= TOL
    assert int(ws.buf[:65536 * 4].count_nonzero()) == 0


@pytest.mark.parametrize("M,kid", [(2, 5), (3, 6), (4, 6), (7, 8)])
def test_small_batch_ring_exact_invariants(sa, M, kid):
    """The small-batch kernels (cluster rings with float2 / float4 entries; M = 7: the streaming
    kernel with 8-wide fp16 entries): row m of x
    set to the basis vector e_{j_m} gives the fp16-rounded column j_m exactly, and
    y(-x) = -y(x) bit-exactly."""
    layer, planes, exps, (q, N, K, g) = _exact_layer(sa, 1, q=3, N=80, K=1024)
    assert sa.gemm_plan(layer, M)[3] == kid
    W = oracle.dequant(planes, exps, g, K)
    js = [0, 7, 256, 300, 511, 1000, K - 1][:M]
    x = torch.zeros((M, K), dtype=torch.float16)
    for m, j in enumerate(js):
        x[m, j] = 1.0
    y = _run(sa, x, layer).cpu().numpy()
    for m, j in enumerate(js):
        assert np.array_equal(y[m], oracle.to_fp16(W[:, j])), (m, j)
    xr = synth.gen_x(M, K, seed=21)
    y1 = _run(sa, xr, layer).float().cpu()
    y2 = _run(sa, -xr, layer).float().cpu()
    assert torch.equal(y2, -y1)
