"""GPU parity of the all-SM streaming LUT-GEMV (kernel id 8, csrc/lut_stream.cu) and of the
fused-projection entry point shiftadd_lut_gemv_fused against the fp64 oracle (bar: reading
R10, floor-normalised relative error <= 2e-3), plus its epoch protocol: many calls of mixed
shapes on one workspace, eagerly and replayed from a CUDA graph, stay bit-identical."""

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


def _case(sa, q, N, K, seed, g=128):
    signs, alpha = synth.gen_layer(q, N, K, g, seed=seed)
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    layer = sa.pack(signs.to(DEV), alpha.to(DEV), g, layout=sa.LAYOUT_TILED)
    return layer, planes, exps


# ragged N (partial last row group, N < 16), one slice (no split-K), chunks straddling slices,
# every q, K up to the LLaMA-2-7B down_proj
SHAPES = [(1, 40, 256), (2, 1000, 512), (3, 777, 2304), (4, 100, 4096), (2, 4096, 11008), (3, 17, 8192),
          (1, 3000, 1024), (4, 2500, 6144)]


@pytest.mark.parametrize("q,N,K", SHAPES)
def test_stream_kernel_parity(sa, q, N, K):
    layer, planes, exps = _case(sa, q, N, K, synth.seed_for(8, q, N))
    x = synth.gen_x(1, K, seed=synth.seed_for(8, 1, K))
    y = sa.lut_gemm(x.to(DEV), layer, splitk=True, pdl=True)
    torch.cuda.synchronize()
    assert sa.gemm_plan(layer, 1)[3] in (3, 8)
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, 128))
    assert err <= TOL, err


@pytest.mark.parametrize("segs", [[(2, 4096), (3, 4096), (2, 4096)],       # LLaMA-2-7B q/k/v, k 3-bit
                                  [(2, 11008), (3, 11008)],                # gate/up, up 3-bit
                                  [(1, 40), (4, 1000), (2, 17), (3, 513)],  # ragged, every q
                                  [(3, 2048)]])
@pytest.mark.parametrize("K", [256, 1024, 4096, 8192])   # 8192: kernel 8 with one slice per CTA (S = 32)
@pytest.mark.parametrize("splitk", [False, True])   # cluster ring (kernel 10) / all-SM streaming (8)
def test_fused_segments_parity(sa, segs, K, splitk):
    if K == 8192 and sum(q * N for q, N in segs) * K / 8 > 16e6:
        pytest.skip("above the one-slice threshold: covered by the K <= 4096 cases")
    x = synth.gen_x(1, K, seed=synth.seed_for(8, 2, K))
    cases = [_case(sa, q, N, K, synth.seed_for(8, 30 + i, q)) for i, (q, N) in enumerate(segs)]
    ys = sa.lut_gemv_fused(x.to(DEV), [c[0] for c in cases], pdl=True, splitk=splitk)
    torch.cuda.synchronize()
    for (layer, planes, exps), y in zip(cases, ys):
        err = oracle.err_floor(y.float().cpu().numpy()[None, :], oracle.gemm(x.numpy(), planes, exps, 128))
        assert err <= TOL, (layer.q, layer.N, err)


def test_fused_matches_separate_calls_within_rounding(sa):
    K = 4096
    x = synth.gen_x(1, K, seed=5).to(DEV)
    layers = [_case(sa, q, 4096, K, synth.seed_for(8, 4, q))[0] for q in (2, 3, 2)]
    fused = sa.lut_gemv_fused(x, layers)
    sep = [sa.lut_gemm(x, L, splitk=True)[0] for L in layers]
    torch.cuda.synchronize()
    for a, b in zip(fused, sep):
        rms = float(b.float().pow(2).mean().sqrt())
        assert float((a.float() - b.float()).abs().max()) <= 2e-3 * max(rms, float(b.float().abs().max()))


def test_epochs_many_calls_one_workspace_and_graph(sa):
    """The epoch counter advances by one per call of kernel 8, whatever its shape; stale words
    of earlier calls (other shapes, same workspace region) are never taken.  Eager calls and a
    CUDA-graph replay of the same sequence give bit-identical outputs."""
    ws = sa.Workspace(DEV)
    specs = [(3, 4736, 8192), (2, 1000, 4096), (3, 4096, 11008), (1, 40, 512)]
    cases = [_case(sa, q, N, K, synth.seed_for(8, 5, i)) for i, (q, N, K) in enumerate(specs)]
    xs = [synth.gen_x(1, K, seed=synth.seed_for(8, 6, i)).to(DEV) for i, (_, _, K) in enumerate(specs)]
    outs = [torch.empty((1, N), dtype=torch.float16, device=DEV) for (_, N, _) in specs]

    def seq():
        for (L, _, _), x, y in zip(cases, xs, outs):
            sa.lut_gemm(x, L, out=y, workspace=ws, pdl=True, splitk=True)

    s = torch.cuda.Stream(DEV)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        seq()
    s.synchronize()
    ref = [y.clone() for y in outs]
    for (L, planes, exps), x, y in zip(cases, xs, ref):
        assert oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.cpu().numpy(), planes, exps, 128)) <= TOL
    with torch.cuda.stream(s):
        for _ in range(10):
            seq()
    s.synchronize()
    for y, r in zip(outs, ref):
        assert torch.equal(y, r)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            seq()
    for y in outs:
        y.zero_()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for _ in range(5):
            g.replay()
    s.synchronize()
    for y, r in zip(outs, ref):
        assert torch.equal(y, r)


def test_stream_basis_vector_and_odd_symmetry_exact(sa):
    """x = e_j gives fp16 of column j of W_hat exactly; y(-x) = -y(x) bit for bit."""
    q, N, K, g = 3, 600, 4096, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(8, 7))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    layer = sa.pack(signs.to(DEV), alpha.to(DEV), g, layout=sa.LAYOUT_TILED)
    W = oracle.dequant(planes, exps, g, K)
    for j in (0, 255, 256, 4095):
        x = torch.zeros((1, K), dtype=torch.float16)
        x[0, j] = 1.0
        y = sa.lut_gemm(x.to(DEV), layer, splitk=True)
        torch.cuda.synchronize()
        want = torch.from_numpy(W[:, j]).to(torch.float16)
        assert torch.equal(y[0].cpu(), want), j
    x = synth.gen_x(1, K, seed=3).to(DEV)
    yp = sa.lut_gemm(x, layer, splitk=True)
    ym = sa.lut_gemm(-x, layer, splitk=True)
    torch.cuda.synchronize()
    assert torch.equal(ym.float(), -yp.float())


@pytest.mark.parametrize("splitk", [False, True])
def test_fused_basis_vector_odd_symmetry_and_determinism(sa, splitk):
    """Fused q/k/v-like segments (q 2/3/2, ragged N) on kernel 10 (cluster) and kernel 8: x = e_j
    gives fp16 of column j of each segment's W_hat exactly; y(-x) = -y(x) and reruns are bit
    for bit identical."""
    K, g = 4096, 128
    segs = [(2, 1000), (3, 777), (2, 1024)]
    cases = []
    for i, (q, N) in enumerate(segs):
        signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(8, 70 + i))
        planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
        cases.append((sa.pack(signs.to(DEV), alpha.to(DEV), g, layout=sa.LAYOUT_TILED),
                      oracle.dequant(planes, exps, g, K)))
    layers = [c[0] for c in cases]
    for j in (0, 255, 256, 4095):
        x = torch.zeros(K, dtype=torch.float16)
        x[j] = 1.0
        ys = sa.lut_gemv_fused(x.to(DEV), layers, splitk=splitk)
        torch.cuda.synchronize()
        for (L, W), y in zip(cases, ys):
            assert torch.equal(y.cpu(), torch.from_numpy(W[:, j]).to(torch.float16)), (j, L.N)
    x = synth.gen_x(1, K, seed=3).view(-1).to(DEV)
    yp = [y.clone() for y in sa.lut_gemv_fused(x, layers, splitk=splitk)]
    ym = sa.lut_gemv_fused(-x, layers, splitk=splitk)
    torch.cuda.synchronize()
    for a, b in zip(yp, ym):
        assert torch.equal(b.float(), -a.float())
    yr = sa.lut_gemv_fused(x, layers, splitk=splitk)
    torch.cuda.synchronize()
    for a, b in zip(yp, yr):
        assert torch.equal(a, b)


# ----------------------------------------------------------------------------- a7 small batch
def _sampled(sa, q, N, K, M, seed, nrows=96, **kw):
    """Device result at a full shape vs the oracle on a row sample (canonical bytes of just
    those rows), floor with the rms of the full device output per batch row."""
    g = 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=seed, device=DEV)
    layer = sa.pack(signs, alpha, g, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(M, K, seed=seed + 1)
    y = sa.lut_gemm(x.to(DEV), layer, pdl=True, **kw)
    torch.cuda.synchronize()
    y = y.float().cpu().numpy()
    rows = np.random.default_rng(seed).choice(N, min(nrows, N), replace=False)
    rows = np.unique(np.concatenate([rows, [0, N - 1]]))
    planes, exps, _ = oracle.pack_canonical(signs[:, rows].cpu().numpy(), alpha[:, rows].cpu().numpy(), g)
    y_ref = oracle.gemm(x.numpy(), planes, exps, g)
    rms = np.sqrt(np.mean(y.astype(np.float64) ** 2, axis=1, keepdims=True))
    den = np.maximum(np.abs(y_ref), rms)
    return float(np.max(np.abs(y[:, rows] - y_ref) / den)), sa.gemm_plan(layer, M)[3]


@pytest.mark.parametrize("M", [5, 8, 16])
@pytest.mark.parametrize("q,N,K", [(2, 4096, 11008), (3, 11008, 4096), (4, 4096, 4096)])
def test_small_batch_single_pass_full_shapes(sa, M, q, N, K):
    """LLaMA-2-7B down_proj / up_proj shapes and a 4-bit layer at M = 5, 8, 16 through the
    streaming kernel's M-wide fp16 LUT entries (one weight pass per 8 rows)."""
    err, kid = _sampled(sa, q, N, K, M, synth.seed_for(8, 40 + M, q))
    assert kid == 8
    assert err <= TOL, err


@pytest.mark.parametrize("M", [2, 3, 4, 6, 7])
@pytest.mark.parametrize("q,N,K", [(2, 4096, 4096), (3, 1000, 2304), (1, 40, 256)])
def test_small_batch_stream_kernel_parity(sa, M, q, N, K):
    """Every entry width (MW = 2, 4, 8) of the streaming kernel, forced, incl. M not a power of 2."""
    signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(8, 50 + M, q))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), 128)
    layer = sa.pack(signs.to(DEV), alpha.to(DEV), 128, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(M, K, seed=synth.seed_for(8, 60 + M))
    y = sa.lut_gemm(x.to(DEV), layer, splitk=True)
    y2 = sa.lut_gemm(x.to(DEV), layer, splitk=True, pdl=True)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm(x.numpy(), planes, exps, 128))
    assert err <= TOL, err


def test_small_batch_mw8_exact_invariants(sa):
    """M = 8 entries: x = e_j in every row gives fp16 of column j exactly (one nonzero group,
    LUT entries exact in fp16 for +-1 sums), and y(-x) = -y(x) bit for bit."""
    q, N, K, g = 2, 300, 2048, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(8, 70))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    layer = sa.pack(signs.to(DEV), alpha.to(DEV), g, layout=sa.LAYOUT_TILED)
    W = oracle.dequant(planes, exps, g, K)
    js = [0, 7, 1000, 2047, 512, 255, 256, 1]
    x = torch.zeros((8, K), dtype=torch.float16)
    for m, j in enumerate(js):
        x[m, j] = 1.0
    y = sa.lut_gemm(x.to(DEV), layer, splitk=True)
    torch.cuda.synchronize()
    for m, j in enumerate(js):
        assert torch.equal(y[m].cpu(), torch.from_numpy(W[:, j]).to(torch.float16)), (m, j)
    xr = synth.gen_x(8, K, seed=4).to(DEV)
    yp = sa.lut_gemm(xr, layer, splitk=True)
    ym = sa.lut_gemm(-xr, layer, splitk=True)
    torch.cuda.synchronize()
    assert torch.equal(ym.float(), -yp.float())


def test_workspace_shared_across_kernel_kinds(sa):
    """One workspace used in turn by the round-1 split-K kernels (1: misaligned exponents, M = 1;
    2: misaligned exponents, M = 8), the streaming kernel (8) on a tiny layer whose CTA 0 finishes
    before most CTAs start (the epoch word must survive the other kernels' fp32 partials), and
    the fused gather's counter region: every result stays at the oracle bar, many times over."""
    ws = sa.Workspace(DEV)
    big, pb, eb = _case(sa, 3, 1000, 2048, synth.seed_for(8, 90))
    buf = torch.empty(big.exps.numel() + 16, dtype=torch.int8, device=DEV)
    ex = buf[3:3 + big.exps.numel()]
    ex.copy_(big.exps)
    moved = sa.PackedLayer(big.planes, ex, big.q, big.N, big.K, big.g, big.layout, big.counts)
    tiny, pt, et = _case(sa, 1, 40, 512, synth.seed_for(8, 91))
    xb = synth.gen_x(8, 2048, seed=92)
    xt = synth.gen_x(1, 512, seed=93)
    ref_b1 = oracle.gemm(xb.numpy()[:1], pb, eb, 128)
    ref_b8 = oracle.gemm(xb.numpy(), pb, eb, 128)
    ref_t = oracle.gemm(xt.numpy(), pt, et, 128)
    xb_d, xt_d = xb.to(DEV), xt.to(DEV)
    for it in range(6):
        y1 = sa.lut_gemm(xb_d[:1], moved, workspace=ws, pdl=True)            # kernel 1
        y8 = sa.lut_gemm(xb_d, moved, workspace=ws, pdl=True)                # kernel 2, M = 8
        ys = [sa.lut_gemm(xt_d, tiny, workspace=ws, pdl=True, splitk=True).clone() for _ in range(8)]   # kernel 8
        torch.cuda.synchronize()
        assert oracle.err_floor(y1.float().cpu().numpy(), ref_b1) <= TOL
        assert oracle.err_floor(y8.float().cpu().numpy(), ref_b8) <= TOL
        for y in ys:
            assert oracle.err_floor(y.float().cpu().numpy(), ref_t) <= TOL, it
    assert int(ws.buf[:65536 * 4 + 16].count_nonzero()) == 0    # counters and the gather counter left zero
