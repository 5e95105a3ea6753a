"""GPU parity of NEXT-f2 (additive PoT, K = 2 terms per scale, Eq. 2)
through the C ABI against the fp64 oracle (oracle.pack_apot2 / gemm_apot2)."""

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


@pytest.mark.parametrize("layout", [1, 0])
def test_apot2_pack_bit_exact(sa, layout):
    q, N, K, g = 3, 40, 512, 128
    s, a = synth.gen_layer(q, N, K, g, seed=synth.seed_for(9, 0))
    a = a.clone()
    a[0, 0, 0] = 0.0
    a[1, 2, 1] = -3.0
    a[2, 5, 3] = 2.0 ** 120        # clamped: no second term
    a[0, 7, 2] = 2.0 ** -5         # exact power of two: no second term
    planes, e1, e2, ncl = oracle.pack_apot2(s.numpy(), a.numpy(), g)
    L = sa.pack_apot2(s.to(DEV), a.to(DEV), g, layout=layout)
    if layout == 1:
        want_p, want_e1 = oracle.to_tiled(planes, e1, g)
        _, want_e2 = oracle.to_tiled(planes, e2, g)
        # padded rows of the last row group carry "no second term" (0), not EXP_ZERO
        pad = oracle.to_tiled(planes, np.zeros_like(e2), g)[1] == oracle.EXP_ZERO
        want_e2 = np.where(pad, 0, want_e2).astype(np.int8)
    else:
        want_p, want_e1, want_e2 = planes, e1, e2
    assert np.array_equal(L.planes.cpu().numpy().reshape(-1), want_p.reshape(-1))
    assert np.array_equal(L.exps.cpu().numpy().reshape(-1), want_e1.reshape(-1))
    assert np.array_equal(L.exps2.cpu().numpy().reshape(-1), want_e2.reshape(-1))
    assert L.counts.cpu().tolist() == [ncl, 0]
    assert int(np.count_nonzero(e2)) > 0.9 * e2.size     # nearly every group has a 2nd term


# K <= 4096: cluster kernel (and the streaming kernel with splitk); K > 4096 -- the LLaMA-2-7B
# down_proj, a 70B-gate-like K = 8192 and a ragged K = 28672 shape -- on the streaming kernel
@pytest.mark.parametrize("q,N,K,splitk", [(3, 768, 768, False), (1, 40, 512, False), (2, 4096, 4096, False),
                                          (3, 16384, 4096, False), (2, 2048, 8192, False), (3, 768, 768, True),
                                          (2, 4096, 4096, True), (2, 4096, 11008, False), (3, 3000, 8192, False),
                                          (4, 600, 28672, False)])
def test_apot2_tiled_gemv_parity(sa, q, N, K, splitk):
    g = 128
    s, a = synth.gen_layer(q, N, K, g, seed=synth.seed_for(9, q, N % 7))
    planes, e1, e2, _ = oracle.pack_apot2(s.numpy(), a.numpy(), g)
    L = sa.pack_apot2(s.to(DEV), a.to(DEV), g, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(1, K, seed=synth.seed_for(9, 99))
    y = sa.lut_gemm(x.to(DEV), L, pdl=True, splitk=splitk)
    torch.cuda.synchronize()
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm_apot2(x.numpy(), planes, e1, e2, g))
    assert err <= TOL, err


@pytest.mark.parametrize("M,g", [(1, 128), (3, 32), (16, 256)])
def test_apot2_canonical_gemm_parity(sa, M, g):
    q, N, K = 3, 300, 1024
    s, a = synth.gen_layer(q, N, K, g, seed=synth.seed_for(9, M, g))
    planes, e1, e2, _ = oracle.pack_apot2(s.numpy(), a.numpy(), g)
    L = sa.pack_apot2(s.to(DEV), a.to(DEV), g, layout=sa.LAYOUT_CANONICAL)
    x = synth.gen_x(M, K, seed=synth.seed_for(9, 98))
    y = sa.lut_gemm(x.to(DEV), L)
    torch.cuda.synchronize()
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm_apot2(x.numpy(), planes, e1, e2, g))
    assert err <= TOL, err


@pytest.mark.parametrize("layout,splitk", [(1, False), (1, True), (0, False)])
def test_apot2_exact_two_term_scales_basis_vectors(sa, layout, splitk):
    """alpha = +-(2^A + sigma 2^B), A - B >= 2, is represented exactly by two terms, so for
    x = e_j the output is fp16(sum_i alpha_i s_i[:, j]) -- computed from alpha, not the oracle."""
    rng = np.random.default_rng(7)
    q, N, K, g = 2, 48, 512, 128
    A = rng.integers(-8, -2, size=(q, N, K // g))
    B = A - rng.integers(2, 7, size=A.shape)
    alpha = (rng.choice([-1.0, 1.0], size=A.shape) *
             (np.ldexp(1.0, A) + rng.choice([-1.0, 1.0], size=A.shape) * np.ldexp(1.0, B))).astype(np.float32)
    s = rng.choice([-1, 1], size=(q, N, K)).astype(np.int8)
    L = sa.pack_apot2(torch.from_numpy(s).to(DEV), torch.from_numpy(alpha).to(DEV), g, layout=layout)
    W = (s.astype(np.float64) * np.repeat(alpha.astype(np.float64), g, axis=2)).sum(axis=0)
    for j in (0, 9, 128, 300, K - 1):
        x = synth.gen_special_x("basis", 1, K, j=j)
        y = sa.lut_gemm(x.to(DEV), L, splitk=splitk).cpu().numpy()
        assert np.array_equal(y[0], oracle.to_fp16(W[:, j]))


def test_apot2_is_more_accurate_than_one_term(sa):
    """The point of K = 2 (Eq. 2): against the unquantised-scale product sum_i alpha_i s_i x,
    the K = 2 kernel output is closer than the K = 1 one."""
    q, N, K, g = 3, 4096, 4096, 128
    s, a = synth.gen_layer(q, N, K, g, seed=11)
    x = synth.gen_x(1, K, seed=12)
    W = (s.double() * a.double().repeat_interleave(g, dim=2)).sum(dim=0)
    y_true = (x.double() @ W.T).numpy()
    L1 = sa.pack(s.to(DEV), a.to(DEV), g, layout=sa.LAYOUT_TILED)
    L2 = sa.pack_apot2(s.to(DEV), a.to(DEV), g, layout=sa.LAYOUT_TILED)
    e1 = oracle.err_normwise(sa.lut_gemm(x.to(DEV), L1).float().cpu().numpy(), y_true)
    e2 = oracle.err_normwise(sa.lut_gemm(x.to(DEV), L2).float().cpu().numpy(), y_true)
    assert e2 < 0.5 * e1, (e1, e2)


def test_apot2_unsupported(sa):
    s, a = synth.gen_layer(1, 64, 512, 128, seed=1, device=DEV)
    L = sa.pack_apot2(s, a, 128, layout=sa.LAYOUT_TILED)
    with pytest.raises(sa.ShiftAddError, match="unsupported"):
        sa.lut_gemm(synth.gen_x(2, 512, seed=1).to(DEV), L)
