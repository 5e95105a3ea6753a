"""GPU parity of NEXT-f4 (Alg. 1 alternating multi-bit BCQ) through the C
ABI against the fp64 oracle (oracle.bcq_quantize).  Both run in fp64, so the integer
decisions (signs) must be identical and the scales agree to fp32 rounding."""

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def sa():
    import paper_2406_05981_b200 as m
    m.lib()
    return m


def _w(N, K, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn((N, K), generator=g) * 0.02).float()


@pytest.mark.parametrize("q", [1, 2, 3, 4])
@pytest.mark.parametrize("T,pot", [(0, False), (3, False), (15, False), (15, True)])
def test_quantize_matches_oracle(sa, q, T, pot):
    N, K, g = 48, 512, 128
    w = _w(N, K, 100 + q)
    s_ref, a_ref = oracle.bcq_quantize(w.numpy(), q, g, T, pot=pot)
    s, a = sa.bcq_quantize(w.to(DEV), q, g, T=T, pot=pot)
    assert np.array_equal(s.cpu().numpy(), s_ref)
    a = a.cpu().numpy().astype(np.float64)
    if pot:
        assert np.array_equal(a, a_ref)
    else:
        assert np.allclose(a, a_ref, rtol=1.2e-7, atol=0)


def test_quantize_rowwise_groups_and_small_groups(sa):
    for (N, K, g, q) in [(16, 1024, 1024, 2), (8, 96, 8, 3), (5, 40, 40, 4)]:
        w = _w(N, K, 7 + g)
        s_ref, a_ref = oracle.bcq_quantize(w.numpy(), q, g, 6)
        s, a = sa.bcq_quantize(w.to(DEV), q, g, T=6)
        assert np.array_equal(s.cpu().numpy(), s_ref), (N, K, g, q)
        assert np.allclose(a.cpu().numpy().astype(np.float64), a_ref, rtol=1.2e-7, atol=0)


def test_quantize_pack_gemv_pipeline(sa):
    """Quantise -> pack -> LUT-GEMV on the device equals the oracle GEMM of the
    oracle-quantised, oracle-packed layer (the whole chain in front of and through a1-a5)."""
    N, K, g, q = 1024, 1024, 128, 3
    w = _w(N, K, 11)
    s, a = sa.bcq_quantize(w.to(DEV), q, g, T=10, pot=True)
    L = sa.pack(s, a, g, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(1, K, seed=12)
    y = sa.lut_gemm(x.to(DEV), L).float().cpu().numpy()
    s_ref, a_ref = oracle.bcq_quantize(w.numpy(), q, g, 10, pot=True)
    planes, exps, _ = oracle.pack_canonical(s_ref, a_ref.astype(np.float32), g)
    assert oracle.err_floor(y, oracle.gemm(x.numpy(), planes, exps, g)) <= 2e-3


def test_alternating_refinement_reduces_error(sa):
    N, K, g, q = 256, 2048, 128, 3
    w = _w(N, K, 13).to(DEV)
    errs = []
    for T in (0, 15):
        s, a = sa.bcq_quantize(w, q, g, T=T)
        wq = (s.float() * a.repeat_interleave(g, dim=2)).sum(dim=0)
        errs.append(float(((w - wq) ** 2).sum()))
    assert errs[1] < 0.95 * errs[0], errs
