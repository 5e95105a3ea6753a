"""GPU parity of NEXT-f1 block-wise scales ("Ours (Lat.)"): device pack
bit-exact against oracle.pack_blockwise (both layouts), the block-wise LUT-GEMV against the
fp64 oracle (reading R10 bar), and exact invariants."""

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


@pytest.mark.parametrize("q,N,K", [(2, 64, 256), (3, 1000, 1024), (1, 40, 512), (4, 4096, 2048)])
def test_pack_blockwise_bit_exact(sa, q, N, K):
    signs, alpha = synth.gen_layer_blockwise(q, N, K, seed=synth.seed_for(11, q, N))
    planes, exps, ncl = oracle.pack_blockwise(signs.numpy(), alpha.numpy())
    canon = sa.pack_blockwise(signs.to(DEV), alpha.to(DEV), layout=sa.LAYOUT_CANONICAL)
    tiled = sa.pack_blockwise(signs.to(DEV), alpha.to(DEV), layout=sa.LAYOUT_TILED)
    torch.cuda.synchronize()
    assert np.array_equal(canon.planes.cpu().numpy(), planes.reshape(-1))
    assert np.array_equal(canon.exps.cpu().numpy(), exps.reshape(-1))
    assert np.array_equal(tiled.exps.cpu().numpy(), exps.reshape(-1))
    pt, _ = oracle.to_tiled(planes, np.zeros((q, N, K // 128), np.int8), 128)
    assert np.array_equal(tiled.planes.cpu().numpy(), pt)
    assert canon.counts.cpu().tolist() == [0, 0]


@pytest.mark.parametrize("q,N,K", [(2, 4096, 4096), (3, 11008, 4096), (2, 4096, 11008), (1, 40, 256),
                                   (4, 1000, 2304), (3, 8, 512)])
def test_blockwise_gemv_parity(sa, q, N, K):
    signs, alpha = synth.gen_layer_blockwise(q, N, K, seed=synth.seed_for(11, 5, N + q))
    planes, exps, _ = oracle.pack_blockwise(signs.numpy(), alpha.numpy())
    layer = sa.pack_blockwise(signs.to(DEV), alpha.to(DEV))
    x = synth.gen_x(1, K, seed=synth.seed_for(11, 6, K))
    y = sa.lut_gemm(x.to(DEV), layer, pdl=True)
    y2 = sa.lut_gemv_blockwise(x.to(DEV), layer)
    torch.cuda.synchronize()
    assert torch.equal(y[0], y2)
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm_blockwise(x.numpy(), planes, exps))
    assert err <= TOL, err


def test_blockwise_exact_invariants(sa):
    """x = e_j gives fp16 of column j of W_hat (block scales included) exactly; y(-x) = -y(x)
    bit for bit; shifting every exponent by d scales y by 2^d exactly."""
    q, N, K = 3, 512, 2048
    signs, alpha = synth.gen_layer_blockwise(q, N, K, seed=synth.seed_for(11, 7))
    planes, exps, _ = oracle.pack_blockwise(signs.numpy(), alpha.numpy())
    layer = sa.pack_blockwise(signs.to(DEV), alpha.to(DEV))
    W = oracle.dequant_blockwise(planes, exps, K)
    for j in (0, 9, 255, 256, 2047):
        x = torch.zeros(K, dtype=torch.float16)
        x[j] = 1.0
        y = sa.lut_gemv_blockwise(x.to(DEV), layer)
        torch.cuda.synchronize()
        assert torch.equal(y.cpu(), torch.from_numpy(W[:, j]).to(torch.float16)), j
    x = synth.gen_x(1, K, seed=8).to(DEV)
    yp = sa.lut_gemv_blockwise(x, layer)
    ym = sa.lut_gemv_blockwise(-x, layer)
    shifted = sa.PackedLayer(layer.planes, layer.exps + 2, q, N, K, 8, layer.layout, layer.counts, blockwise=True)
    ys = sa.lut_gemv_blockwise(x, shifted)
    torch.cuda.synchronize()
    assert torch.equal(ym.float(), -yp.float())
    assert torch.equal(ys.float(), (yp.float() * 4).to(torch.float16).float())
