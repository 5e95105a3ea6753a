"""GPU parity of NEXT-f1 (column-wise scales, "Ours (Acc.)") through the
C ABI against the fp64 oracle (oracle.pack_colwise / gemm_colwise).  Bars as DESIGN.md
§Parity: pack bit-exact; GEMV floor-normalised error <= 2e-3; listed invariants exact."""

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


def _layer(q, N, K, seed):
    s, a = synth.gen_layer_colwise(q, N, K, seed=seed)
    planes, e, ncl = oracle.pack_colwise(s.numpy(), a.numpy())
    return s, a, planes, e


@pytest.mark.parametrize("layout", [1, 0])
def test_colwise_pack_bit_exact(sa, layout):
    q, N, K = 3, 40, 512
    s, a, planes, e = _layer(q, N, K, synth.seed_for(8, 0))
    a = a.clone()
    a[0, 5] = -a[0, 5]                       # negative column scales fold into that column
    a[1, 17] = 0.0                           # zero scale -> EXP_ZERO
    a[2, 3] = 2.0 ** -120                    # clamps
    planes, e, ncl = oracle.pack_colwise(s.numpy(), a.numpy())
    L = sa.pack_colwise(s.to(DEV), a.to(DEV), layout=layout)
    want = oracle.tile_planes(planes) if layout == 1 else planes
    assert np.array_equal(L.planes.cpu().numpy().reshape(-1), want.reshape(-1))
    assert np.array_equal(L.exps.cpu().numpy().reshape(q, K), e)
    assert L.counts.cpu().tolist() == [ncl, 0] and ncl == 1


SHAPES = [
    (3, 768, 768),      # config 0 shape, 3 slices -> clusters of 3
    (1, 40, 512),       # ragged row group, 2 slices
    (2, 1000, 1280),    # ragged rows, 5 slices
    (4, 256, 256),      # one slice (cluster of 1), q = 4
    (2, 4096, 4096),    # OPT-6.7B attention, clusters of 16
    (3, 16384, 4096),   # OPT-6.7B FC1 at full size
]


# K > 4096 (the streaming kernel, per-plane column-scaled LUTs): LLaMA-2-70B gate/up K, the
# LLaMA-2-7B down_proj, a ragged 70B-down-like K = 28672
SHAPES_K = [(3, 8192, 8192), (2, 4096, 11008), (3, 1000, 28672), (1, 40, 4352)]


@pytest.mark.parametrize("q,N,K,splitk", [(q, N, K, False) for q, N, K in SHAPES] +
                         [(q, N, K, True) for q, N, K in SHAPES[:5]] + [(q, N, K, False) for q, N, K in SHAPES_K])
def test_colwise_gemv_parity(sa, q, N, K, splitk):
    s, a, planes, e = _layer(q, N, K, synth.seed_for(8, q, N % 7))
    L = sa.pack_colwise(s.to(DEV), a.to(DEV))
    x = synth.gen_x(1, K, seed=synth.seed_for(8, 99))
    y = sa.lut_gemv_colwise(x.to(DEV), L, pdl=True, splitk=splitk)
    torch.cuda.synchronize()
    err = oracle.err_floor(y.float().cpu().numpy()[None, :], oracle.gemm_colwise(x.numpy(), planes, e))
    assert err <= TOL, err


@pytest.mark.parametrize("q,N,K,M", [(3, 768, 768, 2), (2, 4096, 4096, 3), (4, 1000, 8192, 2), (3, 4096, 11008, 8),
                                     (1, 40, 512, 16)])
def test_colwise_small_batch_parity(sa, q, N, K, M):
    """a7 x column-wise scales: pairs of rows per weight pass (fp16-pair plane LUTs), odd M's
    last row on the M = 1 path; every row within the oracle bar."""
    s, a, planes, e = _layer(q, N, K, synth.seed_for(8, 40 + q, M))
    L = sa.pack_colwise(s.to(DEV), a.to(DEV))
    x = synth.gen_x(M, K, seed=synth.seed_for(8, 41, M))
    y = sa.lut_gemv_colwise(x.to(DEV), L, pdl=True)
    torch.cuda.synchronize()
    assert tuple(y.shape) == (M, N)
    err = oracle.err_floor(y.float().cpu().numpy(), oracle.gemm_colwise(x.numpy(), planes, e))
    assert err <= TOL, err


def test_colwise_pair_rows_basis_vectors_exact(sa):
    """M = 2: row m = e_{j_m} gives the fp16 column j_m exactly (an fp16 LUT entry of one
    scaled activation is exact), and swapping the rows swaps the outputs bit for bit."""
    q, N, K = 3, 80, 1024
    s, a, planes, e = _layer(q, N, K, synth.seed_for(8, 50))
    L = sa.pack_colwise(s.to(DEV), a.to(DEV))
    W = oracle.dequant_colwise(planes, e, K)
    x = torch.zeros((2, K), dtype=torch.float16)
    x[0, 7] = 1.0
    x[1, 600] = 1.0
    y = sa.lut_gemv_colwise(x.to(DEV), L).cpu().numpy()
    assert np.array_equal(y[0], oracle.to_fp16(W[:, 7])) and np.array_equal(y[1], oracle.to_fp16(W[:, 600]))
    xr = synth.gen_x(2, K, seed=9)
    y1 = sa.lut_gemv_colwise(xr.to(DEV), L)
    y2 = sa.lut_gemv_colwise(xr.flip(0).contiguous().to(DEV), L)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2.flip(0))


@pytest.mark.parametrize("K,splitk", [(512, False), (512, True), (8192, False)])
def test_colwise_basis_vector_gives_rounded_column_exactly(sa, K, splitk):
    q, N = 3, 80
    s, a, planes, e = _layer(q, N, K, synth.seed_for(8, 7))
    L = sa.pack_colwise(s.to(DEV), a.to(DEV))
    W = oracle.dequant_colwise(planes, e, K)
    for j in (0, 7, 8, 255, 256, 300, K - 1):
        x = synth.gen_special_x("basis", 1, K, j=j)
        y = sa.lut_gemv_colwise(x.to(DEV), L, splitk=splitk).cpu().numpy()
        assert np.array_equal(y, oracle.to_fp16(W[:, j]))


@pytest.mark.parametrize("K", [1024, 8192])
def test_colwise_column_scaling_equals_exponent_shift_bit_exact(sa, K):
    """x[k] * 2 with exps e  ==  x with e_i[k] + 1 for every plane: the kernel pre-shifts x by
    an exact power of two, so both build identical LUTs and the outputs are identical."""
    q, N = 2, 300
    s, a, _, _ = _layer(q, N, K, synth.seed_for(8, 8))
    L = sa.pack_colwise(s.to(DEV), a.to(DEV))
    a2 = a.clone()
    for k in (3, 500, 1023):
        a2[:, k] *= 2.0
    L2 = sa.pack_colwise(s.to(DEV), a2.to(DEV))
    x = synth.gen_x(1, K, seed=3)
    x2 = x.clone()
    for k in (3, 500, 1023):
        x2[0, k] *= 2.0
    y1 = sa.lut_gemv_colwise(x2.to(DEV), L)
    y2 = sa.lut_gemv_colwise(x.to(DEV), L2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


def test_colwise_constant_exponents_match_rowwise_kernel(sa):
    """Column-wise scales constant per plane are a row-wise layer with g = K: the two CUDA
    paths agree within rounding order, and both meet the oracle bar."""
    q, N, K = 3, 2048, 2048
    s, _ = synth.gen_layer(q, N, K, K, seed=5)
    c = torch.tensor([2.0 ** -3, 2.0 ** -5, 2.0 ** -6])
    a_col = c[:, None].repeat(1, K).contiguous()
    a_row = c[:, None, None].repeat(1, N, 1).contiguous()
    Lc = sa.pack_colwise(s.to(DEV), a_col.to(DEV))
    Lr = sa.pack(s.to(DEV), a_row.to(DEV), K, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(1, K, seed=6)
    yc = sa.lut_gemv_colwise(x.to(DEV), Lc).float().cpu().numpy()
    yr = sa.lut_gemm(x.to(DEV), Lr).float().cpu().numpy()[0]
    planes, e, _ = oracle.pack_colwise(s.numpy(), a_col.numpy())
    ref = oracle.gemm_colwise(x.numpy(), planes, e)
    assert oracle.err_floor(yc[None, :], ref) <= TOL
    assert oracle.err_floor(yr[None, :], ref) <= TOL


def test_colwise_deterministic(sa):
    q, N, K = 3, 4096, 4096
    s, a = synth.gen_layer_colwise(q, N, K, seed=9, device=DEV)
    L = sa.pack_colwise(s, a)
    x = synth.gen_x(1, K, seed=3).to(DEV)
    ys = [sa.lut_gemv_colwise(x, L, pdl=bool(i & 1)).clone() for i in range(4)]
    torch.cuda.synchronize()
    for y in ys[1:]:
        assert torch.equal(y, ys[0])


def test_colwise_unsupported_shapes(sa):
    """The canonical layout and K above 256 x #SMs stay unsupported (reported, never a fallback)."""
    s, a = synth.gen_layer_colwise(1, 64, 8192, seed=1, device=DEV)
    Lc = sa.pack_colwise(s, a, layout=sa.LAYOUT_CANONICAL)
    with pytest.raises(sa.ShiftAddError, match="unsupported"):
        sa.lut_gemv_colwise(synth.gen_x(1, 8192, seed=1).to(DEV), Lc)
    K = 256 * (torch.cuda.get_device_properties(0).multi_processor_count + 1)
    s, a = synth.gen_layer_colwise(1, 16, K, seed=1, device=DEV)
    with pytest.raises(sa.ShiftAddError, match="unsupported"):
        sa.lut_gemv_colwise(synth.gen_x(1, K, seed=1).to(DEV), sa.pack_colwise(s, a))
