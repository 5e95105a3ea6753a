"""§8(d) e2e transfers: shiftadd_copy (kernel copy between pinned host and device memory,
inside the PDL chain).  Bytes are compared exactly."""
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def sa():
    import paper_2406_05981_b200 as m
    m.lib()
    return m


@pytest.mark.parametrize("n", [16, 4096 + 8, 40000])
@pytest.mark.parametrize("pdl,ready", [(False, False), (True, True), (True, False)])
def test_copy_roundtrip_bit_exact(sa, n, pdl, ready):
    h = torch.randint(-2 ** 15, 2 ** 15, (n,), dtype=torch.int16).pin_memory()
    d = torch.empty(n, dtype=torch.int16, device=DEV)
    back = torch.zeros(n, dtype=torch.int16).pin_memory()
    sa.copy(d, h, pdl=pdl, src_ready=ready)
    sa.copy(back, d, pdl=pdl)
    torch.cuda.synchronize()
    assert torch.equal(d.cpu(), h) and torch.equal(back, h)


def test_copy_gemv_chain_in_graph(sa):
    """host x -> device -> LUT-GEMV (PDL) -> host y, captured once and replayed with new host
    inputs each time: every replay returns the oracle's y for that x."""
    q, N, K, g = 3, 2048, 1024, 128
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(8, 1))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    layer = sa.pack(signs.to(DEV), alpha.to(DEV), g)
    xh = torch.empty(K, dtype=torch.float16).pin_memory()
    yh = torch.empty(N, dtype=torch.float16).pin_memory()
    xd = torch.empty(K, dtype=torch.float16, device=DEV)
    yd = torch.empty(N, dtype=torch.float16, device=DEV)
    ws = sa.Workspace(DEV)
    ws.get(sa.workspace_bytes(layer, 1))
    s = torch.cuda.Stream(DEV)

    def step():
        sa.copy(xd, xh, pdl=True, src_ready=True, stream=s)
        sa.lut_gemm(xd.view(1, K), layer, out=yd.view(1, N), workspace=ws, pdl=True, stream=s)
        sa.copy(yh, yd, pdl=True, stream=s)

    xh.copy_(synth.gen_x(1, K, seed=1).view(-1))
    with torch.cuda.stream(s):
        step()
    s.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        step()
    for seed in (2, 3, 4):
        x = synth.gen_x(1, K, seed=seed)
        xh.copy_(x.view(-1))
        with torch.cuda.stream(s):
            gr.replay()
        s.synchronize()
        y_ref = oracle.gemm(x.numpy(), planes, exps, g)
        assert oracle.err_floor(yh.float().numpy().reshape(1, N), y_ref) <= 2e-3
