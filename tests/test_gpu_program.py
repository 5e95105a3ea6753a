"""GPU parity of the persistent decode program (kernel id 9, csrc/lut_program.cu,
shiftadd_lut_gemv_program) against the fp64 oracle (bar: reading R10, floor-normalised relative
error <= 2e-3 per output), through the C ABI:

* a mixed program -- fused q/k/v with 2/3-bit segments, a single-slice call (no split-K), ragged
  N, every q, K up to the LLaMA-2-7B down_proj -- with and without SHIFTADD_CALL_WAIT;
* a true chain: x of call j+1 IS the y buffer of call j (each call waits), compared with the
  oracle applied layer after layer on the fp16-rounded outputs;
* one full-size LLaMA-2-7B block (q/k/v fused, o, gate/up fused, down) at the synthetic 2.2-bit
  allocation's block-31 bit widths;
* repeated launches (launch counter, two partial regions by call parity) eagerly and from a CUDA
  graph with new inputs each time: every launch correct, reruns bit-identical."""

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


def _layer(sa, q, N, K, seed, std=0.02):
    signs, alpha = synth.gen_layer(q, N, K, 128, seed=seed, std=std)
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), 128)
    return sa.pack(signs.to(DEV), alpha.to(DEV), 128, layout=sa.LAYOUT_TILED), planes, exps


def _err(y, x, planes, exps):
    return oracle.err_floor(y.float().cpu().numpy().reshape(1, -1), oracle.gemm(x.reshape(1, -1), planes, exps, 128))


MIXED = [  # (K, [(q, N), ...], wait)
    (4096, [(2, 4096), (3, 4096), (2, 4096)], False),
    (256, [(3, 100), (1, 33)], True),              # S = 1: y stored by the consumers
    (11008, [(2, 4096)], True),
    (1024, [(4, 1000), (1, 40), (2, 17), (3, 513)], False),
    (4096, [(2, 11008), (3, 11008)], True),
    (2304, [(3, 777)], False),
]


@pytest.mark.parametrize("wait_all", [False, True])
def test_program_mixed_calls_parity(sa, wait_all):
    calls, refs = [], []
    for j, (K, segs, wait) in enumerate(MIXED):
        x = synth.gen_x(1, K, seed=synth.seed_for(9, j, K)).view(-1)
        cases = [_layer(sa, q, N, K, synth.seed_for(9, 10 * j + i, q)) for i, (q, N) in enumerate(segs)]
        outs = [torch.full((c[0].N,), float("nan"), dtype=torch.float16, device=DEV) for c in cases]
        calls.append((x.to(DEV), [c[0] for c in cases], outs, wait or wait_all))
        refs.append((x.numpy(), cases, outs))
    prog = sa.Program(calls)
    prog()
    torch.cuda.synchronize()
    for j, (x, cases, outs) in enumerate(refs):
        for (L, planes, exps), y in zip(cases, outs):
            err = _err(y, x, planes, exps)
            assert err <= TOL, (j, L.q, L.N, L.K, err)


def test_program_chain_reads_previous_outputs(sa):
    """x of call j+1 is the output buffer of call j (SHIFTADD_CALL_WAIT on every call): the
    dependency is real, and each output equals the oracle applied to the fp16 output of the
    previous call (the oracle's own chain, never the kernel's values)."""
    shapes = [(2, 4096, 4096), (3, 1024, 4096), (2, 2048, 1024), (3, 4096, 2048), (2, 512, 4096),
              (4, 4096, 512)]   # (q, N, K): N_j == K_{j+1}
    x0 = synth.gen_x(1, 4096, seed=synth.seed_for(9, 99)).view(-1)
    calls, cases = [], []
    x_dev = x0.to(DEV)
    for j, (q, N, K) in enumerate(shapes):
        # std 1/sqrt(K): unit gain per layer, so the chain stays in the fp16 normal range
        case = _layer(sa, q, N, K, synth.seed_for(9, 200 + j), std=K ** -0.5)
        y = torch.full((N,), float("nan"), dtype=torch.float16, device=DEV)
        calls.append((x_dev, [case[0]], [y], True))
        cases.append(case)
        x_dev = y
    sa.Program(calls)()
    torch.cuda.synchronize()
    x = x0.numpy().astype(np.float64)
    for j, ((L, planes, exps), (_, _, outs, _)) in enumerate(zip(cases, calls)):
        ref = oracle.gemm(x.reshape(1, -1), planes, exps, 128)
        y = outs[0].float().cpu().numpy().reshape(1, -1)
        err = oracle.err_floor(y, ref)
        assert err <= TOL, (j, err)
        x = oracle.to_fp16(ref).astype(np.float64).reshape(-1)   # the oracle's fp16 output feeds the next call


def test_program_full_llama_block(sa):
    """One LLaMA-2-7B decoder block at full size, block 31's bit widths (k and up at 3 bits)."""
    blk = [("qkv", 4096, [(2, 4096), (3, 4096), (2, 4096)]), ("o", 4096, [(2, 4096)]),
           ("gate_up", 4096, [(2, 11008), (3, 11008)]), ("down", 11008, [(2, 4096)])]
    calls, refs = [], []
    for j, (name, K, segs) in enumerate(blk):
        x = synth.gen_x(1, K, seed=synth.seed_for(9, 300 + j)).view(-1)
        cases = [_layer(sa, q, N, K, synth.seed_for(9, 310 + 10 * j + i)) for i, (q, N) in enumerate(segs)]
        outs = [torch.empty(c[0].N, dtype=torch.float16, device=DEV) for c in cases]
        calls.append((x.to(DEV), [c[0] for c in cases], outs, j > 0))
        refs.append((name, x.numpy(), cases, outs))
    sa.Program(calls)()
    torch.cuda.synchronize()
    for name, x, cases, outs in refs:
        for (L, planes, exps), y in zip(cases, outs):
            assert _err(y, x, planes, exps) <= TOL, (name, L.q, L.N)


def test_program_repeated_launches_eager_and_graph(sa):
    """Launch counter and partial-region parity across launches: new x every launch, all
    outputs correct; the same inputs give bit-identical outputs eagerly and from a graph."""
    K = 4096
    segs = [[(2, 4096), (3, 4096)], [(3, 2048)], [(2, 4096)]]
    xs = [torch.empty(K, dtype=torch.float16, device=DEV) for _ in segs]
    calls, cases_all = [], []
    for j, sg in enumerate(segs):
        cases = [_layer(sa, q, N, K, synth.seed_for(9, 400 + 10 * j + i)) for i, (q, N) in enumerate(sg)]
        outs = [torch.empty(c[0].N, dtype=torch.float16, device=DEV) for c in cases]
        calls.append((xs[j], [c[0] for c in cases], outs, j > 0))
        cases_all.append((cases, outs))
    prog = sa.Program(calls)
    first = None
    for it in range(4):
        hx = [synth.gen_x(1, K, seed=synth.seed_for(9, 500 + 10 * it + j)).view(-1) for j in range(len(segs))]
        for d, h in zip(xs, hx):
            d.copy_(h)
        prog()
        torch.cuda.synchronize()
        for j, (cases, outs) in enumerate(cases_all):
            for (L, planes, exps), y in zip(cases, outs):
                assert _err(y, hx[j].numpy(), planes, exps) <= TOL, (it, j, L.N)
        if it == 0:
            first = [[o.clone() for o in outs] for _, outs in cases_all]
            h0 = hx
    # graph replays of the first inputs: bit-identical to the eager first launch
    for d, h in zip(xs, h0):
        d.copy_(h)
    st = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        prog(stream=st)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        for (cases, outs), ref in zip(cases_all, first):
            for y, r in zip(outs, ref):
                assert torch.equal(y, r)


def test_chain_matches_individual_calls_bit_for_bit(sa):
    """shiftadd_lut_gemv_chain issues the same kernels as the per-call entry points: outputs are
    bit-identical to lut_gemm / lut_gemv_fused called one by one (and meet the oracle bar)."""
    calls, refs = [], []
    for j, (K, segs, _) in enumerate(MIXED):
        x = synth.gen_x(1, K, seed=synth.seed_for(9, 600 + j, K)).view(-1).to(DEV)
        cases = [_layer(sa, q, N, K, synth.seed_for(9, 610 + 10 * j + i, q)) for i, (q, N) in enumerate(segs)]
        outs = [torch.empty(c[0].N, dtype=torch.float16, device=DEV) for c in cases]
        calls.append((x, [c[0] for c in cases], outs, True))
        refs.append((x, cases))
    sa.Chain(calls)()
    torch.cuda.synchronize()
    for (x, cases), (_, _, outs, _) in zip(refs, calls):
        layers = [c[0] for c in cases]
        if len(layers) == 1:
            ind = [sa.lut_gemm(x, layers[0], pdl=True).view(-1)]
        else:
            ind = sa.lut_gemv_fused(x, layers, pdl=True)
        torch.cuda.synchronize()
        for (L, planes, exps), y, yi in zip(cases, outs, ind):
            assert torch.equal(y, yi), (L.N, L.K)
            assert _err(y, x.cpu().numpy(), planes, exps) <= TOL
