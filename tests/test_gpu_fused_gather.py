"""NEXT-f3: the fused all-gather epilogue (shiftadd_lut_gemv_gather + shiftadd_gather_wait)
with two ranks as two processes sharing cuda:0 -- their gathered buffers and flags are
mapped into each other through CUDA IPC, which is exactly the peer-store + flag protocol a
multi-GPU run uses over NVLink.  Every rank's gathered y must equal the oracle on the whole
(unsharded) layer, for several back-to-back calls (double buffering, epochs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, N, K, g, calls, out_q, graph, M=1):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2406_05981_b200 as sa
    from paper_2406_05981_b200 import dist as sdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(1, 60))
        n0, n1 = sdist.shard_range(N, world, rank)
        L = sa.pack(signs[:, n0:n1].contiguous().cuda(), alpha[:, n0:n1].contiguous().cuda(), g,
                    layout=sa.LAYOUT_TILED)
        layer = sdist.FusedGatherLinear(L, N, max_m=M)
        xs = [synth.gen_x(M, K, seed=70 + c).cuda() for c in range(calls)]
        outs = []
        if not graph:
            for c in range(calls):
                y = layer(xs[c], pdl=bool(c & 1))
                outs.append(y.clone())            # the view is reused two calls later
        else:
            # capture two calls (one per buffer) once, replay for every pair of inputs: the
            # epochs and buffer parity come from the device counter
            xin = torch.empty_like(xs[0])
            ys = [torch.empty(M * world * (N // world), dtype=torch.float16, device="cuda") for _ in range(2)]
            st = torch.cuda.Stream()
            torch.cuda.synchronize()
            gph = torch.cuda.CUDAGraph()
            xin2 = torch.empty_like(xs[0])
            with torch.cuda.graph(gph, stream=st):
                ys[0].copy_(layer(xin, pdl=True, stream=st).view(-1))
                ys[1].copy_(layer(xin2, pdl=True, stream=st).view(-1))
            for c in range(0, calls, 2):
                xin.copy_(xs[c])
                xin2.copy_(xs[c + 1])
                gph.replay()
                torch.cuda.synchronize()
                outs += [ys[0].clone().view(M, -1), ys[1].clone().view(M, -1)]
        torch.cuda.synchronize()
        out_q.put((rank, [o.cpu().numpy() for o in outs], None))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, None, repr(e)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


# K > 4096 shards (the LLaMA-2-70B down_proj / OPT-66B fc2 regime) run on the all-SM streaming
# kernel (8) with the same peer-store + flag protocol; K <= 4096 on the cluster kernel (3)
@pytest.mark.parametrize("q,N,K,graph", [(3, 4096, 4096, False), (2, 1536, 768, False), (3, 4096, 4096, True),
                                         (3, 2048, 9216, False), (2, 1024, 28672, True)])
def test_fused_gather_two_ranks_one_gpu(q, N, K, graph):
    _run_case(q, N, K, graph, 1)


# batch rows (M <= 8): the streaming kernel with M-wide LUT entries, gathered y [M][P n]
@pytest.mark.parametrize("q,N,K,graph,M", [(3, 2048, 4096, False, 3), (2, 1024, 9216, True, 5)])
def test_fused_gather_small_batch_two_ranks_one_gpu(q, N, K, graph, M):
    _run_case(q, N, K, graph, M)


def _run_case(q, N, K, graph, M):
    world, g, calls = 2, 128, 4
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, N, K, g, calls, out_q, graph, M))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, outs, err = out_q.get(timeout=300)
        assert err is None, (rank, err)
        res[rank] = outs
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(1, 60))
    planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
    for c in range(calls):
        x = synth.gen_x(M, K, seed=70 + c)
        ref = oracle.gemm(x.numpy(), planes, exps, g)
        for r in range(world):
            y = res[r][c].astype(np.float32).reshape(M, -1)
            assert oracle.err_floor(y, ref) <= 2e-3, (c, r)
        assert np.array_equal(res[0][c], res[1][c])      # every rank holds the same gathered y
