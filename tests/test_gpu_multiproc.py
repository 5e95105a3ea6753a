"""§8(e) multi-GPU readiness on a one-GPU box: two ranks as two processes sharing cuda:0.

* ``ShardedLinear.from_full`` packs each rank's row shard and runs the real LUT-GEMV kernels;
  ``gather_output`` assembles y (under gloo the all-gather is staged through the host).  Every
  rank's gathered y must equal the oracle on the whole, unsharded layer -- M = 1 and M = 3,
  a cluster-kernel shape and a K > 8192 streaming-kernel shape.
* ``bench.py --gpus 2 --dry-run`` under torchrun: the N > 1 branch (shard construction, per-launch
  gathers) runs two steps and exits 0.

A run over NVLink uses the same code with NCCL and one GPU per rank; this pool's boxes have one
GPU, so only the process-level logic and the sharded kernels are exercised here."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(3, 1024, 4096), (3, 512, 9216)]   # (q, N, K): cluster kernel; K > 8192 -> streaming kernel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2406_05981_b200 import dist as sdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        res = []
        for ci, (q, N, K) in enumerate(CASES):
            signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(3, 70 + ci))
            lin = sdist.ShardedLinear.from_full(signs.cuda(), alpha.cuda(), 128)
            for M in (1, 3):
                x = synth.gen_x(M, K, seed=80 + M + ci).cuda()
                y = lin(x if M > 1 else x.view(-1), pdl=True)
                torch.cuda.synchronize()
                res.append(y.float().cpu().numpy().reshape(M, N))
        out_q.put((rank, res, None))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, None, repr(e)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_sharded_linear_two_ranks_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, ys, err = out_q.get(timeout=600)
        assert err is None, (rank, err)
        res[rank] = ys
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    k = 0
    for ci, (q, N, K) in enumerate(CASES):
        signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(3, 70 + ci))
        planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), 128)
        for M in (1, 3):
            x = synth.gen_x(M, K, seed=80 + M + ci)
            ref = oracle.gemm(x.numpy(), planes, exps, 128)
            for r in range(world):
                assert oracle.err_floor(res[r][k], ref) <= 2e-3, (q, N, K, M, r)
            assert np.array_equal(res[0][k], res[1][k])
            k += 1


def test_bench_dry_run_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3",
           "--gather", "fused"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert res.returncode == 0, (res.stdout + res.stderr)[-4000:]
    lines = [json.loads(s) for s in res.stdout.splitlines() if s.startswith("{")]
    assert lines and lines[-1]["dry_run"] and lines[-1]["n_gpus"] == 2
    assert lines[-1]["launches_per_step"] == 128
    fg = lines[-1]["fused_gather"]   # the 70B down_proj shard with the fused all-gather epilogue
    assert fg["finite"] and fg["rows_per_rank"] == 4096 and fg["us_per_call"] > 0
