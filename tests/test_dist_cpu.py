"""World-size-2 gloo test of the N-shard + all-gather host logic (§8(e)) on CPU.

Each rank computes its row shard of y with the oracle (the GEMV itself needs a GPU), then
``dist.gather_output`` assembles y; the result must equal the unsharded oracle output exactly
(rows are independent), for M = 1 (flat gather) and M = 3 ([P][M][N/P] permute path)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_2406_05981_b200.dist import gather_output, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, N, K, g = 3, 96, 512, 128
        signs, alpha = synth.gen_layer(q, N, K, g, seed=synth.seed_for(3, 0))
        n0, n1 = shard_range(N, world, rank)
        planes, exps, _ = oracle.pack_canonical(signs[:, n0:n1].numpy(), alpha[:, n0:n1].numpy(), g)
        ok = []
        for M in (1, 3):
            x = synth.gen_x(M, K, seed=5 + M).numpy()
            y_loc = torch.from_numpy(oracle.to_fp16(oracle.gemm(x, planes, exps, g)).astype(np.float32))
            y = gather_output(y_loc, None)
            pf, ef, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), g)
            y_ref = oracle.to_fp16(oracle.gemm(x, pf, ef, g)).astype(np.float32)
            ok.append(bool(np.array_equal(y.numpy(), y_ref)) and tuple(y.shape) == (M, N))
        results[rank] = all(ok)
    finally:
        dist.destroy_process_group()


def test_shard_then_gather_equals_unsharded():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert dict(results) == {0: True, 1: True}


def test_shard_range():
    from paper_2406_05981_b200.dist import shard_range
    assert [shard_range(28672, 8, r) for r in (0, 7)] == [(0, 3584), (25088, 28672)]
    with pytest.raises(ValueError):
        shard_range(100, 8, 0)
