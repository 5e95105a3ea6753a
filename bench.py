#!/usr/bin/env python
"""Benchmark of the ShiftAddLLM batch-1 LUT-GEMV hot path on B200 (one JSON line on rank 0).

Metric (BASELINE.json): "us/call & achieved HBM GB/s (vs ~8 TB/s) for batch-1 LUT-GEMV,
1/2/4/8 B200".  `value` is whole-job achieved GB/s of algorithmic bytes (packed planes +
int8 exponents + fp16 x + fp16 y) over a decode step; the per-layer us/call
and roofline fractions (algorithmic and plane bytes) are in `config.layers`.

Workload (N=1): BASELINE.json configs[2] (north_star's target) --
all 224 LLaMA-2-7B decoder projections (32 blocks x q,k,v,o 4096x4096; gate,up 11008x4096;
down 4096x11008) at the synthetic Eq. 4 allocation with a 2.2-bit budget (synth.llama2_7b_
allocation: every k_proj and the up_proj of blocks 20-31 at 3 bits, the rest at 2), g = 128,
batch 1.  A step = one token: the projections are issued in model order as a serving loop
issues them, the ones that read the same activations fused into one launch -- q/k/v
(mixed 2/3-bit: shiftadd_lut_gemv_fused), o, gate/up (same bit width: one concatenated packed
layer through shiftadd_lut_gemm; mixed: shiftadd_lut_gemv_fused), down -- 128 launches per
token, stream-ordered with PDL.  The model's 1.87 GB of packed weights (>> the 126 MB L2) are
resident in HBM in the device-tiled layout; every step reads all of them once, so the L2 is
defeated by the working set itself.  Weights are synthetic greedy-BCQ layers (synth.py),
activations N(0,1) with outlier channels.

Per-layer rows: every LLaMA-2-7B projection shape and fusion of the step, the LLaMA-2-70B MLP
(configs[3], 3-bit, one GPU) and the OPT-6.7B layer set (configs[1]), each timed as a CUDA
graph of back-to-back calls over R >= ceil(4 L2 / layer bytes) rotating weight copies.

N>1 (torchrun): every projection is N-sharded by output rows (column parallel); each launch
is followed by an NCCL all-gather of its outputs; device time max over ranks ("strong":
total work fixed).

--impl reference: the fp64 CPU oracle (oracle/, the test reference) timed on the host cores
on a bounded row sample of the same workload, same metric and unit.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

G = 128
METRIC = "µs/call & achieved HBM GB/s (vs ~8 TB/s) for batch-1 LUT-GEMV, 1/2/4/8 B200"
WORKLOAD = ("LLaMA-2-7B decode step (BASELINE configs[2]): 224 projections, synthetic Eq.4 2.2-bit "
            "allocation (2/3-bit), g=128, M=1, 128 launches/token (q/k/v and gate/up fused)")
SHARE = {"q_proj": "attn_in", "k_proj": "attn_in", "v_proj": "attn_in", "gate_proj": "mlp_in", "up_proj": "mlp_in"}


def alg_bytes(M, q, N, K, g=G):
    return q * N * K // 8 + q * N * (K // g) + 2 * M * K + 2 * M * N


def plane_bytes(q, N, K):
    return q * N * K // 8


KERNEL_NAMES = {0: "gemm_generic_kernel", 1: "gemv_tiled_kernel (grid split-K)", 2: "gemm_tiled_mb_kernel",
                3: "gemv_cluster_ring_kernel (cluster split-K, TMA weight ring)",
                4: "gemv_stream_kernel (grid split-K, TMA weight ring)",
                5: "gemm_cluster_ring_m2_kernel (M = 2)", 6: "gemm_cluster_ring_m4_kernel (M = 3..4)",
                7: "gemm_cluster_ring_m2/m4 kernels (M > 4, row chunks)",
                8: "lut_stream_kernel (all-SM streaming, epoch split-K)",
                9: "lut_program_kernel (persistent decode program)",
                10: "gemv_cluster_fused_kernel (fused segments, cluster split-K, TMA weight ring)"}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clock sampling (NVML)
class ClockSampler:
    """SM clocks and throttle reasons sampled every 5 ms through NVML while active; `mark()`
    brackets windows (the timed region)."""
    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
             "sw_power_cap": 0x4}

    def __init__(self, index=0, period=0.005):
        self.index, self.period = index, period
        self.rows = []
        self.stop = threading.Event()
        self.thread = None
        self.err = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = reasons(h)
                        self.rows.append((time.perf_counter(), sm, rs))
                    except Exception as e:  # pragma: no cover
                        self.err = repr(e)
                    time.sleep(self.period)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception as e:
            self.err = repr(e)
        return self

    def mark(self):
        return time.perf_counter()

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self, t0=None, t1=None):
        rows = [r for r in self.rows if (t0 is None or r[0] >= t0) and (t1 is None or r[0] <= t1)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [], "samples": 0,
                    "note": self.err or "no samples in window"}
        reasons = sorted({n for _, _, rs in rows for n, bit in self.NAMES.items() if rs & bit})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(rows), "source": "NVML, 5 ms period"}


# ------------------------------------------------------------------ distributed helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ the oracle legs
def _oracle_sample(rows):
    """One block's 7 projections (block 31's bit widths: k and up at 3 bits), `rows` output
    rows each, canonical bytes packed by the oracle."""
    import oracle
    qs = synth.llama2_7b_allocation()
    out = []
    for li, (blk, name, N, K) in enumerate(synth.llama2_7b_layers()):
        if blk != 31:
            continue
        q = qs[li]
        signs, alpha = synth.gen_layer(q, rows, K, G, seed=synth.seed_for(2, li))
        planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), G)
        x = synth.gen_x(1, K, seed=synth.seed_for(2, 1000 + li)).numpy()
        out.append((name, x, planes, exps, q, rows, K, signs, alpha))
    return out


def _oracle_pass(data):
    import oracle
    nbytes = 0
    for _, x, planes, exps, q, n, K, _, _ in data:
        oracle.gemm(x, planes, exps, G)
        nbytes += alg_bytes(1, q, n, K)
    return nbytes


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores, on the bench's metric."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = len(os.sched_getaffinity(0))
    rows = 64
    data = _oracle_sample(rows)
    t0 = time.perf_counter()
    _oracle_pass(data)
    t1 = time.perf_counter() - t0
    budget = 120.0
    if (args.steps + args.warmup) * t1 > budget:
        rows = max(16, int(rows * budget / ((args.steps + args.warmup) * t1)) // 16 * 16)
        data = _oracle_sample(rows)
    for _ in range(args.warmup):
        _oracle_pass(data)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        total += _oracle_pass(data)
    dt = time.perf_counter() - t0
    val = total / dt / 1e9
    sample = ("%d output rows of each of the 7 projections of LLaMA-2-7B block 31 per step "
              "(fp64 numpy dequant + matvec)" % rows)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": cores, "blas_threads": _blas_threads(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(sa, dev, seconds=12.0):
    """The oracle as it stands on the host cores on a bounded sample (~seconds of work), once
    with the BLAS thread pool and once single-threaded; plus the parity error of the CUDA path
    on the same sample rows (the sampled layers packed on the device, rows compared one by one)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    rows = 256
    data = _oracle_sample(rows)
    total, passes = 0, 0
    t0 = time.perf_counter()
    while True:
        total += _oracle_pass(data)
        passes += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    single = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            t1 = time.perf_counter()
            nb = _oracle_pass(data)
            single = round(nb / (time.perf_counter() - t1) / 1e9, 5)
    except Exception:
        pass
    # parity of the CUDA path on the sampled rows (same synthetic generator and seeds)
    errs = {}
    for name, x, planes, exps, q, n, K, signs, alpha in data:
        L = sa.pack(signs.to(dev), alpha.to(dev), G, layout=sa.LAYOUT_TILED)
        y = sa.lut_gemm(torch.from_numpy(x).to(dev), L).float().cpu().numpy()
        errs[name] = float(oracle.err_floor(y, oracle.gemm(x, planes, exps, G)))
    return {"value": round(total / dt / 1e9, 5), "unit": "GB/s", "cores": cores, "blas_threads": _blas_threads(),
            "single_thread_value": single, "kind": "oracle",
            "sample": "%d passes over %d output rows of each of the 7 projections of LLaMA-2-7B block 31 "
                      "(fp64 numpy dequant + matvec), %.1f s" % (passes, rows, dt),
            "parity_err_floor_max": max(errs.values()), "parity_err_floor": errs}


# ------------------------------------------------------------------ the decode step
class Launch:
    """One launch of the step: a packed layer (lut_gemm) or fused segments (lut_gemv_fused)."""

    def __init__(self, sa, kind, K, layers, outs, x, names):
        self.sa, self.kind, self.K, self.layers, self.outs, self.x, self.names = sa, kind, K, layers, outs, x, names

    def __call__(self, ws, pdl, x=None):
        x = self.x if x is None else x
        if self.kind == "gemm":
            self.sa.lut_gemm(x.view(1, -1), self.layers[0], out=self.outs[0].view(1, -1), workspace=ws, pdl=pdl)
        else:
            self.sa.lut_gemv_fused(x.view(-1), self.layers, outs=self.outs, workspace=ws, pdl=pdl)

    def kernel(self):
        # fused segments: the cluster TMA ring (kernel 10) for K <= 4096, else the streaming kernel
        if self.kind == "gemm":
            return self.sa.gemm_plan(self.layers[0], 1)[3]
        return 10 if self.K <= 4096 and self.plane_bytes() <= 24e6 else 8

    def alg_bytes(self):
        return sum(plane_bytes(L.q, L.N, L.K) + L.q * L.N * (L.K // G) + 2 * L.N for L in self.layers) + 2 * self.K

    def plane_bytes(self):
        return sum(plane_bytes(L.q, L.N, L.K) for L in self.layers)


def build_step(sa, dev, ws_size, rank):
    """The 128 launches of one LLaMA-2-7B token (this rank's row shards)."""
    layers = synth.llama2_7b_layers()
    qs = synth.llama2_7b_allocation()
    blocks = {}
    for li, ((blk, name, N, K), q) in enumerate(zip(layers, qs)):
        blocks.setdefault(blk, []).append((li, name, N, K, q))
    launches = []
    for blk in sorted(blocks):
        groups, order = {}, []
        for li, name, N, K, q in blocks[blk]:
            key = SHARE.get(name, name)
            if key not in groups:
                groups[key] = []
                order.append(key)
            groups[key].append((li, name, N, K, q))
        for key in order:
            members = groups[key]
            K = members[0][3]
            x = synth.gen_x(1, K, seed=synth.seed_for(2, 5000 + 10 * blk + len(launches)), device=dev).view(-1)
            gen = []
            for li, name, N, _, q in members:
                n_loc = N // ws_size
                signs, alpha = synth.gen_layer(q, n_loc, K, G, seed=synth.seed_for(2, li, rank), device=dev)
                gen.append((name, q, n_loc, signs, alpha))
            qset = {q for _, q, _, _, _ in gen}
            if len(gen) == 1 or len(qset) == 1:
                signs = torch.cat([s for _, _, _, s, _ in gen], dim=1)
                alpha = torch.cat([a for _, _, _, _, a in gen], dim=1)
                L = sa.pack(signs, alpha, G, layout=sa.LAYOUT_TILED)
                out = torch.empty(L.N, dtype=torch.float16, device=dev)
                launches.append(Launch(sa, "gemm", K, [L], [out], x, [g[0] for g in gen]))
            else:
                Ls = [sa.pack(s, a, G, layout=sa.LAYOUT_TILED) for _, _, _, s, a in gen]
                outs = [torch.empty(L.N, dtype=torch.float16, device=dev) for L in Ls]
                launches.append(Launch(sa, "fused", K, Ls, outs, x, [g[0] for g in gen]))
            del gen
    return launches


def graph_time_us(fn, reps, stream):
    """Device time of one call of fn, from CUDA events around a replay of a graph of `reps`
    back-to-back calls on `stream` (after a warm replay)."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for t in range(reps):
            fn(t)
    with torch.cuda.stream(stream):
        g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
    stream.synchronize()
    del g
    return e0.elapsed_time(e1) * 1e3 / reps


# per-layer rows: (label, [(N, q), ...] segments sharing x, K, fused_kind)
LAYER_ROWS = [
    ("llama7b q/v/o 4096x4096 q2", [(4096, 2)], 4096, "gemm"),
    ("llama7b k 4096x4096 q3", [(4096, 3)], 4096, "gemm"),
    ("llama7b qkv fused (q2,q3,q2)", [(4096, 2), (4096, 3), (4096, 2)], 4096, "fused"),
    ("llama7b gate/up 11008x4096 q2", [(11008, 2)], 4096, "gemm"),
    ("llama7b up 11008x4096 q3", [(11008, 3)], 4096, "gemm"),
    ("llama7b gate_up concat 22016x4096 q2", [(22016, 2)], 4096, "gemm"),
    ("llama7b gate_up fused (q2,q3)", [(11008, 2), (11008, 3)], 4096, "fused"),
    ("llama7b down 4096x11008 q2", [(4096, 2)], 11008, "gemm"),
    ("llama70b gate/up 28672x8192 q3", [(28672, 3)], 8192, "gemm"),
    ("llama70b down 8192x28672 q3", [(8192, 3)], 28672, "gemm"),
    ("opt6.7b attn 4096x4096 q2", [(4096, 2)], 4096, "gemm"),
    ("opt6.7b attn 4096x4096 q3", [(4096, 3)], 4096, "gemm"),
    ("opt6.7b fc1 16384x4096 q2", [(16384, 2)], 4096, "gemm"),
    ("opt6.7b fc1 16384x4096 q3", [(16384, 3)], 4096, "gemm"),
]


def time_layer_row(sa, dev, stream, ws, l2, peak, label, segs, K, kind, ws_size):
    segs = [(N // ws_size, q) for N, q in segs]
    lb = sum(alg_bytes(1, q, N, K) for N, q in segs) - 2 * K * (len(segs) - 1)
    R = max(2, -(-4 * l2 // lb))
    base = []
    for r in range(2):
        base.append([sa.pack(*synth.gen_layer(q, N, K, G, seed=synth.seed_for(2, 9000 + N + q, r), device=dev),
                             G, layout=sa.LAYOUT_TILED) for N, q in segs])
    copies = []
    for r in range(R):
        b = base[r % 2]
        copies.append(b if r < 2 else [sa.PackedLayer(L.planes.clone(), L.exps.clone(), L.q, L.N, L.K, L.g,
                                                      L.layout, L.counts) for L in b])
    x = synth.gen_x(1, K, seed=synth.seed_for(2, 9999), device=dev).view(-1)
    outs = [torch.empty(N, dtype=torch.float16, device=dev) for N, _ in segs]
    torch.cuda.synchronize(dev)
    if kind == "gemm":
        def fn(t):
            sa.lut_gemm(x.view(1, -1), copies[t % R][0], out=outs[0].view(1, -1), workspace=ws, pdl=True)
        kid = sa.gemm_plan(copies[0][0], 1)[3]
    else:
        def fn(t):
            sa.lut_gemv_fused(x, copies[t % R], outs=outs, workspace=ws, pdl=True)
        kid = 10 if K <= 4096 and sum(plane_bytes(q, N, K) for N, q in segs) <= 24e6 else 8
    with torch.cuda.stream(stream):
        for t in range(3):
            fn(t)
    stream.synchronize()
    us = graph_time_us(fn, max(R, 60), stream)
    pb = sum(plane_bytes(q, N, K) for N, q in segs)
    del copies, base
    torch.cuda.empty_cache()
    return {"layer": label, "segments": [{"N": N, "q": q} for N, q in segs], "K": K, "kernel": kid,
            "us_per_call": round(us, 3), "GBps": round(lb / us * 1e-3, 1), "plane_GBps": round(pb / us * 1e-3, 1),
            "frac": round(lb / us * 1e-3 / peak, 4), "plane_frac": round(pb / us * 1e-3 / peak, 4),
            "rotating_copies": R, "l2_defeat": "R x %.1f MB = %.0f MB > 4 x L2" % (lb / 1e6, R * lb / 1e6)}


def fused_gather_row(sa, sdist, dev, stream, group, ws_size, rank, peak, short):
    """NEXT-f3 at N > 1: this rank's shard of the LLaMA-2-70B down_proj (8192 x 28672, 3-bit,
    configs[3]) through FusedGatherLinear -- the GEMV's owner CTAs store y into every rank's
    gathered buffer, a flag wait replaces the NCCL all-gather -- timed as a graph of back-to-back
    calls (each followed by its wait), max over ranks."""
    N, K, q = 8192, 28672, 3
    n = N // ws_size
    signs, alpha = synth.gen_layer(q, n, K, G, seed=synth.seed_for(3, 2, rank), device=dev)
    layer = sdist.FusedGatherLinear(sa.pack(signs, alpha, G, layout=sa.LAYOUT_TILED), N, group)
    del signs, alpha
    x = synth.gen_x(1, K, seed=synth.seed_for(3, 3), device=dev).view(-1)
    reps = 4 if short else 40
    with torch.cuda.stream(stream):
        for _ in range(4):
            y = layer(x, pdl=True, stream=stream)
    stream.synchronize()
    ok = bool(torch.isfinite(y.float()).all())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            layer(x, pdl=True, stream=stream)
    with torch.cuda.stream(stream):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
    stream.synchronize()
    us = torch.tensor([e0.elapsed_time(e1) * 1e3 / reps], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(us, op=torch.distributed.ReduceOp.MAX, group=group)
    us = float(us.item())
    b = alg_bytes(1, q, n, K)
    return {"layer": "llama70b down 8192x28672 q3, N-shard %d + fused gather" % ws_size, "K": K, "rows_per_rank": n,
            "us_per_call": round(us, 3), "GBps_per_rank": round(b / us * 1e-3, 1),
            "frac_per_rank": round(b / us * 1e-3 / peak, 4), "finite": ok,
            "how": "graph of %d calls (GEMV with peer-store epilogue + flag wait), max over ranks" % reps}


# ------------------------------------------------------------------ product arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="shiftadd", choices=["shiftadd", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-layers", action="store_true", help="skip the per-layer rows")
    ap.add_argument("--no-program", action="store_true", help="skip the persistent-program (kernel 9) row")
    ap.add_argument("--dry-run", action="store_true", help="N>1 plumbing only: build the shards, run 2 steps")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "fused"],
                    help="N>1: also time the LLaMA-2-70B down_proj shard with the all-gather fused into the "
                         "GEMV epilogue (peer stores + flags, NEXT-f3)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import paper_2406_05981_b200 as sa
    from paper_2406_05981_b200 import dist as sdist
    ws_size, rank, local = dist_env()
    if ws_size != args.gpus:
        raise SystemExit("--gpus %d but WORLD_SIZE %d" % (args.gpus, ws_size))
    ndev = torch.cuda.device_count()
    if ws_size > ndev and not args.dry_run:
        raise SystemExit("--gpus %d needs %d visible GPUs (%d visible); --dry-run shares them" % (ws_size, ws_size, ndev))
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    group = None
    backend = None
    if ws_size > 1:
        import torch.distributed as dist
        # one GPU per rank over NCCL; a dry run with fewer GPUs than ranks (the test boxes have
        # one) shares them and gathers through the host over gloo
        backend = "nccl" if ws_size <= ndev else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        group = dist.group.WORLD
    sa.lib()
    stream = torch.cuda.Stream(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    peak, peak_src = load_peaks()

    # ---- the model (this rank's shards), resident in HBM
    launches = build_step(sa, dev, ws_size, rank)
    wsp = sa.Workspace(dev)
    need = 0
    for Lc in launches:
        need = max(need, sa.workspace_bytes(Lc.layers[0], 1) if Lc.kind == "gemm" else sa.workspace_bytes_fused(Lc.layers))
    wsp.get(need)
    gathered = [[torch.empty(ws_size * o.numel(), dtype=torch.float16, device=dev) for o in Lc.outs]
                for Lc in launches] if group is not None else None
    torch.cuda.synchronize(dev)
    step_bytes_full = sum(Lc.alg_bytes() for Lc in launches) * ws_size - (ws_size - 1) * sum(2 * Lc.K for Lc in launches)
    step_planes_full = sum(Lc.plane_bytes() for Lc in launches) * ws_size

    def step(_t=0):
        for li, Lc in enumerate(launches):
            Lc(wsp, True)
            if group is not None:
                for o, gbuf in zip(Lc.outs, gathered[li]):
                    if backend == "gloo":
                        sdist.gather_output(o.view(1, -1), group, out=gbuf.view(1, -1))
                    else:
                        torch.distributed.all_gather_into_tensor(gbuf, o, group=group)

    with torch.cuda.stream(stream):
        for _ in range(2):
            step()
    stream.synchronize()
    fused_row = fused_gather_row(sa, sdist, dev, stream, group, ws_size, rank, peak, args.dry_run) \
        if group is not None and args.gather == "fused" else None
    if args.dry_run:
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": ws_size, "launches_per_step": len(launches),
                              "fused_gather": fused_row}), flush=True)
        if group is not None:
            torch.distributed.destroy_process_group()
        return 0

    # one CUDA graph per step (128 launches with PDL edges, plus the all-gathers when N > 1)
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step, stream=stream):
        step()
    stream.synchronize()

    def barrier():
        if group is not None:
            torch.distributed.barrier(device_ids=[local_dev])
        torch.cuda.synchronize(dev)

    with ClockSampler(local_dev) as clk:
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                g_step.replay()
        barrier()
        m0 = clk.mark()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                g_step.replay()
            ev1.record(stream)
        barrier()
        m1 = clk.mark()
        ms = ev0.elapsed_time(ev1)
        t_dev = torch.tensor([ms], dtype=torch.float64, device=dev)
        if group is not None:
            torch.distributed.all_reduce(t_dev, op=torch.distributed.ReduceOp.MAX, group=group)
        ms = float(t_dev.item())
        value = step_bytes_full * args.steps / (ms * 1e-3) / 1e9

        # ---- the dominant kernel of the step, timed live: a graph of exactly the step's
        # launches of that kernel, in step order, on the launch stream
        by_kernel = {}
        for Lc in launches:
            by_kernel.setdefault(Lc.kernel(), []).append(Lc)
        kern_rows = []
        for kid, ls in sorted(by_kernel.items()):
            def sub(_t, ls=ls):
                for Lc in ls:
                    Lc(wsp, True)
            us = graph_time_us(sub, 5, stream)
            b = sum(Lc.alg_bytes() for Lc in ls)
            pbk = sum(Lc.plane_bytes() for Lc in ls)
            kern_rows.append({"kernel": kid, "name": KERNEL_NAMES[kid], "launches_per_step": len(ls),
                              "us_per_launch": round(us / len(ls), 3), "us_per_step": round(us, 2),
                              "alg_bytes_per_launch": b // len(ls), "GBps": round(b / us * 1e-3, 1),
                              "plane_GBps": round(pbk / us * 1e-3, 1)})
        dom = max(kern_rows, key=lambda r: r["us_per_step"])

        # ---- the same step as ONE persistent launch (kernel 9, shiftadd_lut_gemv_program):
        # every call waits for the previous one's outputs, as the PDL chain does (N = 1 only)
        program_row = None
        if group is None and not args.no_program:
            prog = sa.Program([(Lc.x, Lc.layers, Lc.outs, j > 0) for j, Lc in enumerate(launches)])
            us_p = graph_time_us(lambda _t: prog(stream=stream), 20, stream)
            program_row = {"kernel": 9, "name": KERNEL_NAMES[9], "us_per_token": round(us_p, 2),
                           "GBps": round(step_bytes_full / us_p * 1e-3, 1),
                           "frac": round(step_bytes_full / us_p * 1e-3 / peak, 4),
                           "note": "one cooperative launch per token, calls ordered by a completion counter; "
                                   "slower than the 128-launch PDL chain (DESIGN.md §6, kernel 9)"}
            del prog

        # ---- per-layer rows (this rank's shard shapes)
        per_layer = []
        if not args.no_layers:
            for label, segs, K, kind in LAYER_ROWS:
                per_layer.append(time_layer_row(sa, dev, stream, wsp, l2, peak, label, segs, K, kind, ws_size))
        m2 = clk.mark()
        clocks = clk.summary(m0, m1)
        if clocks.get("samples", 0) < 3:
            clocks = clk.summary(m0, m2)
            clocks["window"] = "timed step region + the kernel/per-layer timing that follows it"
        else:
            clocks["window"] = "timed step region"

    # ---- roofline of the dominant kernel (algorithmic bytes per launch / live launch time)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("kernels", {}).get(str(dom["kernel"]))
    f_ghz = (clocks.get("sm_mhz") or 1965.0) / 1e3
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # co-roofs: shared-memory data path -- per 32 key bytes one lookup
    # wavefront + 0.25 (TMA write) + 0.25 (LDS.128 read) + 1/16 exponent reads -> 32/1.5625 B/clk/SM;
    # issue -- 4 warp-instructions/clk/SM at ~3.5 instructions per lookup wavefront of 32 key bytes
    smem_roof = sms * (32 / 1.5625) * f_ghz
    issue_roof = sms * 4 * 32 / 3.5 * f_ghz
    roofline = {"bound": "hbm", "achieved": dom["GBps"], "peak": peak, "unit": "GB/s",
                "frac": round(dom["GBps"] / peak, 4), "traffic": traffic, "peak_source": peak_src,
                "kernel": dom["name"], "kernel_id": dom["kernel"],
                "algorithmic_bytes_per_launch_avg": dom["alg_bytes_per_launch"],
                "plane_frac": round(dom["plane_GBps"] / peak, 4),
                "co_roofs": {"smem_data_path_GBps": round(smem_roof, 1), "issue_GBps": round(issue_roof, 1),
                             "binding": "hbm" if peak < min(smem_roof, issue_roof) else
                             ("smem" if smem_roof < issue_roof else "issue"),
                             "clock_ghz": f_ghz},
                "how": "CUDA events around a replay of a graph of exactly the step's launches of this kernel "
                       "(step order, PDL, launch stream); achieved = their algorithmic bytes / that time",
                "kernels": kern_rows}

    # ---- e2e through the public API with host buffers: every step copies that step's inputs
    # (the 128 activation vectors, one pinned buffer) host -> device and its outputs device ->
    # host, by shiftadd_copy kernels inside the PDL chain; replayed from a CUDA graph (N = 1).
    xs_off, ys_off = [0], [0]
    for Lc in launches:
        xs_off.append(xs_off[-1] + Lc.K)
        ys_off.append(ys_off[-1] + sum(o.numel() for o in Lc.outs))
    xh = torch.cat([Lc.x.cpu() for Lc in launches]).pin_memory()
    yh = torch.empty(ys_off[-1], dtype=torch.float16).pin_memory()
    xd = torch.empty(xs_off[-1], dtype=torch.float16, device=dev)
    yd = torch.empty(ys_off[-1], dtype=torch.float16, device=dev)
    torch.cuda.synchronize(dev)
    e2e_outs = []
    for li, Lc in enumerate(launches):
        o, parts = ys_off[li], []
        for y in Lc.outs:
            parts.append(yd[o:o + y.numel()])
            o += y.numel()
        e2e_outs.append(parts)

    def e2e_step():
        sa.copy(xd, xh, pdl=True, src_ready=True, stream=stream)
        for li, Lc in enumerate(launches):
            x = xd[xs_off[li]:xs_off[li + 1]]
            if Lc.kind == "gemm":
                sa.lut_gemm(x.view(1, -1), Lc.layers[0], out=e2e_outs[li][0].view(1, -1), workspace=wsp, pdl=True)
            else:
                sa.lut_gemv_fused(x, Lc.layers, outs=e2e_outs[li], workspace=wsp, pdl=True)
            if group is not None:
                for o, gbuf in zip(e2e_outs[li], gathered[li]):
                    torch.distributed.all_gather_into_tensor(gbuf, o, group=group)
        sa.copy(yh, yd, pdl=True, stream=stream)

    with torch.cuda.stream(stream):
        e2e_step()
    stream.synchronize()
    g_e2e = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_e2e, stream=stream):
        e2e_step()
    e2e_steps = max(20, min(args.steps, 200))
    with torch.cuda.stream(stream):
        for _ in range(3):
            g_e2e.replay()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(e2e_steps):
            g_e2e.replay()
        e1.record(stream)
    barrier()
    assert torch.isfinite(yh.float()).all()   # the last step's outputs reached the host
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if group is not None:
        torch.distributed.all_reduce(e2e_ms, op=torch.distributed.ReduceOp.MAX, group=group)
    e2e_val = step_bytes_full * e2e_steps / (float(e2e_ms.item()) * 1e-3) / 1e9
    # the same step issued eagerly every time (no graph), host cost included: (a) through the
    # per-projection Python API (130 ctypes calls per token), (b) through shiftadd_lut_gemv_chain
    # (3 C calls per token: copy in, the 128 launches from C, copy out); N = 1
    def eager_time(fn, n):
        with torch.cuda.stream(stream):
            fn()
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(n):
                fn()
        e1.record(stream)
        barrier()
        return (time.perf_counter() - t0) / n, e0.elapsed_time(e1) / n * 1e-3

    eager_wall, eager_dev = eager_time(e2e_step, 20)
    chain_wall = chain_dev = None
    if group is None:
        chain = sa.Chain([(xd[xs_off[li]:xs_off[li + 1]], Lc.layers, e2e_outs[li], True)
                          for li, Lc in enumerate(launches)])

        def chain_step():
            sa.copy(xd, xh, pdl=True, src_ready=True, stream=stream)
            chain(stream=stream)
            sa.copy(yh, yd, pdl=True, stream=stream)
        chain_wall, chain_dev = eager_time(chain_step, 50)

    if rank == 0:
        us_step = ms / args.steps * 1e3
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws_size, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "dtype_detail": "u8 key bytes index fp32 LUT entries, fp32 accumulate, fp16 x in / y out",
            "data": "synthetic greedy-BCQ layers (synth.py), random activations with outlier channels",
            "config": {"workload": WORKLOAD, "us_per_token": round(us_step, 2),
                       "us_per_call_avg": round(us_step / len(launches), 3), "launches_per_step": len(launches),
                       "bytes_per_step": step_bytes_full, "plane_bytes_per_step": step_planes_full,
                       "plane_GBps": round(step_planes_full * args.steps / (ms * 1e-3) / 1e9, 1),
                       "frac": round(value / peak, 4),
                       "plane_frac": round(step_planes_full * args.steps / (ms * 1e-3) / 1e9 / peak, 4),
                       "l2_defeat": "inputs larger than L2: the step reads all %.2f GB of resident weights "
                                    "once (L2 %d MB)" % (step_bytes_full / ws_size / 1e9, l2 >> 20),
                       "parallelism": ("N-shard x%d + NCCL all-gather per launch" % ws_size) if ws_size > 1
                       else "single GPU", "pdl": True, "persistent_program": program_row,
                       "fused_gather": fused_row, "layers": per_layer},
            "roofline": roofline,
            "clocks": clocks,
            "gpu_launches": args.steps * len(launches),
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": xh.numel() * 2,
                    "d2h_bytes_per_step": yh.numel() * 2, "steps": e2e_steps,
                    "how": "graph-replayed steps with the step's pinned host inputs copied in and outputs "
                           "copied out by shiftadd_copy kernels inside the PDL chain",
                    "eager": {"value": round(step_bytes_full / eager_dev / 1e9, 2), "unit": "GB/s",
                              "us_per_step": round(eager_dev * 1e6, 1), "wall_us_per_step": round(eager_wall * 1e6, 1),
                              "how": "the same step issued through the Python API each time (no graph): "
                                     "130 ctypes calls per token, CUDA events; wall = host clock"},
                    "eager_chain": None if chain_dev is None else {
                        "value": round(step_bytes_full / chain_dev / 1e9, 2), "unit": "GB/s",
                        "us_per_step": round(chain_dev * 1e6, 1), "wall_us_per_step": round(chain_wall * 1e6, 1),
                        "how": "no graph: copy in, shiftadd_lut_gemv_chain (the 128 launches issued from C), "
                               "copy out -- 3 API calls per token"}},
        }
        if ws_size == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg(sa, dev)
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
