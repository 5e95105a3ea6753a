#!/usr/bin/env python
"""Benchmark of the ShiftAddLLM batch-1 LUT-GEMV hot path on B200 (one JSON line on rank 0).

Metric (BASELINE.json): "us/call & achieved HBM GB/s (vs ~8 TB/s) for batch-1 LUT-GEMV,
1/2/4/8 B200".  `value` is whole-job achieved GB/s of algorithmic bytes (packed planes +
int8 exponents + fp16 x + fp16 y); per-layer us/call are in `config.layers`.

Workload (N=1): BASELINE.json configs[1], the OPT-6.7B layer set -- attention 4096x4096 and
FC1 (N=16384, K=4096), each at 2 and 3 bits, g=128, batch 1.  One step = one LUT-GEMV call
per layer (4 launches: mixed 2/3-bit dispatch, §8 a6), weights resident in HBM in the
device-tiled layout, x resident.  L2 is defeated by rotating over R independent copies of the
layer set (R * set bytes >= 4 x L2).  Weights are synthetic greedy-BCQ layers (synth.py).

N>1 (torchrun): every layer is N-sharded by output rows over the ranks (column parallel);
a step is each rank's shard GEMV followed by an NCCL all-gather of y per layer; the timed
region is barrier + sync on both sides, device time max over ranks; value = full-layer
bytes / that time ("scaling": "strong" -- total work fixed).

--impl reference: the fp64 CPU oracle (oracle/, the test reference) timed on the host
cores on a bounded row sample of the same workload, same metric and unit.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
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
LAYERS = synth.opt_6p7b_layer_set()          # (name, N, K, q)
METRIC = "achieved HBM GB/s (algorithmic bytes) of batch-1 LUT-GEMV, OPT-6.7B layer set"
WORKLOAD = "OPT-6.7B layer set: attn 4096x4096 + FC1 16384x4096, q=2 and q=3, g=128, M=1"


def alg_bytes(M, q, N, K, g=G):
    return q * N * K // 8 + q * N * (K // g) + 2 * M * K + 2 * M * N


KERNEL_NAMES = {0: "gemm_generic_kernel", 1: "gemv_tiled_kernel (grid split-K)", 2: "gemm_tiled_mb_kernel",
                3: "gemv_cluster_ring_kernel (cluster split-K, TMA weight ring)",
                4: "gemv_stream_kernel (grid split-K, TMA weight ring)",
                5: "gemm_cluster_ring_m2_kernel (M = 2)", 6: "gemm_cluster_ring_m4_kernel (M = 3..4)",
                7: "gemm_cluster_ring_m2/m4 kernels (M > 4, row chunks)"}


def kernel_names(layers):
    """The kernel(s) the bench layers launch (shiftadd_gemm_plan kernel ids)."""
    import paper_2406_05981_b200 as sa
    ids = sorted({sa.gemm_plan(L, 1)[3] for L in layers})
    return " + ".join(KERNEL_NAMES[i] for i in ids)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clock sampling
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 50 ms while active."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.2)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        return len(self.lines)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self, start=0, end=None):
        rows = []
        for ln in self.lines[start:end]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:]))
            except ValueError:
                continue
        if not rows:
            rows_all = self.lines
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": "no nvidia-smi samples" if not rows_all else "no samples in window"}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, fl in rows for i, v in enumerate(fl) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ distributed helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ reference arm (oracle)
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    try:
        from threadpoolctl import threadpool_info
        blas_threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        blas_threads = None
    cores = len(os.sched_getaffinity(0))
    rows = 64

    def make(rows_):
        out = []
        for li, (name, N, K, q) in enumerate(LAYERS):
            signs, alpha = synth.gen_layer(q, rows_, K, G, seed=synth.seed_for(1, li))
            planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), G)
            x = synth.gen_x(1, K, seed=synth.seed_for(1, 100 + li)).numpy()
            out.append((x, planes, exps, q, rows_, K))
        return out

    def step(data):
        nbytes = 0
        for x, planes, exps, q, n, K in data:
            oracle.gemm(x, planes, exps, G)
            nbytes += alg_bytes(1, q, n, K)
        return nbytes

    data = make(rows)
    t0 = time.perf_counter()
    step(data)
    t1 = time.perf_counter() - t0
    budget = 120.0
    if (args.steps + args.warmup) * t1 > budget:
        rows = max(16, int(rows * budget / ((args.steps + args.warmup) * t1)) // 16 * 16)
        data = make(rows)
    for _ in range(args.warmup):
        step(data)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        total += step(data)
    dt = time.perf_counter() - t0
    val = total / dt / 1e9
    sample = "%d output rows of each of the 4 layers per step (fp64 numpy dequant + matvec)" % rows
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": cores, "blas_threads": blas_threads,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(seconds=12.0):
    """The oracle as it stands on the host cores, bounded sample (~seconds of work)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info
        blas_threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        blas_threads = None
    rows = 256
    data = []
    for li, (name, N, K, q) in enumerate(LAYERS):
        signs, alpha = synth.gen_layer(q, rows, K, G, seed=synth.seed_for(1, li))
        planes, exps, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), G)
        x = synth.gen_x(1, K, seed=synth.seed_for(1, 100 + li)).numpy()
        data.append((x, planes, exps, q, rows, K))
    total = 0
    passes = 0
    t0 = time.perf_counter()
    while True:
        for x, planes, exps, q, n, K in data:
            oracle.gemm(x, planes, exps, G)
            total += alg_bytes(1, q, n, K)
        passes += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": round(total / dt / 1e9, 4), "unit": "GB/s", "cores": cores, "blas_threads": blas_threads,
            "kind": "oracle",
            "sample": "%d passes over %d output rows of each of the 4 layers (fp64 numpy dequant + matvec), %.1f s"
                      % (passes, rows, dt)}


# ------------------------------------------------------------------ product arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="shiftadd", choices=["shiftadd", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: NCCL all_gather_into_tensor after each GEMV, or the fused-gather "
                         "epilogue (NEXT-f3: peer stores over CUDA IPC/NVLink + flag wait)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import paper_2406_05981_b200 as sa
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit("--gpus %d but WORLD_SIZE %d" % (args.gpus, ws))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    sa.lib()
    stream = torch.cuda.Stream(dev)
    pdl = not args.no_pdl
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size

    # ---- per-rank shards of every layer, R rotating copies (each > 4 x L2 in total)
    shard = []
    for (name, N, K, q) in LAYERS:
        n_loc = N // ws
        shard.append((name, N, K, q, n_loc, rank * n_loc))
    set_bytes = sum(alg_bytes(1, q, n, K) for (_, _, K, q, n, _) in shard)
    R = max(2, -(-4 * l2 // set_bytes))
    copies = []
    with torch.cuda.stream(stream):
        for r in range(R):
            cur = []
            for li, (name, N, K, q, n_loc, n0) in enumerate(shard):
                signs, alpha = synth.gen_layer(q, n_loc, K, G, seed=synth.seed_for(1, li, 7919 * r + rank),
                                               device=dev)
                cur.append(sa.pack(signs, alpha, G, layout=sa.LAYOUT_TILED, stream=stream))
                del signs, alpha
            copies.append(cur)
        xs = [synth.gen_x(1, K, seed=synth.seed_for(1, 100 + li), device=dev)
              for li, (_, _, K, _, _, _) in enumerate(shard)]
        ys = [torch.empty((1, n_loc), dtype=torch.float16, device=dev) for (_, _, _, _, n_loc, _) in shard]
        yfull = [torch.empty((ws, n_loc), dtype=torch.float16, device=dev) for (_, _, _, _, n_loc, _) in shard]
        wsp = sa.Workspace(dev)
        wsp.get(max(sa.workspace_bytes(L, 1) for L in copies[0]))
    stream.synchronize()

    fused = None
    if group is not None and args.gather == "fused":
        from paper_2406_05981_b200.dist import FusedGatherLinear
        fused = [FusedGatherLinear(copies[0][li], N, group=group) for li, (_, N, _, _, _, _) in enumerate(shard)]

    def step(t):
        cur = copies[t % R]
        for li in range(len(shard)):
            if fused is not None:
                fused[li](xs[li], pdl=pdl, stream=stream, layer=cur[li])
                continue
            sa.lut_gemm(xs[li], cur[li], out=ys[li], workspace=wsp, pdl=pdl)
            if group is not None:
                torch.distributed.all_gather_into_tensor(yfull[li], ys[li], group=group)

    # CUDA graphs: one graph holds a full rotation (R steps = 4R GEMV launches with PDL edges
    # between consecutive kernels), plus one single-step graph per copy for a remainder, so
    # neither the host launch rate nor per-graph launch gaps limit the device.
    with torch.cuda.stream(stream):
        for t in range(3):
            step(t)
    stream.synchronize()
    g_round = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_round, stream=stream):
        for r in range(R):
            step(r)
    singles = []
    for r in range(R):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            step(r)
        singles.append(gr)
    stream.synchronize()

    def run_steps(k):
        """Exactly k steps: k // R full rotations, then k % R single steps."""
        for _ in range(k // R):
            g_round.replay()
        for t in range(k % R):
            singles[t].replay()

    # ---- timed region: barrier + sync, K steps with CUDA events on the launch stream
    def barrier():
        if group is not None:
            torch.distributed.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            run_steps(args.warmup)
        barrier()
        m0 = clk.mark()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            run_steps(args.steps)
            ev1.record(stream)
        barrier()
        m1 = clk.mark()
        ms = ev0.elapsed_time(ev1)
        clocks = clk.summary(m0, m1)
        if clocks.get("samples", 0) == 0:
            clocks = clk.summary()
            clocks["window"] = "whole bench run (timed region shorter than the 50 ms sample period)"
    t_dev = torch.tensor([ms], dtype=torch.float64, device=dev)
    if group is not None:
        torch.distributed.all_reduce(t_dev, op=torch.distributed.ReduceOp.MAX, group=group)
    ms = float(t_dev.item())
    full_bytes = sum(alg_bytes(1, q, N, K) for (_, N, K, q) in LAYERS)
    value = full_bytes * args.steps / (ms * 1e-3) / 1e9

    # ---- per-layer us/call and the dominant kernel's roofline (GEMV-only, this rank)
    per_layer = []
    kern_bytes = 0
    kern_ms = 0.0
    reps = 200
    for li, (name, N, K, q, n_loc, n0) in enumerate(shard):
        gl = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gl, stream=stream):
            for t in range(reps):
                sa.lut_gemm(xs[li], copies[t % R][li], out=ys[li], workspace=wsp, pdl=pdl)
        with torch.cuda.stream(stream):
            gl.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gl.replay()
            e1.record(stream)
        stream.synchronize()
        lm = e0.elapsed_time(e1) / reps
        del gl
        b = alg_bytes(1, q, n_loc, K)
        kern_bytes += b
        kern_ms += lm
        per_layer.append({"layer": name, "N": n_loc, "K": K, "q": q, "us_per_call": round(lm * 1e3, 3),
                          "GBps": round(b / (lm * 1e-3) / 1e9, 1),
                          "plane_GBps": round(q * n_loc * K / 8 / (lm * 1e-3) / 1e9, 1)})
    peak, peak_src = load_peaks()
    achieved = kern_bytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("traffic_bytes_per_launch_avg")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                "kernel": kernel_names(copies[0]),
                "algorithmic_bytes_per_launch_avg": kern_bytes // len(shard),
                "how": "per layer: CUDA events around one replay of a graph of %d back-to-back launches "
                       "(rotating copies) on the launch stream; achieved = sum bytes / sum times" % reps}

    # ---- e2e through the public API with host buffers.  Every step copies that step's inputs
    # (the four layers' x, one pinned host buffer) host -> device, runs the four GEMVs (plus
    # the all-gathers when N > 1) and reads the four outputs back device -> host (one pinned
    # buffer).  With N = 1 the steps are replayed from a CUDA graph (R steps per graph, the
    # copies inside it), as a serving loop would issue them; with N > 1 they are issued eagerly.
    Ks = [K for (_, _, K, _, _, _) in shard]
    Nf = [N for (_, N, _, _) in LAYERS]
    xoff = [0]
    for K in Ks:
        xoff.append(xoff[-1] + K)
    yoff = [0]
    for N in Nf:
        yoff.append(yoff[-1] + N)
    xh_all = torch.cat([x.reshape(-1).cpu() for x in xs]).pin_memory()
    yh_all = torch.empty(yoff[-1], dtype=torch.float16).pin_memory()
    with torch.cuda.stream(stream):
        xd_all = torch.empty(xoff[-1], dtype=torch.float16, device=dev)
        yd_all = torch.empty(yoff[-1], dtype=torch.float16, device=dev)
    torch.cuda.synchronize(dev)

    def e2e_step(t):
        cur = copies[t % R]
        # the step's inputs host -> device and outputs device -> host by shiftadd_copy (a kernel
        # reading / writing the pinned buffers over PCIe inside the PDL chain; copy-engine
        # memcpy nodes cost ~10 us of latency each for these kilobytes)
        sa.copy(xd_all, xh_all, pdl=pdl, src_ready=True, stream=stream)
        for li in range(len(shard)):
            xv = xd_all[xoff[li]:xoff[li + 1]].view(1, -1)
            yv = yd_all[yoff[li]:yoff[li + 1]].view(1, -1)
            if fused is not None:
                yv.copy_(fused[li](xv, stream=stream, layer=cur[li]))
            elif group is not None:
                sa.lut_gemm(xv, cur[li], out=ys[li], workspace=wsp, pdl=pdl)
                torch.distributed.all_gather_into_tensor(yv.view(-1), ys[li].view(-1), group=group)
            else:
                sa.lut_gemm(xv, cur[li], out=yv, workspace=wsp, pdl=pdl)
        sa.copy(yh_all, yd_all, pdl=pdl, stream=stream)

    e2e_rounds = max(2, min(args.steps, 500) // R)
    e2e_steps = e2e_rounds * R
    with torch.cuda.stream(stream):
        for t in range(3):
            e2e_step(t)
    stream.synchronize()
    g_e2e = None
    if group is None:
        g_e2e = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_e2e, stream=stream):
            for t in range(R):
                e2e_step(t)
        with torch.cuda.stream(stream):
            g_e2e.replay()
        stream.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for r_ in range(e2e_rounds):
            if g_e2e is not None:
                g_e2e.replay()
            else:
                for t in range(R):
                    e2e_step(t)
        e1.record(stream)
    barrier()
    # the last step's outputs really arrived on the host
    assert torch.isfinite(yh_all.float()).all()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if group is not None:
        torch.distributed.all_reduce(e2e_ms, op=torch.distributed.ReduceOp.MAX, group=group)
    e2e_val = full_bytes * e2e_steps / (float(e2e_ms.item()) * 1e-3) / 1e9
    h2d = xh_all.numel() * xh_all.element_size()
    d2h = yh_all.numel() * yh_all.element_size()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8 keys, fp32 LUT/accumulate, fp16 in/out",
            "data": "synthetic greedy-BCQ layers (synth.py), random activations with outlier channels",
            "config": {"workload": WORKLOAD, "layers": per_layer, "rotating_copies": R,
                       "l2_defeat": "inputs larger than L2: %d rotating copies, %.0f MB per rank" %
                                    (R, R * set_bytes / 1e6),
                       "parallelism": "N-shard x%d + NCCL all-gather" % ws if ws > 1 else "single GPU",
                       "pdl": pdl, "us_per_call_avg": round(ms / args.steps / len(LAYERS) * 1e3, 3)},
            "roofline": roofline,
            "clocks": clocks,
            "gpu_launches": args.steps * len(LAYERS),
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps},
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg()
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
