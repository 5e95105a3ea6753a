"""Extra measurements for the other BASELINE.json configs (one JSON line each; dev tool).

  python tools/bench_extra.py [--only NAME ...] [--out profiles/r1_extra.jsonl]

  llama7b_decode   config 2: all 224 LLaMA-2-7B projections with the synthetic 2.2-bit Eq. 4
                   allocation (synth.llama2_7b_allocation), one batch-1 GEMV each, in model
                   order in one CUDA graph (PDL on): us per token and achieved GB/s.
  llama7b_decode_fused  config 2 with same-q q/k/v and gate/up fused by rows (shared x: one
                   LUT build and one launch per group), same bytes per token.
  llama7b_batch    config 2, M in {1,2,4,8,16}: one decoder block (7 projections), M rows.
  llama70b_mlp     config 3 on one GPU: gate/up/down 3-bit, us per call.
  opt66b_decode    config 4 on one GPU: 64 x 6 OPT-66B projections at q in {2,3}, us per token.
  config0          OPT-125M q_proj 768x768 3-bit.

Weights are synthetic greedy-BCQ layers generated on the device (synth.gen_layer), packed
with shiftadd_pack (tiled layout).  Model-sized working sets are far above L2.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

G = 128
PEAK = 6539.5   # MEASURED_PEAKS.json hbm_gbs on this pool


def alg(M, q, N, K):
    return q * N * K // 8 + q * N * (K // G) + 2 * M * K + 2 * M * N


def pack_layer(q, N, K, seed, dev):
    s, a = synth.gen_layer(q, N, K, G, seed=seed, device=dev)
    L = sa.pack(s, a, G, layout=sa.LAYOUT_TILED)
    del s, a
    return L


def time_graph(fn, reps=5):
    torch.cuda.synchronize()   # inputs were made on the default stream; fn runs on s
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us per replay


def llama7b_decode(dev, M=1):
    layers = synth.llama2_7b_layers()
    qs = synth.llama2_7b_allocation()
    packed = []
    nbytes = 0
    for i, ((blk, name, N, K), q) in enumerate(zip(layers, qs)):
        packed.append(pack_layer(q, N, K, synth.seed_for(2, i), dev))
        nbytes += alg(M, q, N, K)
    xs = {K: synth.gen_x(M, K, seed=5, device=dev) for K in (4096, 11008)}
    outs = [torch.empty((M, L.N), dtype=torch.float16, device=dev) for L in packed]
    ws = sa.Workspace(dev)
    ws.get(max(sa.workspace_bytes(L, M) for L in packed))

    def run():
        for L, o in zip(packed, outs):
            sa.lut_gemm(xs[L.K], L, out=o, workspace=ws, pdl=True)

    us = time_graph(run)
    avg_bits = sum(qs) / len(qs)
    return {"name": "llama7b_decode", "config": "LLaMA-2-7B 224 projections, synthetic Eq.4 allocation avg %.3f bits, "
            "g=128, M=%d" % (avg_bits, M), "us_per_token": round(us, 1), "GBps": round(nbytes / us * 1e-3, 1),
            "frac_of_peak": round(nbytes / us * 1e-3 / PEAK, 4), "bytes_per_token": nbytes,
            "us_per_call_avg": round(us / len(packed), 3)}


def llama7b_decode_fused(dev, M=1):
    """Config 2 with the usual fused projections: in every block the projections that read the
    same activations (q/k/v; gate/up) and got the same bit width are one packed layer with
    their rows concatenated (one LUT build and one launch for the group; y is split by views).
    Same bytes per token as llama7b_decode."""
    layers = synth.llama2_7b_layers()
    qs = synth.llama2_7b_allocation()
    share = {"q_proj": "attn_in", "k_proj": "attn_in", "v_proj": "attn_in", "gate_proj": "mlp_in", "up_proj": "mlp_in"}
    groups = {}
    order = []
    for i, ((blk, name, N, K), q) in enumerate(zip(layers, qs)):
        key = (blk, share.get(name, name), q, K)
        if key not in groups:
            groups[key] = 0
            order.append(key)
        groups[key] += N
    packed = []
    nbytes = 0
    for j, key in enumerate(order):
        blk, _, q, K = key
        N = groups[key]
        packed.append(pack_layer(q, N, K, synth.seed_for(2, 1000 + j), dev))
        nbytes += alg(M, q, N, K)
    xs = {K: synth.gen_x(M, K, seed=5, device=dev) for K in (4096, 11008)}
    outs = [torch.empty((M, L.N), dtype=torch.float16, device=dev) for L in packed]
    ws = sa.Workspace(dev)
    ws.get(max(sa.workspace_bytes(L, M) for L in packed))

    def run():
        for L, o in zip(packed, outs):
            sa.lut_gemm(xs[L.K], L, out=o, workspace=ws, pdl=True)

    us = time_graph(run)
    return {"name": "llama7b_decode_fused", "config": "LLaMA-2-7B 224 projections as %d launches (same-q q/k/v and "
            "gate/up fused by rows), synthetic Eq.4 allocation, g=128, M=%d" % (len(packed), M),
            "us_per_token": round(us, 1), "GBps": round(nbytes / us * 1e-3, 1),
            "frac_of_peak": round(nbytes / us * 1e-3 / PEAK, 4), "bytes_per_token": nbytes,
            "launches_per_token": len(packed)}


def llama7b_batch(dev):
    out = []
    blk = [(n, N, K) for (b, n, N, K) in synth.llama2_7b_layers() if b == 31]
    qs = [q for (b, n, N, K), q in zip(synth.llama2_7b_layers(), synth.llama2_7b_allocation()) if b == 31]
    # 8 rotating copies of the block so the working set exceeds L2
    copies = [[pack_layer(q, N, K, synth.seed_for(2, 900 + 10 * r + i), dev) for i, ((n, N, K), q) in enumerate(zip(blk, qs))]
              for r in range(8)]
    ws = sa.Workspace(dev)
    for M in (1, 2, 4, 8, 16):
        xs = {K: synth.gen_x(M, K, seed=6, device=dev) for K in (4096, 11008)}
        outs = [torch.empty((M, N), dtype=torch.float16, device=dev) for (n, N, K) in blk]
        ws.get(max(sa.workspace_bytes(L, M) for L in copies[0]))
        nbytes = sum(alg(M, q, N, K) for (n, N, K), q in zip(blk, qs)) * len(copies)

        def run():
            for c in copies:
                for L, o in zip(c, outs):
                    sa.lut_gemm(xs[L.K], L, out=o, workspace=ws, pdl=True)

        us = time_graph(run)
        out.append({"name": "llama7b_batch", "M": M, "config": "LLaMA-2-7B block 31 (7 projections, q=%s), 8 rotating "
                    "copies" % qs, "us_per_block": round(us / len(copies), 2), "GBps": round(nbytes / us * 1e-3, 1),
                    "row_tokens_per_s": round(M * len(copies) / (us * 1e-6), 0)})
    return out


def llama70b_mlp(dev):
    out = []
    for name, N, K in synth.llama2_70b_mlp():
        copies = [pack_layer(3, N, K, synth.seed_for(3, r), dev) for r in range(4)]
        x = synth.gen_x(1, K, seed=7, device=dev)
        y = torch.empty((1, N), dtype=torch.float16, device=dev)
        ws = sa.Workspace(dev)
        ws.get(sa.workspace_bytes(copies[0], 1))

        def run():
            for _ in range(3):
                for L in copies:
                    sa.lut_gemm(x, L, out=y, workspace=ws, pdl=True)

        us = time_graph(run) / (3 * len(copies))
        b = alg(1, 3, N, K)
        out.append({"name": "llama70b_mlp", "layer": name, "N": N, "K": K, "q": 3, "us_per_call": round(us, 2),
                    "GBps": round(b / us * 1e-3, 1), "frac_of_peak": round(b / us * 1e-3 / PEAK, 4)})
        del copies
        torch.cuda.empty_cache()
    return out


def opt66b_decode(dev, q, Ms=(1,)):
    layers = synth.opt_66b_layers() * 64
    packed = []
    for i, (name, N, K) in enumerate(layers):
        packed.append(pack_layer(q, N, K, synth.seed_for(4, i % 6, i // 6), dev))
    res = [_opt66b_run(dev, q, M, layers, packed) for M in Ms]
    del packed
    torch.cuda.empty_cache()
    return res


def _opt66b_run(dev, q, M, layers, packed):
    nbytes = sum(alg(M, q, N, K) for _, N, K in layers)
    xs = {K: synth.gen_x(M, K, seed=8, device=dev) for K in (9216, 36864)}
    outs = [torch.empty((M, L.N), dtype=torch.float16, device=dev) for L in packed]
    ws = sa.Workspace(dev)
    ws.get(max(sa.workspace_bytes(L, M) for L in packed))

    def run():
        for L, o in zip(packed, outs):
            sa.lut_gemm(xs[L.K], L, out=o, workspace=ws, pdl=True)

    us = time_graph(run, reps=3)
    return {"name": "opt66b_decode", "q": q, "M": M,
            "config": "OPT-66B 384 projections (64 x q,k,v,out,fc1,fc2), one GPU, M=%d" % M,
            "ms_per_step": round(us * 1e-3, 3), "GBps": round(nbytes / us * 1e-3, 1),
            "frac_of_peak": round(nbytes / us * 1e-3 / PEAK, 4), "bytes_per_step": nbytes,
            "row_tokens_per_s": round(M / (us * 1e-6), 1)}


def config0(dev):
    copies = [pack_layer(3, 768, 768, synth.seed_for(0, r), dev) for r in range(64)]
    x = synth.gen_x(1, 768, seed=9, device=dev)
    y = torch.empty((1, 768), dtype=torch.float16, device=dev)
    ws = sa.Workspace(dev)
    ws.get(sa.workspace_bytes(copies[0], 1))

    def run():
        for L in copies:
            sa.lut_gemm(x, L, out=y, workspace=ws, pdl=True)

    us = time_graph(run) / len(copies)
    b = alg(1, 3, 768, 768)
    return {"name": "config0", "config": "OPT-125M q_proj 768x768 3-bit", "us_per_call": round(us, 2),
            "GBps": round(b / us * 1e-3, 1)}


def quantize(dev):
    """NEXT-f4: Alg. 1 on the device (fp64), OPT-6.7B FC1 (16384 x 4096) and attention
    (4096 x 4096) weights, g = 128, q = 3, T = 15, PoT projection on."""
    out = []
    for name, N, K in (("attn", 4096, 4096), ("fc1", 16384, 4096)):
        gen = torch.Generator(device=dev).manual_seed(5)
        w = torch.randn((N, K), generator=gen, device=dev) * 0.02
        sa.bcq_quantize(w, 3, 128, T=15, pot=True)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        s, a = sa.bcq_quantize(w, 3, 128, T=15, pot=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        wq = (s.float() * a.repeat_interleave(128, dim=2)).sum(dim=0)
        rel = float(((w - wq) ** 2).sum() / (w ** 2).sum())
        out.append({"name": "quantize", "layer": name, "N": N, "K": K, "q": 3, "g": 128, "T": 15, "pot": True,
                    "ms": round(ms, 3), "weights_per_s": round(N * K / (ms * 1e-3), 0),
                    "rel_sq_error": round(rel, 5)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    jobs = {
        "config0": lambda: [config0(dev)],
        "llama7b_decode": lambda: [llama7b_decode(dev)],
        "llama7b_decode_fused": lambda: [llama7b_decode_fused(dev)],
        "llama7b_batch": lambda: llama7b_batch(dev),
        "llama70b_mlp": lambda: llama70b_mlp(dev),
        # BASELINE configs[4] on one GPU: 2/3/4-bit, batch 1 and 8
        "opt66b_decode": lambda: opt66b_decode(dev, 2, (1, 8)) + opt66b_decode(dev, 3, (1, 8)) +
        opt66b_decode(dev, 4, (1, 8)),
        "quantize": lambda: quantize(dev),
    }
    lines = []
    for name, fn in jobs.items():
        if a.only and name not in a.only:
            continue
        t0 = time.time()
        for r in fn():
            r["wall_s"] = round(time.time() - t0, 1)
            print(json.dumps(r), flush=True)
            lines.append(r)
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "a") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
