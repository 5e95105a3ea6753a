"""Device time per LUT-GEMV call (CUDA graph of back-to-back launches over rotating copies
that exceed L2).  Development tool; bench.py is the contract.
Usage: python tools/time_gemv.py [--pdl] [--m M] N:K:q [N:K:q ...]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.environ.get("SHIFTADD_LIB", "").endswith(".so"):   # an alternative build, for A/B timing
    sa._LIB_PATH = os.path.join(ROOT, os.environ["SHIFTADD_LIB"])
elif os.environ.get("SHIFTADD_LIB") == "dev":   # the dev build and its experiment variants
    import ctypes
    sa._LIB_PATH = os.path.join(ROOT, "paper_2406_05981_b200", "libshiftadd_dev.so")
    sa.lib().shiftadd_dev_set_variant.argtypes = [ctypes.c_int]
    sa.lib().shiftadd_dev_set_variant(int(os.environ.get("VARIANT", "0")))

ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="+")
ap.add_argument("--pdl", action="store_true")
ap.add_argument("--splitk", action="store_true")
ap.add_argument("--cluster", action="store_true", help="thread-block-cluster kernels (FLAG_CLUSTER)")
ap.add_argument("--colwise", action="store_true", help="NEXT-f1 column-wise scales (M = 1)")
ap.add_argument("--apot2", action="store_true", help="NEXT-f2 additive PoT, K = 2 terms")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
peak = 6550.7
for spec in a.shapes:
    N, K, q = map(int, spec.split(":"))
    lb = q * N * K // 8 + (q * K if a.colwise else (2 if a.apot2 else 1) * q * N * K // 128)
    R = max(2, -(-4 * l2 // lb))
    copies = []
    for r in range(R):
        if r < 2:
            if a.colwise:
                signs, alpha = synth.gen_layer_colwise(q, N, K, seed=synth.seed_for(1, 0, r), device=dev)
                copies.append(sa.pack_colwise(signs, alpha))
            elif a.apot2:
                signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(1, 0, r), device=dev)
                copies.append(sa.pack_apot2(signs, alpha, 128, layout=sa.LAYOUT_TILED))
            else:
                signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(1, 0, r), device=dev)
                copies.append(sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED))
            del signs, alpha
        else:
            base = copies[r % 2]
            copies.append(sa.PackedLayer(base.planes.clone(), base.exps.clone(), q, N, K, base.g, base.layout,
                                         base.counts, colwise=base.colwise,
                                         exps2=None if base.exps2 is None else base.exps2.clone()))
    x = synth.gen_x(a.m, K, seed=1, device=dev)
    y = torch.empty((a.m, N), dtype=torch.float16, device=dev)
    ws = sa.Workspace(dev)
    # Everything above was enqueued on the default stream: without this sync the caching
    # allocator may hand y the memory of a just-freed temporary whose kernels have not run,
    # and the GEMV on stream s would overwrite it.
    torch.cuda.synchronize(dev)
    s = torch.cuda.Stream(dev)
    def call(L):
        if a.colwise:
            sa.lut_gemv_colwise(x, L, out=y.view(-1), pdl=a.pdl, workspace=ws, splitk=a.splitk)
        else:
            sa.lut_gemm(x, L, out=y, workspace=ws, pdl=a.pdl, splitk=a.splitk, cluster=a.cluster)

    with torch.cuda.stream(s):
        for t in range(3):
            call(copies[t % R])
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for t in range(a.reps):
            call(copies[t % R])
    with torch.cuda.stream(s):
        g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    us = e0.elapsed_time(e1) / a.reps * 1e3
    tot = lb + 2 * a.m * K + 2 * a.m * N
    print("N=%6d K=%6d q=%d M=%2d  %8.2f us  %7.1f GB/s  frac %.3f  (R=%d, %s)" % (
        N, K, q, a.m, us, tot / us * 1e-3, tot / us * 1e-3 / peak, R, "colwise" if a.colwise else ("apot2 g=128" if a.apot2 else "rowwise g=128")),
        flush=True)
    del copies, g
    torch.cuda.empty_cache()
