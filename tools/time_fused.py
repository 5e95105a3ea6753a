"""Device time per fused LUT-GEMV launch (shiftadd_lut_gemv_fused) over rotating copies, graph
of back-to-back calls with PDL (dev tool).  Usage: python tools/time_fused.py K:N1q1,N2q2,... ...
(e.g. 4096:4096q2,4096q3,4096q2).  SHIFTADD_LIB=dev and VARIANT=n select the dev build's variant."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2406_05981_b200 as sa
import synth
if os.environ.get("SHIFTADD_LIB", "").endswith(".so"):   # an alternative build, for A/B timing
    sa._LIB_PATH = os.path.join(ROOT, os.environ["SHIFTADD_LIB"])
elif os.environ.get("SHIFTADD_LIB") == "dev":
    sa._LIB_PATH = os.path.join(ROOT, "paper_2406_05981_b200", "libshiftadd_dev.so")
    L = sa.lib()
    L.shiftadd_dev_set_variant.argtypes = [ctypes.c_int]
    L.shiftadd_dev_set_variant(int(os.environ.get("VARIANT", "0")))
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
for spec in sys.argv[1:]:
    K, segs = spec.split(":")
    K = int(K)
    segs = [tuple(map(int, s.split("q"))) for s in segs.split(",")]
    lb = sum(q * N * K // 8 + q * N * K // 128 + 2 * N for N, q in segs) + 2 * K
    R = max(2, -(-4 * l2 // lb))
    base = [[sa.pack(*synth.gen_layer(q, N, K, 128, seed=synth.seed_for(1, r, N + q), device=dev), 128,
                     layout=sa.LAYOUT_TILED) for N, q in segs] for r in range(2)]
    copies = [base[r % 2] if r < 2 else [sa.PackedLayer(L.planes.clone(), L.exps.clone(), L.q, L.N, L.K, L.g, L.layout,
                                                       L.counts) for L in base[r % 2]] for r in range(R)]
    x = synth.gen_x(1, K, seed=1, device=dev).view(-1)
    outs = [torch.empty(N, dtype=torch.float16, device=dev) for N, _ in segs]
    ws = sa.Workspace(dev)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(dev)
    def call(t):
        if len(segs) == 1:
            sa.lut_gemm(x.view(1, -1), copies[t % R][0], out=outs[0].view(1, -1), workspace=ws, pdl=True)
        else:
            sa.lut_gemv_fused(x, copies[t % R], outs=outs, workspace=ws, pdl=True, splitk=os.environ.get("SPLITK") == "1")
    with torch.cuda.stream(s):
        for t in range(3):
            call(t)
    s.synchronize()
    reps = max(R, 60)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for t in range(reps):
            call(t)
    with torch.cuda.stream(s):
        g.replay()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print("%s: %.2f us  %.1f GB/s  frac %.3f" % (spec, us, lb / us * 1e-3, lb / us * 1e-3 / 6540.8), flush=True)
