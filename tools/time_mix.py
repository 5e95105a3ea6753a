"""Per-step device time of a chain that cycles through several layer shapes (dev tool).

  python tools/time_mix.py [--nopdl] N:K:q N:K:q ...     (one step = one call per shape)

Each shape gets R rotating weight copies (> 4x L2 in total); the chain is captured in one
CUDA graph of `reps` steps and timed with CUDA events.  Compare with the sum of the shapes'
solo per-call times (tools/time_gemv.py) to see what switching kernels costs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
PDL = "--nopdl" not in sys.argv
dev = torch.device("cuda:0")
shapes = [tuple(map(int, s.split(":"))) for s in args]
total = sum(q * N * K // 8 for N, K, q in shapes)
R = max(2, (4 * 126 * 2 ** 20) // total + 1)
copies = []
for r in range(R):
    cur = []
    for i, (N, K, q) in enumerate(shapes):
        s, a = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(7, i, r), device=dev)
        cur.append(sa.pack(s, a, 128, layout=sa.LAYOUT_TILED))
        del s, a
    copies.append(cur)
xs = {K: synth.gen_x(1, K, seed=3, device=dev) for _, K, _ in shapes}
ys = [torch.empty((1, N), dtype=torch.float16, device=dev) for N, _, _ in shapes]
ws = sa.Workspace(dev)
ws.get(max(sa.workspace_bytes(L, 1) for L in copies[0]))
torch.cuda.synchronize()   # inputs were made on the default stream
stream = torch.cuda.Stream()
reps = 20 * R


def run():
    for t in range(reps):
        for i, L in enumerate(copies[t % R]):
            sa.lut_gemm(xs[L.K], L, out=ys[i], workspace=ws, pdl=PDL)


with torch.cuda.stream(stream):
    run()
stream.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    run()
with torch.cuda.stream(stream):
    g.replay()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
stream.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
print("%-60s %8.2f us/step  %7.1f GB/s planes  (pdl=%d, R=%d, kernels %s)" % (
    " ".join(args), us, total / us * 1e-3, PDL, R, [sa.gemm_plan(L, 1)[3] for L in copies[0]]))
