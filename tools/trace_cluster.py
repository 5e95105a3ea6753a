"""Per-CTA phase timeline of the cluster split-K M=1 kernel (development tool).
Usage: SHIFTADD_CLUSTER_TRACE=1 python tools/trace_pair.py N K q [--pdl]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

assert os.environ.get("SHIFTADD_CLUSTER_TRACE") == "1"
N, K, q = map(int, sys.argv[1:4])
PDL = "--pdl" in sys.argv
dev = torch.device("cuda:0")
signs, alpha = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
layers = [sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED)]
for r in range(5):
    layers.append(sa.PackedLayer(layers[0].planes.clone(), layers[0].exps.clone(), q, N, K, 128, 1, layers[0].counts))
x = synth.gen_x(1, K, seed=2, device=dev)
ws = sa.Workspace(dev)
need = 65536 * 4
ws.buf = torch.zeros(need + 512 * 256, dtype=torch.uint8, device=dev)
for i in range(12):
    sa.lut_gemm(x, layers[i % 6], workspace=ws, pdl=PDL)
torch.cuda.synchronize()
G, _, _, kid = sa.gemm_plan(layers[0], 1)
assert kid == 3, kid
tr = ws.buf[need:need + G * 256].cpu().numpy().view(np.uint64).reshape(G, 32).astype(np.int64)
t0 = tr[:, 0].min()
print("N=%d K=%d q=%d G=%d pdl=%d  (us from first CTA start)" % (N, K, q, G, PDL))
for nm, c in [("start", 0), ("pre_x", 8), ("x_arrived", 9), ("x_staged", 1), ("luts_built", 2), ("stage0_full", 10),
              ("last_full", 11), ("loop_end", 3), ("cl_sync", 4), ("end", 5)]:
    v = (tr[:, c] - t0) / 1000.0
    print("  %-10s min %7.2f  med %7.2f  max %7.2f" % (nm, v.min(), np.median(v), v.max()))
le = (tr[:, 3] - t0) / 1000.0
o = np.argsort(-le)
print("  slowest loop_end:", ", ".join("cta %d %.2f sm %d Mw %d" % (i, le[i], tr[i, 6], tr[i, 7]) for i in o[:6]))
print("  Mw values:", sorted(set(tr[:, 7].tolist())))
sm = tr[:, 6]
cnt = {}
for s_ in sm.tolist():
    cnt[s_] = cnt.get(s_, 0) + 1
hist = {}
for v in cnt.values():
    hist[v] = hist.get(v, 0) + 1
print("  CTAs per SM histogram:", dict(sorted(hist.items())), " SMs used:", len(cnt))
for k in sorted(hist):
    sel = np.array([cnt[s_] == k for s_ in sm.tolist()])
    print("    SMs with %d CTA(s): loop_end median %.2f us (n=%d)" % (k, np.median(le[sel]), sel.sum()))
