"""Per-CTA phase timeline of the M=1 kernel (SHIFTADD_EXP=4 trace mode; development tool).
Usage: SHIFTADD_EXP=4 python tools/trace_gemv.py N K q"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

assert os.environ.get("SHIFTADD_EXP") in ("4", "5")
N, K, q = map(int, sys.argv[1:4])
PDL = "--pdl" in sys.argv
dev = torch.device("cuda:0")
signs, alpha = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
layers = [sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED)]
for r in range(5):
    layers.append(sa.PackedLayer(layers[0].planes.clone(), layers[0].exps.clone(), q, N, K, 128, 1, layers[0].counts))
x = synth.gen_x(1, K, seed=2, device=dev)
S, RG = K // 256, -(-N // 16)
need = 65536 * 4 + S * RG * 16 * 4
ws = sa.Workspace(dev)
ws.buf = torch.zeros(need + 4096 * 128, dtype=torch.uint8, device=dev)
for i in range(12):
    sa.lut_gemm(x, layers[i % 6], workspace=ws, pdl=PDL)
torch.cuda.synchronize()
G = sa.gemm_plan(layers[0], 1)[0]
full = ws.buf[need:need + G * 128].cpu().numpy().view(np.uint64).reshape(G, 16).astype(np.int64)
tr = full[:, [0, 8, 9, 1, 2, 3, 4]]
t0 = tr[:, 0].min()
rel = (tr - t0) / 1000.0
names = ["start", "x_arrived", "own_built", "lut_built", "main_end", "barrier", "end"]
print("N=%d K=%d q=%d G=%d pdl=%d  (us from first CTA start)" % (N, K, q, G, PDL))
for i, nm in enumerate(names):
    col = rel[:, i]
    print("  %-10s min %7.2f  med %7.2f  max %7.2f" % (nm, col.min(), np.median(col), col.max()))

main = rel[:, 4]
order = np.argsort(-main)
print("  slowest CTAs (main_end us, smid, segments, u0):")
for i in order[:8]:
    print("    cta %3d  %7.2f  sm %3d  seg %d  u0 %d" % (i, main[i], full[i, 5], full[i, 6], full[i, 7]))
print("  fastest:", ", ".join("cta %d %.2f sm %d seg %d" % (i, main[i], full[i, 5], full[i, 6]) for i in order[-4:]))
two = full[:, 6] > 1
if two.any():
    print("  main_end median: 1-seg CTAs %.2f, 2-seg CTAs %.2f (%d of them)" % (np.median(main[~two]), np.median(main[two]), two.sum()))
sm = full[:, 5]
per_sm = {}
for i in range(G):
    per_sm.setdefault(int(sm[i]), []).append(main[i])
