"""Per-CTA phase timeline of the M=1 kernel (SHIFTADD_EXP=4 trace mode; development tool).
Usage: SHIFTADD_EXP=4 python tools/trace_gemv.py N K q"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

assert os.environ.get("SHIFTADD_EXP") == "4"
N, K, q = map(int, sys.argv[1:4])
dev = torch.device("cuda:0")
signs, alpha = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
layers = [sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED)]
for r in range(5):
    layers.append(sa.PackedLayer(layers[0].planes.clone(), layers[0].exps.clone(), q, N, K, 128, 1, layers[0].counts))
x = synth.gen_x(1, K, seed=2, device=dev)
S, RG = K // 256, -(-N // 16)
need = 256 + S * RG * 16 * 4
ws = sa.Workspace(dev)
ws.buf = torch.zeros(need + 4096 * 64, dtype=torch.uint8, device=dev)
for i in range(12):
    sa.lut_gemm(x, layers[i % 6], workspace=ws)
torch.cuda.synchronize()
G = sa.gemm_plan(layers[0], 1)[0]
tr = ws.buf[need:need + G * 64].cpu().numpy().view(np.uint64).reshape(G, 8)[:, :5].astype(np.int64)
t0 = tr[:, 0].min()
rel = (tr - t0) / 1000.0
names = ["start", "lut_built", "main_end", "barrier", "end"]
print("N=%d K=%d q=%d G=%d  (us from first CTA start)" % (N, K, q, G))
for i, nm in enumerate(names):
    col = rel[:, i]
    print("  %-10s min %7.2f  med %7.2f  max %7.2f" % (nm, col.min(), np.median(col), col.max()))
