"""Per-CTA phase timeline of the TMA-ring split-K kernel (kernel 4; development tool).
Usage: SHIFTADD_STREAM_TRACE=1 python tools/trace_stream.py N K q [--pdl]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

assert os.environ.get("SHIFTADD_STREAM_TRACE") == "1"
N, K, q = map(int, sys.argv[1:4])
PDL = "--pdl" in sys.argv
dev = torch.device("cuda:0")
signs, alpha = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
layers = [sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED)]
del signs, alpha
for r in range(3):
    layers.append(sa.PackedLayer(layers[0].planes.clone(), layers[0].exps.clone(), q, N, K, 128, 1, layers[0].counts))
x = synth.gen_x(1, K, seed=2, device=dev)
ws = sa.Workspace(dev)
S, RG = K // 256, (N + 15) // 16
need = 65536 * 4 + S * RG * 16 * 4
ws.buf = torch.zeros(need + 148 * 128 + 4096, dtype=torch.uint8, device=dev)
for i in range(8):
    sa.lut_gemm(x, layers[i % 4], workspace=ws, pdl=PDL)
torch.cuda.synchronize()
G, _, _, kid = sa.gemm_plan(layers[0], 1)
assert kid == 4, kid
tr = ws.buf[need:need + G * 128].cpu().numpy().view(np.uint64).reshape(G, 16).astype(np.int64)
t0 = tr[:, 0].min()
print("N=%d K=%d q=%d G=%d pdl=%d  (us from first CTA start)" % (N, K, q, G, PDL))
for nm, c in [("start", 0), ("pdl_wait", 1), ("luts_built", 2), ("stage0_full", 3), ("loop_end", 4),
              ("arrived", 5), ("counters_ok", 6), ("end", 7)]:
    v = (tr[:, c] - t0) / 1000.0
    print("  %-12s min %7.2f  med %7.2f  max %7.2f" % (nm, v.min(), np.median(v), v.max()))
