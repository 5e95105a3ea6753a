"""Launch a few LUT-GEMV calls of one shape for ncu (not a benchmark: ncu serialises and
cold-caches every launch).  Usage: python tools/prof_gemv.py N K q [M] [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

N, K, q = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
M = int(sys.argv[4]) if len(sys.argv) > 4 else 1
n = int(sys.argv[5]) if len(sys.argv) > 5 else 3
dev = torch.device("cuda:0")
copies = []
for r in range(2):
    signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(1, 0, r), device=dev)
    copies.append(sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED))
    del signs, alpha
x = synth.gen_x(M, K, seed=1, device=dev)
for t in range(n):
    y = sa.lut_gemm(x, copies[t % 2])
torch.cuda.synchronize()
print("ok", N, K, q, M, sa.gemm_plan(copies[0], M))
