"""Run one layer shape through lut_gemm a few times with syncs (for compute-sanitizer).
  python tools/debug_oob.py N K q [--pdl]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

N, K, q = map(int, sys.argv[1:4])
PDL = "--pdl" in sys.argv
dev = torch.device("cuda:0")
s, a = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
L = sa.pack(s, a, 128, layout=sa.LAYOUT_TILED)
torch.cuda.synchronize()
print("plan", sa.gemm_plan(L, 1), flush=True)
x = synth.gen_x(1, K, seed=2, device=dev)
guard = torch.full((1, N + 4096), 7.0, dtype=torch.float16, device=dev)
ws = sa.Workspace(dev)
for i in range(3):
    sa.lut_gemm(x, L, out=guard[:, :N], workspace=ws, pdl=PDL)
    torch.cuda.synchronize()
print("guard intact:", bool((guard[:, N:] == 7.0).all()), flush=True)
