"""Parity of the small-batch paths (M = 2..16) against the fp64 oracle (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle, synth
import paper_2406_05981_b200 as sa
dev = torch.device("cuda:0")
for (N, K, q) in [(1000, 1024, 3), (4096, 4096, 2), (4096, 11008, 2), (11008, 4096, 3), (777, 2304, 4), (40, 256, 1)]:
    signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(9, N, K))
    layer = sa.pack(signs.to(dev), alpha.to(dev), 128, layout=sa.LAYOUT_TILED)
    pc, ec, _ = oracle.pack_canonical(signs.numpy(), alpha.numpy(), 128)
    for M in (2, 3, 4, 5, 8, 16):
        x = synth.gen_x(M, K, seed=synth.seed_for(9, M))
        yref = oracle.gemm(x.numpy(), pc, ec, 128)
        y = sa.lut_gemm(x.to(dev), layer, pdl=True); torch.cuda.synchronize()
        y2 = sa.lut_gemm(x.to(dev), layer); torch.cuda.synchronize()
        err = oracle.err_floor(y.float().cpu().numpy(), yref)
        print("N=%d K=%d q=%d M=%d plan=%s err=%.2e det=%s" % (N, K, q, M, sa.gemm_plan(layer, M), err, torch.equal(y, y2)), flush=True)
print("check done")
