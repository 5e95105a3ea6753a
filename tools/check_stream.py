"""Parity of the streaming kernel (id 8) against the fp64 oracle on a few shapes (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle, synth
import paper_2406_05981_b200 as sa
dev = torch.device("cuda:0")
for (N, K, q) in [(768, 768, 3) if False else (768, 1024, 3), (4096, 4096, 2), (4096, 4096, 3), (11008, 4096, 3),
                  (4096, 11008, 2), (1000, 512, 4), (40, 256, 1), (28672, 8192, 3)]:
    signs, alpha = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(9, N, K))
    layer = sa.pack(signs.to(dev), alpha.to(dev), 128, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(1, K, seed=synth.seed_for(9, 1))
    rows = slice(0, N) if N * K <= 4096 * 11008 else slice(0, 512)
    pc, ec, _ = oracle.pack_canonical(signs[:, rows].numpy(), alpha[:, rows].numpy(), 128)
    yref = oracle.gemm(x.numpy(), pc, ec, 128)
    plan = sa.gemm_plan(layer, 1)
    outs = []
    for rep in range(3):
        y = sa.lut_gemm(x.to(dev), layer, pdl=(rep == 2))
        torch.cuda.synchronize()
        outs.append(y.cpu())
    same = all(torch.equal(outs[0], o) for o in outs)
    err = oracle.err_floor(outs[0][:, rows].float().numpy(), yref)
    yc = sa.lut_gemm(x.to(dev), layer, splitk=True); torch.cuda.synchronize()
    errc = oracle.err_floor(yc.cpu()[:, rows].float().numpy(), yref)
    print("N=%d K=%d q=%d plan=%s err=%.2e (splitk path %.2e) deterministic=%s" % (N, K, q, plan, err, errc, same), flush=True)
print("check done")
