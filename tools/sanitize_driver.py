"""One small call of every device path, for compute-sanitizer (tests/test_gpu_sanitizers.py).
Exits non-zero if any result misses the oracle bar, so a sanitizer run also checks results."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

if os.environ.get("SHIFTADD_LIB_PATH"):   # e.g. the bounds-checked build (tools/check_build.sh)
    sa._LIB_PATH = os.environ["SHIFTADD_LIB_PATH"]

dev = torch.device("cuda:0")
bad = []


def check(name, y, ref):
    err = oracle.err_floor(y.float().cpu().numpy().reshape(ref.shape), ref)
    if not err <= 2e-3:
        bad.append((name, err))


def rowwise(q, N, K, M, **kw):
    s, a = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(12, N, K))
    p, e, _ = oracle.pack_canonical(s.numpy(), a.numpy(), 128)
    L = sa.pack(s.to(dev), a.to(dev), 128, layout=sa.LAYOUT_TILED)
    x = synth.gen_x(M, K, seed=M)
    y = sa.lut_gemm(x.to(dev), L, pdl=True, **kw)
    torch.cuda.synchronize()
    check("rowwise q%d N%d K%d M%d %s %s" % (q, N, K, M, kw, sa.gemm_plan(L, M)), y, oracle.gemm(x.numpy(), p, e, 128))


rowwise(3, 256, 1024, 1)                      # cluster kernel (3)
rowwise(3, 272, 1024, 1, splitk=True)         # streaming kernel (8), straddling chunks
rowwise(2, 64, 256, 1, splitk=True)           # streaming, S = 1
rowwise(2, 256, 6144, 1)                      # streaming, one slice per CTA (S = 24)
rowwise(3, 100, 9216, 1)                      # streaming, weight-balanced split
rowwise(3, 272, 1024, 2)                      # cluster ring M = 2 (5)
rowwise(3, 272, 1024, 3)                      # cluster ring M = 3..4 (6)
for M in (2, 4, 8, 12):                       # streaming MW = 2, 4, 8 and two row chunks
    rowwise(2, 200, 1024, M, splitk=True)
# fused segments
K = 1024
x = synth.gen_x(1, K, seed=3)
cases = []
for i, (q, N) in enumerate([(2, 96), (3, 40), (1, 33)]):
    s, a = synth.gen_layer(q, N, K, 128, seed=synth.seed_for(12, 50 + i))
    p, e, _ = oracle.pack_canonical(s.numpy(), a.numpy(), 128)
    cases.append((sa.pack(s.to(dev), a.to(dev), 128, layout=sa.LAYOUT_TILED), p, e))
for splitk in (False, True):                  # cluster ring (10) / streaming (8)
    ys = sa.lut_gemv_fused(x.to(dev), [c[0] for c in cases], pdl=True, splitk=splitk)
    torch.cuda.synchronize()
    for (L, p, e), y in zip(cases, ys):
        check("fused splitk=%s" % splitk, y, oracle.gemm(x.numpy(), p, e, 128))
# persistent decode program (9): call 1 reads call 0's output (SHIFTADD_CALL_WAIT)
sA, aA = synth.gen_layer(2, 256, 1024, 128, seed=synth.seed_for(12, 71))
sB, aB = synth.gen_layer(3, 64, 256, 128, seed=synth.seed_for(12, 72))
pA, eA, _ = oracle.pack_canonical(sA.numpy(), aA.numpy(), 128)
pB, eB, _ = oracle.pack_canonical(sB.numpy(), aB.numpy(), 128)
LA = sa.pack(sA.to(dev), aA.to(dev), 128, layout=sa.LAYOUT_TILED)
LB = sa.pack(sB.to(dev), aB.to(dev), 128, layout=sa.LAYOUT_TILED)
xa = synth.gen_x(1, 1024, seed=7)
yA = torch.empty(256, dtype=torch.float16, device=dev)
yB = torch.empty(64, dtype=torch.float16, device=dev)
sa.Program([(xa.to(dev), [LA], [yA], False), (yA, [LB], [yB], True)])()
torch.cuda.synchronize()
refA = oracle.gemm(xa.numpy(), pA, eA, 128)
check("program call 0", yA, refA)
check("program call 1", yB, oracle.gemm(oracle.to_fp16(refA).astype("float64"), pB, eB, 128))
# block-wise: scaled LUTs (N % 128 == 0) and per-query scales
for N in (256, 40):
    s, a = synth.gen_layer_blockwise(2, N, 1024, seed=synth.seed_for(12, 60, N))
    p, e, _ = oracle.pack_blockwise(s.numpy(), a.numpy())
    L = sa.pack_blockwise(s.to(dev), a.to(dev))
    xb = synth.gen_x(1, 1024, seed=4)
    y = sa.lut_gemv_blockwise(xb.to(dev), L, pdl=True)
    torch.cuda.synchronize()
    check("blockwise N%d" % N, y, oracle.gemm_blockwise(xb.numpy(), p, e))
# column-wise scales: cluster kernel, streaming kernel (K > 4096), pairs of rows
for (qc, Nc, Kc, Mc) in ((2, 200, 1024, 1), (3, 100, 8192, 1), (2, 96, 1024, 3)):
    sc, ac = synth.gen_layer_colwise(qc, Nc, Kc, seed=synth.seed_for(12, 80, Kc + Mc))
    pc, ec, _ = oracle.pack_colwise(sc.numpy(), ac.numpy())
    Lc = sa.pack_colwise(sc.to(dev), ac.to(dev))
    xc2 = synth.gen_x(Mc, Kc, seed=8 + Mc)
    yc = sa.lut_gemv_colwise(xc2.to(dev), Lc, pdl=True)
    torch.cuda.synchronize()
    check("colwise K%d M%d" % (Kc, Mc), yc.reshape(Mc, Nc), oracle.gemm_colwise(xc2.numpy(), pc, ec))
# additive PoT, two terms: cluster kernel and the streaming kernel (K > 4096)
for (qa, Na, Ka) in ((2, 128, 1024), (3, 100, 6144)):
    sA2, aA2 = synth.gen_layer(qa, Na, Ka, 128, seed=synth.seed_for(12, 90, Ka))
    pA2, e1A2, e2A2, _ = oracle.pack_apot2(sA2.numpy(), aA2.numpy(), 128)
    LA2 = sa.pack_apot2(sA2.to(dev), aA2.to(dev), 128, layout=sa.LAYOUT_TILED)
    xA2 = synth.gen_x(1, Ka, seed=9)
    yA2 = sa.lut_gemm(xA2.to(dev), LA2, pdl=True)
    torch.cuda.synchronize()
    check("apot2 K%d" % Ka, yA2, oracle.gemm_apot2(xA2.numpy(), pA2, e1A2, e2A2, 128))
# canonical layout (generic kernel)
s, a = synth.gen_layer(2, 64, 512, 64, seed=5)
p, e, _ = oracle.pack_canonical(s.numpy(), a.numpy(), 64)
L = sa.pack(s.to(dev), a.to(dev), 64, layout=sa.LAYOUT_CANONICAL)
xc = synth.gen_x(3, 512, seed=6)
y = sa.lut_gemm(xc.to(dev), L)
torch.cuda.synchronize()
check("canonical", y, oracle.gemm(xc.numpy(), p, e, 64))
if bad:
    print("PARITY FAILURES", bad)
    sys.exit(3)
print("sanitize driver ok")
