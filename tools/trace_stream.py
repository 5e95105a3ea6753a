"""Per-CTA phase trace of the streaming kernel (id 8) in a chain of back-to-back calls
(development tool; needs tools/dev_build.sh).  Prints min/avg/max of each phase (us) relative
to the first CTA start of the last call.  Usage: python tools/trace_stream.py N:K:q ..."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2406_05981_b200 as sa
import synth
sa._LIB_PATH = os.path.join(ROOT, "paper_2406_05981_b200", "libshiftadd_dev.so")
L = sa.lib()
L.shiftadd_dev_set_trace.argtypes = [ctypes.c_void_p]
L.shiftadd_dev_set_variant.argtypes = [ctypes.c_int]
variant = int(os.environ.get("VARIANT", "0"))
L.shiftadd_dev_set_variant(variant)
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
PER_SM = {}
names = ["start", "wait", "lut", "stage0", "loop0", "owner", "loopall", "t0data"]
for spec in sys.argv[1:]:
    N, K, q = map(int, spec.split(":"))
    lb = q * N * K // 8
    R = max(2, -(-4 * l2 // lb))
    signs, alpha = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
    base = sa.pack(signs, alpha, 128, layout=sa.LAYOUT_TILED)
    copies = [base] + [sa.PackedLayer(base.planes.clone(), base.exps.clone(), q, N, K, 128, base.layout, base.counts)
                       for _ in range(R - 1)]
    x = synth.gen_x(1, K, seed=1, device=dev)
    y = torch.empty((1, N), dtype=torch.float16, device=dev)
    ws = sa.Workspace(dev)
    tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for t in range(3):
            sa.lut_gemm(x, copies[t % R], out=y, workspace=ws, pdl=True)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for t in range(2 * R):
            sa.lut_gemm(x, copies[t % R], out=y, workspace=ws, pdl=True)
    with torch.cuda.stream(s):
        g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (2 * R)
    L.shiftadd_dev_set_trace(ctypes.c_void_p(tr.data_ptr()))
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()
    L.shiftadd_dev_set_trace(None)
    t = tr.view(148, 16)[:, :8].cpu().double()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    out = []
    for k, nm in enumerate(names):
        col = rel[:, k]
        col = col[t[:, k] > 0]
        if len(col):
            out.append("%s %.2f/%.2f/%.2f" % (nm, col.min(), col.mean(), col.max()))
    print("v%d N=%d K=%d q=%d %.2f us/call: %s" % (variant, N, K, q, us, "  ".join(out)), flush=True)
    cyc = tr.view(148, 16)[:, 8:15].cpu().double()
    print("   cycles (warp 0): unit1 wait %.0f dot %.0f emit %.0f; loop after LUT %.0f; owner: t0 data %.0f first-stale %.0f spins %.1f (avg)" %
          tuple(cyc.mean(0).tolist()), flush=True)
    print("   max: t0 data %.0f spins %.0f" % (cyc[:, 4].max(), cyc[:, 6].max()), flush=True)
    # per-CTA: does the loop end follow the CTA's start (streaming-bound) or not (consumer-bound)?
    st, le = rel[:, 0], rel[:, 4]
    ok = (t[:, 0] > 0) & (t[:, 4] > 0)
    st, le = st[ok], le[ok]
    cc = float(torch.corrcoef(torch.stack([st, le]))[0, 1])
    order = torch.argsort(st)
    print("   corr(start, loop end) = %.2f; earliest starters' loop end %.2f, latest starters' %.2f" % (
        cc, float(le[order[:20]].mean()), float(le[order[-20:]].mean())), flush=True)
    # per-SM loop duration (LUT done -> loop end): is the slowness a property of the SM?
    smid = tr.view(148, 16)[:, 15].cpu().long()
    dur = (rel[:, 4] - rel[:, 2])
    PER_SM.setdefault(spec, {})
    for c in range(148):
        PER_SM[spec][int(smid[c])] = float(dur[c])
if len(PER_SM) >= 2:
    specs = list(PER_SM)
    a, b = PER_SM[specs[0]], PER_SM[specs[1]]
    sms = sorted(set(a) & set(b))
    va = torch.tensor([a[s] for s in sms]); vb = torch.tensor([b[s] for s in sms])
    print("per-SM loop duration correlation between %s and %s: %.2f" % (specs[0], specs[1],
          float(torch.corrcoef(torch.stack([va, vb]))[0, 1])))
    slow = sorted(sms, key=lambda s: -a[s])[:12]
    print("slowest SMs in %s:" % specs[0], slow, " their rank in %s:" % specs[1],
          [sorted(sms, key=lambda s: -b[s]).index(s) for s in slow])
