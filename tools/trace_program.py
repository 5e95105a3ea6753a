"""Per-call phase trace of the persistent decode program (kernel 9) on the LLaMA-2-7B step
(development tool; needs tools/dev_build.sh).  For each call kind (q/k/v, o, gate/up, down)
prints the mean over calls of: completion-to-completion time (max over CTAs), and the mean
over CTAs of each phase -- dependency wait, x + LUT build, lookup loop (warp 0), owner waiting
for partials, owner sums + completion -- plus the producer's first-stage issue time relative
to the consumers' call start.  Usage: python tools/trace_program.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402

sa._LIB_PATH = os.path.join(ROOT, "paper_2406_05981_b200", "libshiftadd_dev.so")
L = sa.lib()
L.shiftadd_dev_set_program_trace.argtypes = [ctypes.c_void_p]
L.shiftadd_dev_set_program_variant.argtypes = [ctypes.c_int]
VARIANT = int(os.environ.get("VARIANT", "0"))   # 1: the producer does not prefetch across calls
L.shiftadd_dev_set_program_variant(VARIANT)
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    launches = bench.build_step(sa, dev, 1, 0)
    calls = [(Lc.x, Lc.layers, Lc.outs, j > 0) for j, Lc in enumerate(launches)]
    prog = sa.Program(calls)
    n = len(calls)
    G = torch.cuda.get_device_properties(dev).multi_processor_count
    for _ in range(3):
        prog()
    torch.cuda.synchronize()
    tr = torch.zeros(G * n * 8, dtype=torch.int64, device=dev)
    L.shiftadd_dev_set_program_trace(ctypes.c_void_p(tr.data_ptr()))
    prog()
    torch.cuda.synchronize()
    L.shiftadd_dev_set_program_trace(None)
    t = tr.view(G, n, 8).double().cpu()
    t0 = t[:, 0, 0].min()
    t = (t - t0) / 1e3   # us
    kinds = {}
    for j in range(n):
        kinds.setdefault(j % 4, []).append(j)
    names = {0: "q/k/v", 1: "o", 2: "gate/up", 3: "down"}
    done = t[:, :, 5].max(dim=0).values
    print("total %.1f us for %d calls" % (float(done[-1]), n))
    print("variant %d" % VARIANT)
    print("%-8s %7s %7s %7s %7s %7s %7s %8s %7s" % ("call", "c2c", "wait", "lut", "loop", "owner", "final", "prod-lead",
                                                  "x-lat"))
    for k, js in kinds.items():
        c2c = sum(float(done[j] - (done[j - 1] if j else 0.0)) for j in js) / len(js)
        ph = [0.0] * 5
        lead = xl = 0.0
        for j in js:
            for p in range(5):
                ph[p] += float((t[:, j, p + 1] - t[:, j, p]).mean())
            lead += float((t[:, j, 1] - t[:, j, 6]).mean())
            xl += float((t[:, j, 7] - t[:, j, 1]).mean())
        ph = [v / len(js) for v in ph]
        print("%-8s %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %8.2f %7.2f" % (names[k], c2c, *ph, lead / len(js), xl / len(js)))
    # spread of the loop end across CTAs, and of the completion
    for k in (0, 2, 3):
        spread(t, kinds[k][5], names[k])




def spread(t, j, label):
    import statistics
    d = (t[:, j, 3] - t[:, j, 2]).tolist()
    st = t[:, j, 2].tolist()
    en = t[:, j, 3].tolist()
    q = lambda v: "min %.2f med %.2f max %.2f" % (min(v), statistics.median(v), max(v))
    print("%s call %d: loop start %s | loop dur %s | loop end %s" % (label, j, q(st), q(d), q(en)))
    order = sorted(range(len(d)), key=lambda c: d[c])
    print("   slowest CTAs:", [(c, round(d[c], 2)) for c in order[-6:]], "fastest:", [(c, round(d[c], 2)) for c in order[:4]])


if __name__ == "__main__":
    main()
