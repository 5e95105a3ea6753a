"""Device time of one LLaMA-2-7B decode step (224 projections, synthetic 2.2-bit allocation) as
(a) 128 stream-ordered PDL launches (bench.py's step) and (b) one persistent decode-program
launch (kernel 9, shiftadd_lut_gemv_program), each replayed from a CUDA graph.  Every call of
the program waits for the previous one (SHIFTADD_CALL_WAIT), as the PDL chain does.

    python tools/time_program.py [--steps 50]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    import paper_2406_05981_b200 as sa
    dev = torch.device("cuda", 0)
    launches = bench.build_step(sa, dev, 1, 0)
    ws = sa.Workspace(dev)
    ws.get(max(sa.workspace_bytes(L.layers[0], 1) if L.kind == "gemm" else sa.workspace_bytes_fused(L.layers)
               for L in launches))
    step_bytes = sum(L.alg_bytes() for L in launches)
    stream = torch.cuda.Stream(dev)

    def chain(_t=0):
        for L in launches:
            L(ws, True)

    calls = [(L.x, L.layers, L.outs, j > 0) for j, L in enumerate(launches)]
    prog = sa.Program(calls)

    def program(_t=0):
        prog(stream=stream)

    for name, fn in (("chain", chain), ("program", program)):
        us = bench.graph_time_us(lambda t: [fn(t) for _ in range(1)], args.steps, stream)
        print("%-8s %8.1f us/token  %7.1f GB/s" % (name, us, step_bytes / us * 1e-3), flush=True)
    # parity of the program against the chain's own outputs (same inputs, same weights)
    chain()
    torch.cuda.synchronize()
    ref = [[o.clone() for o in L.outs] for L in launches]
    prog()
    torch.cuda.synchronize()
    worst = 0.0
    for L, r in zip(launches, ref):
        for o, rr in zip(L.outs, r):
            d = float((o.float() - rr.float()).abs().max())
            s = max(float(rr.float().pow(2).mean().sqrt()), 1e-6)
            worst = max(worst, d / s)
    print("program vs chain: max |diff| / rms = %.3g" % worst)


if __name__ == "__main__":
    main()
