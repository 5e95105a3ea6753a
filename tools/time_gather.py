"""Single-GPU cost of the NEXT-f3 fused-gather epilogue (dev tool).  One process plays rank 0
of P = 2: the 'peer' gathered buffer is a local allocation and the absent rank's flag is
pre-set, so this isolates the epilogue's extra stores, the completion signal and the wait
kernel (NVLink itself is not measurable on a 1-GPU box).
  python tools/time_gather.py N:K:q ..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_05981_b200 as sa  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
L_ = sa.lib()
for spec in sys.argv[1:]:
    N, K, q = map(int, spec.split(":"))
    R = max(2, -(-4 * 126 * 2 ** 20 // (q * N * K // 8)))
    s, a = synth.gen_layer(q, N, K, 128, seed=1, device=dev)
    base = sa.pack(s, a, 128, layout=sa.LAYOUT_TILED)
    copies = [base] + [sa.PackedLayer(base.planes.clone(), base.exps.clone(), q, N, K, 128, 1, base.counts)
                       for _ in range(R - 1)]
    x = synth.gen_x(1, K, seed=2, device=dev)
    y = torch.empty((1, N), dtype=torch.float16, device=dev)
    ybufs = [[torch.zeros(2 * N, dtype=torch.float16, device=dev) for _ in range(2)] for _ in range(2)]
    flags = [torch.zeros(2, dtype=torch.int32, device=dev) for _ in range(2)]
    flags[0][1] = 0x7fffffff            # the absent rank 1 has "already published" every epoch
    y_ptrs = torch.tensor([ybufs[0][0].data_ptr(), ybufs[1][0].data_ptr(), ybufs[0][1].data_ptr(),
                           ybufs[1][1].data_ptr()], dtype=torch.int64, device=dev)
    epoch = torch.zeros(1, dtype=torch.int32, device=dev)
    dummy_epoch = torch.zeros(1, dtype=torch.int32, device=dev)
    f_ptrs = torch.tensor([flags[0].data_ptr(), flags[1].data_ptr()], dtype=torch.int64, device=dev)
    ws = sa.Workspace(dev)
    ws.get(max(sa.workspace_bytes(base, 1), 256 * 1024 + 16))
    torch.cuda.synchronize()
    st = torch.cuda.Stream(dev)
    reps = 200
    ep = [0]

    def plain(t):
        sa.lut_gemm(x, copies[t % R], out=y, workspace=ws, pdl=True, stream=st)

    def fused(t):
        ep[0] += 1
        L = copies[t % R]
        r = L_.shiftadd_lut_gemv_gather(x.data_ptr(), L.planes.data_ptr(), L.exps.data_ptr(), 1, N, K, q, 128,
                                        y_ptrs.data_ptr(), f_ptrs.data_ptr(), 2, 0, epoch.data_ptr(), ws.buf.data_ptr(),
                                        ws.buf.numel(), 1, st.cuda_stream)
        assert r == 0, L_.shiftadd_last_error()
        r = L_.shiftadd_gather_wait(flags[0].data_ptr(), 2, epoch.data_ptr(), st.cuda_stream)
        assert r == 0

    def fused_nowait(t):
        ep[0] += 1
        L = copies[t % R]
        r = L_.shiftadd_lut_gemv_gather(x.data_ptr(), L.planes.data_ptr(), L.exps.data_ptr(), 1, N, K, q, 128,
                                        y_ptrs.data_ptr(), f_ptrs.data_ptr(), 2, 0, dummy_epoch.data_ptr(),
                                        ws.buf.data_ptr(), ws.buf.numel(), 1, st.cuda_stream)
        assert r == 0

    def plain_wait(t):
        plain(t)
        r = L_.shiftadd_gather_wait(flags[0][1:].data_ptr(), 1, dummy_epoch.data_ptr(), st.cuda_stream)
        assert r == 0

    res = {}
    for name, fn in (("plain", plain), ("fused", fused), ("fused_nowait", fused_nowait), ("plain_wait", plain_wait)):
        with torch.cuda.stream(st):
            for t in range(3):
                fn(t)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for t in range(reps):
                fn(t)
        with torch.cuda.stream(st):
            g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
        st.synchronize()
        res[name] = e0.elapsed_time(e1) / reps * 1e3
    ok = torch.equal(ybufs[0][0][:N], ybufs[1][0][:N]) and torch.equal(ybufs[0][1][:N], ybufs[1][1][:N])
    print("N=%6d K=%5d q=%d  plain %.2f  fused+wait %.2f  fused only %.2f  plain+wait %.2f us  copies equal: %s"
          % (N, K, q, res["plain"], res["fused"], res["fused_nowait"], res["plain_wait"], ok), flush=True)
