"""§8(e) multi-GPU: N-sharded (column-parallel) LUT-GEMV with an NCCL all-gather of y.

Output rows are independent (per-row scale groups stay local, no partial-sum reduction), so
rank r of P owns rows [r*N/P, (r+1)*N/P) of every layer -- its own packed planes/exponents --
and the only exchange is one all-gather of y over NVLink/NVSwitch (the next layer needs the
whole y).  x is replicated (in a model it is the previous layer's gathered output).  For
M > 1 the gathered buffer is [P][M][N/P] and is permuted to [M][N].

BASELINE.json north_star: "partitioned across 2/4/8 GPUs ... by output rows N
(column-parallel), with an NCCL all-gather of y over NVLink".
"""

from __future__ import annotations

import torch
import torch.distributed as dist

import ctypes

from . import FLAG_PDL, LAYOUT_TILED, PackedLayer, Workspace, _check, lib, lut_gemm, pack

__all__ = ["shard_range", "gather_output", "ShardedLinear", "FusedGatherLinear"]


def shard_range(N: int, world: int, rank: int):
    """Rows [n0, n1) owned by ``rank``; equal shards (all_gather_into_tensor needs them)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if N % world:
        raise ValueError("N=%d is not divisible by the world size %d" % (N, world))
    n = N // world
    return rank * n, (rank + 1) * n


def gather_output(y_local: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather the row shards y_local [M][N/P] of every rank into y [M][N]."""
    world = dist.get_world_size(group)
    M, n = y_local.shape
    if world == 1:
        return y_local
    if y_local.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host tensors only: stage through the host (several ranks sharing one GPU
        # in tests, or a CPU-only process group) -- the collective's plumbing, not the compute
        y_host = gather_output(y_local.cpu(), group)
        if out is not None:
            out.copy_(y_host.view(out.shape))
            return out
        return y_host.to(y_local.device)
    if M == 1:
        flat = out.view(-1) if out is not None else torch.empty(world * n, dtype=y_local.dtype,
                                                                device=y_local.device)
        dist.all_gather_into_tensor(flat, y_local.reshape(-1).contiguous(), group=group)
        return flat.view(1, world * n)
    buf = torch.empty((world * M, n), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(buf, y_local.contiguous(), group=group)
    y = buf.view(world, M, n).permute(1, 0, 2).reshape(M, world * n)
    if out is not None:
        out.copy_(y)
        return out
    return y


class ShardedLinear:
    """One reparameterised linear layer, row-sharded over the ranks of ``group``."""

    def __init__(self, layer: PackedLayer, N_full: int, group=None):
        self.layer = layer
        self.N = N_full
        self.group = group
        self.workspace = Workspace(layer.device)

    @classmethod
    def from_full(cls, signs: torch.Tensor, alpha: torch.Tensor, g: int, group=None,
                  layout: int = LAYOUT_TILED) -> "ShardedLinear":
        """Pack this rank's rows of a full layer (signs [q][N][K], alpha [q][N][K/g])."""
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        N = signs.shape[1]
        n0, n1 = shard_range(N, world, rank)
        layer = pack(signs[:, n0:n1].contiguous(), alpha[:, n0:n1].contiguous(), g, layout=layout)
        return cls(layer, N, group)

    def __call__(self, x: torch.Tensor, pdl: bool = False) -> torch.Tensor:
        x2 = x.unsqueeze(0) if x.dim() == 1 else x
        y_local = lut_gemm(x2, self.layer, workspace=self.workspace, pdl=pdl)
        if not dist.is_initialized():
            return y_local
        return gather_output(y_local, self.group)


def _share(t: torch.Tensor):
    """Picklable CUDA IPC description of ``t`` (torch's own reducer)."""
    from torch.multiprocessing.reductions import reduce_tensor
    return reduce_tensor(t)


def _open(desc):
    fn, args = desc
    return fn(*args)


class FusedGatherLinear:
    """NEXT-f3: row-sharded layer whose GEMV epilogue writes y straight into every rank's
    gathered buffer (shiftadd_lut_gemv_gather), followed by an on-stream flag wait
    (shiftadd_gather_wait) -- no NCCL call on the data path.

    Each rank allocates two gathered buffers [max_m][P*n] (double-buffered by call parity, see
    include/shiftadd.h) and a flag array uint32[P]; their CUDA IPC handles are exchanged once
    over ``group`` (any backend; gloo works) and mapped into every process.  Peers on other
    GPUs are reached over NVLink through the IPC mappings; ranks may also share one GPU
    (that is how the single-GPU test exercises the protocol)."""

    def __init__(self, layer: PackedLayer, N_full: int, group=None, max_m: int = 1):
        self.layer = layer
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = layer.N
        self.max_m = max_m
        if self.n * self.P != N_full:
            raise ValueError("N_full must equal P * local rows")
        if not 1 <= max_m <= 8:
            raise ValueError("max_m must be in [1, 8]")
        dev = layer.device
        self.ybuf = [torch.zeros(max_m * self.P * self.n, dtype=torch.float16, device=dev) for _ in range(2)]
        self.flags = torch.zeros(self.P, dtype=torch.int32, device=dev)
        mine = [_share(self.ybuf[0]), _share(self.ybuf[1]), _share(self.flags)]
        allh = [None] * self.P
        dist.all_gather_object(allh, mine, group=group)
        self._peers = []                                  # keep mapped tensors alive
        yp = [[], []]
        fp = []
        for r in range(self.P):
            if r == self.rank:
                t = [self.ybuf[0], self.ybuf[1], self.flags]
            else:
                t = [_open(d) for d in allh[r]]
                self._peers.append(t)
            yp[0].append(t[0].data_ptr())
            yp[1].append(t[1].data_ptr())
            fp.append(t[2].data_ptr())
        self.y_ptrs = torch.tensor(yp[0] + yp[1], dtype=torch.int64, device=dev)   # [2P]: buffer b of rank r
        self.flag_ptrs = torch.tensor(fp, dtype=torch.int64, device=dev)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)                 # device call counter
        self.workspace = Workspace(dev)
        from . import workspace_bytes
        self.workspace.get(max(workspace_bytes(layer, max_m), 256 * 1024 + 16))
        self.calls = 0                                                             # host mirror (parity)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    def __call__(self, x: torch.Tensor, pdl: bool = False, stream=None, layer: PackedLayer | None = None):
        """y [M][P*n] for x [K] or [M][K] fp16 (M <= max_m); the returned view is valid until call + 2.
        ``layer`` may substitute another packed layer of the same shape (rotating copies).
        The call counter is on the device (graph capture works); the returned view follows
        the host's count of calls, so a replayed graph should hold an even number of calls
        of this layer when its outputs are read."""
        L = layer if layer is not None else self.layer
        xv = x.reshape(-1, L.K) if x.dim() == 2 else x.reshape(1, -1)
        M = xv.shape[0]
        if xv.dtype != torch.float16 or xv.shape[1] != L.K or not 1 <= M <= self.max_m:
            raise ValueError("x must be fp16 [K] or [M][K] with M <= max_m")
        xv = xv.contiguous()
        self.calls += 1
        par = self.calls & 1
        dev = L.device
        sptr = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
        ws = self.workspace.buf
        lib_ = lib()
        st = lib_.shiftadd_lut_gemm_gather(xv.data_ptr(), L.K, L.planes.data_ptr(), L.exps.data_ptr(), L.layout, M,
                                          self.n, L.K, L.q, L.g, self.y_ptrs.data_ptr(), self.flag_ptrs.data_ptr(),
                                          self.P, self.rank, self.epoch.data_ptr(), ws.data_ptr(), ws.numel(),
                                          FLAG_PDL if pdl else 0, sptr)
        if st:
            _check(st, "shiftadd_lut_gemm_gather")
        st = lib_.shiftadd_gather_wait(self.flags.data_ptr(), self.P, self.epoch.data_ptr(), sptr)
        if st:
            _check(st, "shiftadd_gather_wait")
        return self.ybuf[par][:M * self.P * self.n].view(M, -1)
