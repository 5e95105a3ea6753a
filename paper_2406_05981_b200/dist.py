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

from . import LAYOUT_TILED, PackedLayer, Workspace, lut_gemm, pack

__all__ = ["shard_range", "gather_output", "ShardedLinear"]


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
