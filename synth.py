"""Seeded synthetic inputs shared by tests/, bench.py and smoke() (DESIGN.md §Input recipe).

This module holds none of the hot path's arithmetic (no packing, no PoT rounding, no LUT,
no shift, no GEMV).  It produces *unpacked* BCQ layers -- int8 sign planes in {-1,+1} and
fp32 scale factors alpha -- and fp16 activations, with the shapes and value structure of the
paper's workloads.  Both the CUDA path and the oracle receive the same tensors.

Layer recipe (§3, Eq. 1 greedy init, PAPER.md:129-134 -- the offline quantiser's
first step, which is *input synthesis* here and not an §8 row):
    W ~ N(0, 0.02^2)  (fp32), per output row n and scale group G of g columns:
    r_0 = W;  b_i = sign(r_{i-1}) (sign(0) = +1);  alpha_i = mean |r_{i-1}|_G;
    r_i = r_{i-1} - alpha_i b_i.
alpha stays full precision; rounding it to a power of two is pack's job (§8 a1).

Activations (PAPER.md:212 -- LLM activations carry outlier channels):
    x fp16 ~ N(0, 1), with max(1, K/256) channels (the same for every row) scaled by 20.

Everything is generated with an explicit ``torch.Generator`` seeded from
``BASE_SEED + 1000*config + 10*layer + rank``; CPU and CUDA generators give different streams,
so parity tests always generate on CPU and copy to the device.
"""

from __future__ import annotations

import torch

BASE_SEED = 20240609

__all__ = [
    "BASE_SEED", "seed_for", "gen_layer", "gen_x", "gen_special_x", "llama2_7b_layers",
    "llama2_7b_allocation", "opt_6p7b_layer_set", "opt_66b_layers", "llama2_70b_mlp",
    "CONFIGS",
]


def seed_for(config: int, layer: int = 0, rank: int = 0) -> int:
    return BASE_SEED + 1000 * config + 10 * layer + rank


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def gen_layer(q: int, N: int, K: int, g: int, seed: int, device="cpu", std: float = 0.02,
              row_chunk: int = 4096):
    """Greedy-BCQ synthetic layer: returns (signs int8 [q][N][K], alpha fp32 [q][N][K/g])."""
    if K % g:
        raise ValueError("g must divide K")
    gen = _gen(seed, device)
    signs = torch.empty((q, N, K), dtype=torch.int8, device=device)
    alpha = torch.empty((q, N, K // g), dtype=torch.float32, device=device)
    for n0 in range(0, N, row_chunk):
        n1 = min(N, n0 + row_chunk)
        r = torch.randn((n1 - n0, K), generator=gen, device=device, dtype=torch.float32) * std
        for i in range(q):
            b = torch.where(r >= 0, 1.0, -1.0)
            a = r.abs().view(n1 - n0, K // g, g).mean(dim=2)
            signs[i, n0:n1] = b.to(torch.int8)
            alpha[i, n0:n1] = a
            r = r - (a.repeat_interleave(g, dim=1) * b)
    return signs, alpha


def gen_layer_colwise(q: int, N: int, K: int, seed: int, device="cpu", std: float = 0.02):
    """Greedy BCQ with column-wise scales (NEXT-f1): plane i takes
    b_i = sign(r), alpha_i[k] = mean_n |r[n][k]| (one scale per input column), r -= alpha_i b_i.
    Returns (signs int8 [q][N][K], alpha fp32 [q][K])."""
    gen = _gen(seed, device)
    r = torch.randn((N, K), generator=gen, device=device, dtype=torch.float32) * std
    signs = torch.empty((q, N, K), dtype=torch.int8, device=device)
    alpha = torch.empty((q, K), dtype=torch.float32, device=device)
    for i in range(q):
        b = torch.where(r >= 0, 1.0, -1.0)
        a = r.abs().mean(dim=0)
        signs[i] = b.to(torch.int8)
        alpha[i] = a
        r = r - a[None, :] * b
    return signs, alpha


def gen_layer_blockwise(q: int, N: int, K: int, seed: int, device="cpu", std: float = 0.02):
    """Greedy BCQ with block-wise scales (NEXT-f1 "Ours (Lat.)"): plane i
    takes b_i = sign(r), alpha_i[b][c] = mean |r| over the N/8 rows of block b and the 8
    columns of group c, r -= alpha_i b_i.  Returns (signs int8 [q][N][K], alpha fp32 [q][8][K/8])."""
    gen = _gen(seed, device)
    r = torch.randn((N, K), generator=gen, device=device, dtype=torch.float32) * std
    signs = torch.empty((q, N, K), dtype=torch.int8, device=device)
    alpha = torch.empty((q, 8, K // 8), dtype=torch.float32, device=device)
    for i in range(q):
        b = torch.where(r >= 0, 1.0, -1.0)
        a = r.abs().view(8, N // 8, K // 8, 8).mean(dim=(1, 3))          # [8][K/8]
        signs[i] = b.to(torch.int8)
        alpha[i] = a
        r = r - a.repeat_interleave(N // 8, dim=0).repeat_interleave(8, dim=1) * b
    return signs, alpha


def gen_x(M: int, K: int, seed: int, device="cpu", outlier_scale: float = 20.0):
    """fp16 activations [M][K]: N(0,1) with max(1, K//256) outlier channels x outlier_scale."""
    gen = _gen(seed, device)
    x = torch.randn((M, K), generator=gen, device=device, dtype=torch.float32)
    n_out = max(1, K // 256)
    idx = torch.randperm(K, generator=gen, device=device)[:n_out]
    x[:, idx] *= outlier_scale
    return x.to(torch.float16)


def gen_special_x(kind: str, M: int, K: int, seed: int = 0, j: int = 0):
    """Edge-case activations for parity: 'basis' (e_j), 'zero', 'ones', 'max' (+-65504 mix)."""
    if kind == "basis":
        x = torch.zeros((M, K), dtype=torch.float16)
        x[:, j] = 1.0
        return x
    if kind == "zero":
        return torch.zeros((M, K), dtype=torch.float16)
    if kind == "ones":
        return torch.ones((M, K), dtype=torch.float16)
    if kind == "max":
        gen = _gen(seed, "cpu")
        s = torch.where(torch.rand((M, K), generator=gen) < 0.5, -1.0, 1.0)
        return (s * 65504.0).to(torch.float16)
    raise ValueError(kind)


# ------------------------------------------------------------------ workload shapes (N, K)
def opt_6p7b_layer_set():
    """BASELINE.json configs[1]: OPT-6.7B attn 4096x4096 and FC1 (N=16384, K=4096), q in {2,3}."""
    return [("attn", 4096, 4096, 2), ("attn", 4096, 4096, 3),
            ("fc1", 16384, 4096, 2), ("fc1", 16384, 4096, 3)]


def llama2_7b_layers():
    """32 blocks x (q,k,v,o 4096x4096; gate,up N=11008,K=4096; down N=4096,K=11008)."""
    out = []
    for blk in range(32):
        for name in ("q_proj", "k_proj", "v_proj", "o_proj"):
            out.append((blk, name, 4096, 4096))
        out.append((blk, "gate_proj", 11008, 4096))
        out.append((blk, "up_proj", 11008, 4096))
        out.append((blk, "down_proj", 4096, 11008))
    return out


def llama2_7b_allocation():
    """Synthetic Eq. 4 allocation with budget 2.2 bits:
    3 bits for every k_proj and for up_proj of blocks 20-31, 2 bits elsewhere
    (44 of 224 layers at 3 bits = 492 bits = floor(2.2*224); Fig. 7: K layers, FC1 and later
    blocks get more bits).  Returns a list of q aligned with llama2_7b_layers()."""
    q = []
    for blk, name, _, _ in llama2_7b_layers():
        hi = name == "k_proj" or (name == "up_proj" and blk >= 20)
        q.append(3 if hi else 2)
    return q


def llama2_70b_mlp():
    return [("gate_proj", 28672, 8192), ("up_proj", 28672, 8192), ("down_proj", 8192, 28672)]


def opt_66b_layers():
    """Per block: q,k,v,out 9216x9216; fc1 N=36864,K=9216; fc2 N=9216,K=36864 (x64 blocks)."""
    return [("q_proj", 9216, 9216), ("k_proj", 9216, 9216), ("v_proj", 9216, 9216),
            ("out_proj", 9216, 9216), ("fc1", 36864, 9216), ("fc2", 9216, 36864)]


CONFIGS = {
    0: "OPT-125M q_proj 768x768, 3-bit, g=128, M=1",
    1: "OPT-6.7B layer set (attn 4096x4096, FC1 16384x4096) at 2/3-bit, g=128, M=1",
    2: "LLaMA-2-7B projections, mixed 2/3-bit, g=128, M=1..16",
    3: "LLaMA-2-70B MLP 3-bit, N-sharded over 2/4/8 GPUs",
    4: "OPT-66B all linear layers 2/3/4-bit, M in {1,8}, 8 GPUs",
}
