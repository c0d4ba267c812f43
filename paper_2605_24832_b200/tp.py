"""Tensor-parallel output projection of the decode step (BASELINE configs[4]).

With attention sharded by KV head, rank r holds the attention output of its query
heads only.  The row-parallel o-proj multiplies that [n_tok, Hq/N * d] slice by its
rows of W_o ([Hq * d, hidden], rows [r * Hq/N * d, (r+1) * Hq/N * d)) and the N
partial [n_tok, hidden] products are summed by ONE all-reduce per layer: NCCL over
NVLink in production (the only collective the north_star allows in the end-to-end
step besides the unmask partials' all-gather), host-staged gloo when validating
the sharded path with several ranks on one GPU.  The GEMM is cuBLAS bf16 (a plain
library GEMM); the activations are synthetic (no checkpoints), W_o is random-init
from a seed shared by every rank, so the sharded sum reproduces the unsharded
product.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class RowParallelOProj:
    def __init__(self, num_layers: int, num_q_heads: int, head_dim: int, hidden: int, world: int = 1,
                 rank: int = 0, device="cuda", seed: int = 0, group=None):
        if num_q_heads % world:
            raise ValueError("world size must divide the query heads")
        self.world, self.rank, self.group = world, rank, group
        self.hidden = hidden
        rows = num_q_heads * head_dim
        per = rows // world
        self.weights = []
        g = torch.Generator(device=device)
        for layer in range(num_layers):
            g.manual_seed(seed * 7919 + layer)
            w = torch.randn((rows, hidden), generator=g, device=device, dtype=torch.float32)
            w = (w * rows ** -0.5).to(torch.bfloat16)
            self.weights.append(w[rank * per:(rank + 1) * per].contiguous())
        self.out = None

    def __call__(self, layer: int, attn_out: torch.Tensor) -> torch.Tensor:
        """attn_out [n_tok, Hq/N, d] bf16 -> summed [n_tok, hidden] bf16."""
        n = attn_out.shape[0]
        x = attn_out.reshape(n, -1)
        if self.out is None or self.out.shape[0] < n:
            self.out = torch.empty((max(n, 1), self.hidden), dtype=torch.bfloat16, device=attn_out.device)
        y = self.out[:n]
        torch.matmul(x, self.weights[layer], out=y)
        if self.world > 1:
            if dist.get_backend(self.group) == "gloo":
                h = y.float().cpu()
                dist.all_reduce(h, group=self.group)
                y.copy_(h.to(torch.bfloat16))
            else:
                dist.all_reduce(y, group=self.group)
        return y
