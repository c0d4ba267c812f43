"""Multi-GPU decomposition of the decode step (one process per GPU, NCCL).

Attention shards by KV head: rank r of N owns KV heads
[r*Hkv/N, (r+1)*Hkv/N) and their G query heads each, and holds only those heads'
KV pages — K1/K2 have no exchange at all.  The unmask shards by vocabulary: each
rank reduces its vocab slice of every window row to {max, sum exp, argmax}
partials (12 bytes per row and split); ONE all-gather of those partials lets every
rank run the same deterministic merge (optimus_unmask_finalize, fixed order), so
commit decisions are bitwise identical on all ranks without broadcasting them.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import ops


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    kv_heads: tuple     # [lo, hi)
    q_heads: tuple      # [lo, hi)
    vocab: tuple        # [lo, hi)


def shard_for(rank: int, world: int, num_q_heads: int, num_kv_heads: int, vocab: int) -> Shard:
    if num_kv_heads % world:
        raise ValueError("world size must divide the number of KV heads")
    g = num_q_heads // num_kv_heads
    per = num_kv_heads // world
    kv = (rank * per, (rank + 1) * per)
    return Shard(rank, world, kv, (kv[0] * g, kv[1] * g),
                 (rank * vocab // world, (rank + 1) * vocab // world))


class TensorParallelUnmask:
    """K3 over a vocabulary shard + all-gather of the partials + replicated merge."""

    def __init__(self, world: int, rank: int, vocab_offset: int, group=None):
        self.world = world
        self.rank = rank
        self.vocab_offset = vocab_offset
        self.group = group
        self._gather = None

    def __call__(self, dec, dm, logits, row_src) -> ops.UnmaskResult:
        m = dm.host
        n_vsplit = ops.unmask_splits(max(m.n_rows, 1), dec.cfg.vocab)
        part = ops.unmask_partials(logits, row_src, m.n_rows, n_vsplit, vocab_offset=self.vocab_offset)
        need = (self.world, max(m.n_rows, 1), n_vsplit, 3)
        if self._gather is None or self._gather.numel() < self.world * part.numel():
            self._gather = torch.empty(self.world * part.numel(), dtype=torch.float32, device=part.device)
        out = self._gather[: self.world * part.numel()].view(need)
        if dist.get_backend(self.group) == "gloo":
            # host-staged exchange (validation runs of the sharded path on one GPU)
            host = [torch.empty_like(part, device="cpu") for _ in range(self.world)]
            dist.all_gather(host, part.cpu(), group=self.group)
            out.copy_(torch.stack(host).view(need))
        else:
            dist.all_gather_into_tensor(out, part.contiguous(), group=self.group)
        return ops.unmask_finalize(out, self.world, m.n_rows, n_vsplit, dm.cu_rows,
                                   dec.cfg.confidence_threshold, dec.cfg.fallback)
