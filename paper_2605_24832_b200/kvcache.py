"""Paged KV cache, page pool and block tables.

The reference has no KV memory at all (``SPEC.md:14,270``: "no KV memory
paging"); this is the B200 layer beneath its ``Request`` objects.

Layout in HBM (one tensor per K and V, all layers):
    k[L][num_pages][Hkv][page_size][head_dim]  bf16
    v[L][num_pages][Hkv][page_size][head_dim]  fp16 (default) or bf16
so each (layer, page, head) is a contiguous page_size x head_dim tile — the unit
the attention kernel stages with one TMA box per 64 columns.  A request's
absolute position s (prompt + output position) lives in page
``block_table[s // page_size]`` at row ``s % page_size`` (SURVEY §8c rule S).

Pages are allocated from a host free list when a request's positions need
them (prompt at admission, each decode block as it opens) and returned when the
request finishes; a request holds at most ``max_pages`` pages.
"""

from __future__ import annotations

from typing import Dict, Iterable, Optional

import numpy as np
import torch

from .errors import ConfigError


class PagePool:
    """LIFO free list of physical page ids."""

    def __init__(self, num_pages: int):
        if num_pages < 1:
            raise ConfigError("num_pages must be >= 1")
        self.num_pages = num_pages
        self._free = list(range(num_pages - 1, -1, -1))

    @property
    def free_pages(self) -> int:
        return len(self._free)

    def alloc(self, n: int) -> list:
        if n > len(self._free):
            raise ConfigError(f"KV cache exhausted: need {n} pages, {len(self._free)} free")
        out = self._free[-n:][::-1] if n else []
        if n:
            del self._free[-n:]
        return out

    def free(self, pages: Iterable[int]) -> None:
        self._free.extend(reversed(list(pages)))


class BlockTables:
    """Per-slot page lists plus the dense int32 table the kernels read.

    Slots are batch rows of the device state; a request keeps its slot from
    admission to completion.
    """

    def __init__(self, pool: PagePool, max_slots: int, max_pages: int, page_size: int):
        self.pool = pool
        self.page_size = page_size
        self.max_pages = max_pages
        self.table = np.zeros((max_slots, max_pages), dtype=np.int32)
        self.n_pages = np.zeros(max_slots, dtype=np.int32)
        self._slot_of: Dict[int, int] = {}
        self._free_slots = list(range(max_slots - 1, -1, -1))

    def slot(self, request_id: int) -> Optional[int]:
        return self._slot_of.get(request_id)

    def admit(self, request_id: int, n_positions: int, slot: Optional[int] = None) -> int:
        """Give a request a batch slot (the most recently freed one, or `slot` if
        given and free) and pages for n_positions."""
        if request_id in self._slot_of:
            raise ConfigError(f"request {request_id} already admitted")
        if not self._free_slots:
            raise ConfigError("no free batch slot")
        if slot is not None:
            if slot not in self._free_slots:
                raise ConfigError(f"batch slot {slot} is not free")
            self._free_slots.remove(slot)
            s = slot
        else:
            s = self._free_slots.pop()
        self._slot_of[request_id] = s
        self.n_pages[s] = 0
        self.ensure(s, n_positions)
        return s

    def ensure(self, slot: int, n_positions: int) -> None:
        """Make positions [0, n_positions) addressable for this slot."""
        need = (n_positions + self.page_size - 1) // self.page_size
        have = int(self.n_pages[slot])
        if need <= have:
            return
        if need > self.max_pages:
            raise ConfigError(
                f"request needs {need} pages > max_pages {self.max_pages} "
                f"(page_size {self.page_size})"
            )
        pages = self.pool.alloc(need - have)
        self.table[slot, have:need] = pages
        self.n_pages[slot] = need

    def release(self, request_id: int) -> None:
        s = self._slot_of.pop(request_id)
        n = int(self.n_pages[s])
        self.pool.free(self.table[s, :n].tolist())
        self.table[s, :n] = 0  # no stale page ids survive in a free slot's row
        self.n_pages[s] = 0
        self._free_slots.append(s)


class PagedKVCache:
    """Device KV storage for ``num_layers`` layers."""

    def __init__(self, num_layers: int, num_pages: int, num_kv_heads: int, page_size: int,
                 head_dim: int, device="cuda", dtype=torch.bfloat16, v_dtype=torch.float16):
        if page_size < 8 or page_size > 1024 or page_size & (page_size - 1):
            raise ConfigError("page_size must be a power of two in [8, 1024]")
        if head_dim not in (64, 128):
            raise ConfigError("head_dim must be 64 or 128")
        shape = (num_layers, num_pages, num_kv_heads, page_size, head_dim)
        if v_dtype not in (torch.bfloat16, torch.float16):
            raise ConfigError("v_dtype must be bf16 or fp16")
        # K is bf16 (the model's dtype).  V defaults to fp16: the bf16 values are
        # stored exactly (|v| < 65504), and the attention kernel can then form P.V
        # with an 11-bit fp16 P in a single tensor-core MMA.
        self.k = torch.zeros(shape, dtype=dtype, device=device)
        self.v = torch.zeros(shape, dtype=v_dtype, device=device)
        self.num_layers = num_layers
        self.num_pages = num_pages
        self.num_kv_heads = num_kv_heads
        self.page_size = page_size
        self.head_dim = head_dim

    def layer(self, l: int):
        return self.k[l], self.v[l]

    @property
    def nbytes(self) -> int:
        return self.k.numel() * self.k.element_size() * 2
