"""Per-step metadata: from ``ChunkPlan``s to the packed arrays the kernels read.

For the batch of one decode step (requests in batch order, their plans from
``plan_chunk``/``plan_batch``) this builds, on the host:

* the query layout — request r's tokens are ``kv_positions`` then ``window``
  (ChunkPlan order, reference engine.py:28-37), ``cu_seqlens`` over requests;
* rule V inputs: output position p is *visible* iff it was
  DECODED_CACHED before the step or is planned now; ``vis_base`` is the
  32-aligned absolute position below which every key is visible, and
  ``vis_words`` holds one bit per absolute key in ``[vis_base, key_end)``;
  ``key_end`` is the last key any query of the request can see (block-causal
  cap ``(max_q // B + 1) * B``);
* the window-row layout for the unmask kernel (``cu_rows``, ``row_tok``,
  ``row_pos``).

Everything is packed into ONE pinned int32 buffer and shipped with a single
H2D copy (``DeviceMeta.upload``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from .core import TokenState

_I32 = np.int32


@dataclass
class StepMetaHost:
    n_req: int
    n_tok: int
    n_rows: int
    cu_seqlens: np.ndarray
    tok_req: np.ndarray
    tok_pos: np.ndarray
    prompt_len: np.ndarray
    key_end: np.ndarray
    vis_base: np.ndarray
    vis_off: np.ndarray
    vis_words: np.ndarray
    cu_rows: np.ndarray
    row_tok: np.ndarray
    row_pos: np.ndarray
    row_req: np.ndarray
    block_tables: np.ndarray
    commits_expected_rows: int = 0

    @property
    def max_pages(self) -> int:
        return self.block_tables.shape[1]


def request_visibility(states: np.ndarray, plan) -> np.ndarray:
    """Rule V state part: visible output positions for this step."""
    vis = states == TokenState.DECODED_CACHED
    if plan.kv_positions or plan.window:
        vis = vis.copy()
        if plan.kv_positions:
            vis[list(plan.kv_positions)] = True
        if plan.window:
            vis[list(plan.window)] = True
    return vis


def build_step_meta(requests: Sequence, plans: Sequence, block_size: int,
                    block_tables: np.ndarray) -> StepMetaHost:
    """Pack one step.  ``block_tables`` rows are in batch order."""
    n_req = len(requests)
    counts = np.fromiter((len(p.kv_positions) + len(p.window) for p in plans), dtype=_I32, count=n_req)
    wins = np.fromiter((len(p.window) for p in plans), dtype=_I32, count=n_req)
    cu = np.zeros(n_req + 1, dtype=_I32)
    np.cumsum(counts, out=cu[1:])
    cu_rows = np.zeros(n_req + 1, dtype=_I32)
    np.cumsum(wins, out=cu_rows[1:])
    n_tok = int(cu[-1])
    n_rows = int(cu_rows[-1])
    tok_pos = np.empty(n_tok, dtype=_I32)
    tok_req = np.repeat(np.arange(n_req, dtype=_I32), counts)
    prompt = np.empty(n_req, dtype=_I32)
    key_end = np.zeros(n_req, dtype=_I32)
    vis_base = np.zeros(n_req, dtype=_I32)
    vis_off = np.zeros(n_req + 1, dtype=_I32)
    row_tok = np.empty(n_rows, dtype=_I32)
    row_pos = np.empty(n_rows, dtype=_I32)
    row_req = np.repeat(np.arange(n_req, dtype=_I32), wins)
    word_chunks = []
    n_words = 0
    for r, (req, plan) in enumerate(zip(requests, plans)):
        t0 = int(cu[r])
        nkv = len(plan.kv_positions)
        nw = len(plan.window)
        if nkv:
            tok_pos[t0:t0 + nkv] = plan.kv_positions
        if nw:
            tok_pos[t0 + nkv:t0 + nkv + nw] = plan.window
            r0 = int(cu_rows[r])
            row_pos[r0:r0 + nw] = plan.window
            row_tok[r0:r0 + nw] = np.arange(t0 + nkv, t0 + nkv + nw, dtype=_I32)
        P = int(req.prompt_tokens)
        prompt[r] = P
        vis_off[r] = n_words
        if nkv + nw == 0:
            vis_base[r] = 0
            key_end[r] = 0
            continue
        vis = request_visibility(req.states, plan)
        invisible = np.flatnonzero(~vis)
        cp = int(invisible[0]) if invisible.size else len(vis)
        visible = np.flatnonzero(vis)
        last = int(visible[-1]) if visible.size else -1
        max_q = int(tok_pos[t0:t0 + nkv + nw].max())
        end_out = min(last + 1, (max_q // block_size + 1) * block_size)
        ke = P + end_out
        key_end[r] = ke
        vb = ((P + cp) // 32) * 32
        if vb > ke:
            vb = (ke // 32) * 32
        vis_base[r] = vb
        if ke > vb:
            nbits = ((ke - vb + 31) // 32) * 32
            bits = np.zeros(nbits, dtype=bool)
            # absolute positions [vb, ke): prompt part visible, output part from vis
            a0 = vb - P  # output index of the first bit (may be negative)
            if a0 < 0:
                bits[: min(-a0, ke - vb)] = True
                lo_out, lo_bit = 0, -a0
            else:
                lo_out, lo_bit = a0, 0
            hi_out = ke - P
            if hi_out > lo_out:
                bits[lo_bit:lo_bit + (hi_out - lo_out)] = vis[lo_out:hi_out]
            words = np.packbits(bits, bitorder="little").view(np.uint32)
            word_chunks.append(words)
            n_words += words.size
    vis_off[n_req] = n_words
    vis_words = np.concatenate(word_chunks) if word_chunks else np.zeros(1, dtype=np.uint32)
    return StepMetaHost(
        n_req=n_req, n_tok=n_tok, n_rows=n_rows, cu_seqlens=cu, tok_req=tok_req,
        tok_pos=tok_pos, prompt_len=prompt, key_end=key_end, vis_base=vis_base,
        vis_off=vis_off, vis_words=vis_words, cu_rows=cu_rows, row_tok=row_tok,
        row_pos=row_pos, row_req=row_req, block_tables=np.ascontiguousarray(block_tables, dtype=_I32),
    )


_FIELDS = ("cu_seqlens", "tok_req", "tok_pos", "prompt_len", "key_end", "vis_base", "vis_off",
           "vis_words", "cu_rows", "row_tok", "row_pos", "row_req", "block_tables")


@dataclass
class DeviceMeta:
    """Device views of a StepMetaHost, shipped in one H2D copy."""

    host: StepMetaHost
    buf: torch.Tensor
    views: dict = field(default_factory=dict)
    h2d_bytes: int = 0

    def __getattr__(self, name):
        views = self.__dict__.get("views")
        if views is not None and name in views:
            return views[name]
        raise AttributeError(name)

    @staticmethod
    def upload(meta: StepMetaHost, device, pinned: Optional[torch.Tensor] = None,
               dev_buf: Optional[torch.Tensor] = None, stream=None) -> "DeviceMeta":
        arrays = []
        for name in _FIELDS:
            a = getattr(meta, name)
            a = a.view(np.int32) if a.dtype == np.uint32 else a.astype(np.int32, copy=False)
            arrays.append((name, a))
        # 16-byte align every field (kernels use int4/uint4 loads on some of them)
        offs, total = {}, 0
        for name, a in arrays:
            offs[name] = total
            total += ((a.size + 3) // 4) * 4
        total = max(total, 4)
        if pinned is None or pinned.numel() < total:
            pinned = torch.empty(total, dtype=torch.int32, pin_memory=torch.cuda.is_available())
        host = pinned.numpy()
        for name, a in arrays:
            host[offs[name]:offs[name] + a.size] = a.reshape(-1)
        if dev_buf is None or dev_buf.numel() < total:
            dev_buf = torch.empty(total, dtype=torch.int32, device=device)
        dev_buf[:total].copy_(pinned[:total], non_blocking=True)
        views = {}
        for name, a in arrays:
            v = dev_buf[offs[name]:offs[name] + a.size]
            if name == "block_tables":
                v = v.view(meta.block_tables.shape)
            views[name] = v
        dm = DeviceMeta(meta, dev_buf, views, total * 4)
        dm.__dict__["pinned"] = pinned
        return dm
