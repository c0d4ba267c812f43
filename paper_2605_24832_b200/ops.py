"""Torch-facing wrappers of the C-ABI kernels (K1 append, K2 attention, K3 unmask).

Torch is only the allocator/stream provider here: every wrapper checks that its
tensors live on a CUDA device, passes raw pointers through ctypes, and maps a
non-zero status to ``ConfigError`` / ``DeviceError``.  Nothing here computes on
the CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import ConfigError

FALLBACK_MODES = {"earliest": 0, "top1": 1, "none": 2}


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _cuda(*tensors: Optional[torch.Tensor]) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ConfigError("B200 kernels take CUDA tensors only (no CPU path)")


def _stream(stream: Optional[torch.cuda.Stream] = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _v_dtype(v_cache: torch.Tensor) -> int:
    if v_cache.dtype == torch.bfloat16:
        return 0
    if v_cache.dtype == torch.float16:
        return 1
    raise ConfigError("V cache must be bf16 or fp16")


def sm_count() -> int:
    return int(_lib.call("optimus_device_sm_count"))


# --------------------------------------------------------------------------- K1
def kv_append(
    k_new: torch.Tensor,
    v_new: torch.Tensor,
    tok_req: torch.Tensor,
    tok_pos: torch.Tensor,
    prompt_len: torch.Tensor,
    block_tables: torch.Tensor,
    k_cache: torch.Tensor,
    v_cache: torch.Tensor,
    slot_mapping_out: Optional[torch.Tensor] = None,
    stream=None,
    slot_abs: Optional[torch.Tensor] = None,
) -> None:
    """Scatter ``k_new``/``v_new`` ``[n_tok, Hkv, d]`` into ``[num_pages, Hkv, P, d]`` caches.
    With ``slot_abs`` (the step's :func:`slot_mapping`) the slots are read, not
    re-derived (``optimus_kv_append_slots``)."""
    _cuda(k_new, v_new, tok_req, tok_pos, prompt_len, block_tables, k_cache, v_cache, slot_mapping_out)
    n_tok = k_new.shape[0]
    num_pages, hkv, page, d = k_cache.shape
    if k_new.dtype != torch.bfloat16 or v_new.dtype != torch.bfloat16 or k_cache.dtype != torch.bfloat16:
        raise ConfigError("kv_append: new K/V rows and the K cache are bf16")
    if k_new.stride(-1) != 1 or k_new.stride(-2) != d or v_new.stride(0) != k_new.stride(0):
        raise ConfigError("kv_append: K/V rows must be [n_tok, Hkv, d] with unit inner strides")
    if slot_abs is not None:
        _cuda(slot_abs)
        if slot_mapping_out is not None:
            raise ConfigError("kv_append: slot_mapping_out is the slot map itself with slot_abs")
        st = _lib.call("optimus_kv_append_slots", _ptr(k_new), _ptr(v_new), k_new.stride(0), _ptr(slot_abs),
                       n_tok, hkv, d, page, _ptr(k_cache), _ptr(v_cache), num_pages, _v_dtype(v_cache),
                       _stream(stream))
        _lib.check(st, "optimus_kv_append_slots")
        return
    st = _lib.call(
        "optimus_kv_append",
        _ptr(k_new), _ptr(v_new), k_new.stride(0),
        _ptr(tok_req), _ptr(tok_pos), _ptr(prompt_len), _ptr(block_tables),
        block_tables.shape[1], n_tok, hkv, d, page,
        _ptr(k_cache), _ptr(v_cache), num_pages, _ptr(slot_mapping_out), _v_dtype(v_cache),
        _stream(stream),
    )
    _lib.check(st, "optimus_kv_append")


def slot_mapping(
    tok_req: torch.Tensor,
    tok_pos: torch.Tensor,
    prompt_len: torch.Tensor,
    block_tables: torch.Tensor,
    page_size: int,
    n_tok: Optional[int] = None,
    out: Optional[torch.Tensor] = None,
    stream=None,
) -> torch.Tensor:
    """Rule S once per step: int32 ``[n_tok, 2]`` = (absolute position, slot) for the
    first ``n_tok`` tokens (default: all of ``tok_req``)."""
    _cuda(tok_req, tok_pos, prompt_len, block_tables, out)
    n_tok = tok_req.shape[0] if n_tok is None else int(n_tok)
    if n_tok > tok_req.shape[0] or n_tok > tok_pos.shape[0]:
        raise ConfigError("slot_mapping: n_tok exceeds the token arrays")
    if out is None:
        out = torch.empty((max(n_tok, 1), 2), dtype=torch.int32, device=tok_req.device)
    st = _lib.call("optimus_slot_mapping", _ptr(tok_req), _ptr(tok_pos), _ptr(prompt_len),
                   _ptr(block_tables), block_tables.shape[1], n_tok, page_size, _ptr(out), _stream(stream))
    _lib.check(st, "optimus_slot_mapping")
    return out


# --------------------------------------------------------------------------- K2 plan
@dataclass
class AttnPlan:
    """Output of the host work planner, resident on the device."""

    grid: int
    n_work: int
    n_groups: int
    n_partials: int
    work: torch.Tensor      # int32 [n_work, 8]
    cta_off: torch.Tensor   # int32 [grid + 1]
    groups: torch.Tensor    # int32 [n_groups, 8]
    work_host: np.ndarray
    cta_off_host: np.ndarray
    groups_host: np.ndarray
    single_tile: bool = False  # every (request, KV head) is one query tile: K1 may fold into K2


def single_query_tile(cu_seqlens_q: np.ndarray, num_q_heads: int, num_kv_heads: int) -> bool:
    """True when no request's query tokens span two MMA tiles (q_r x Hq/Hkv <= 128):
    the planner then emits one token group per (request, KV head), the precondition of
    the fused append (optimus_paged_attn_append)."""
    if len(cu_seqlens_q) < 2:
        return True
    return int(np.diff(cu_seqlens_q).max()) * (num_q_heads // num_kv_heads) <= 128


def plan_attention(
    cu_seqlens_q: np.ndarray,
    key_end: np.ndarray,
    num_q_heads: int,
    num_kv_heads: int,
    grid: Optional[int] = None,
    min_split_tiles: int = 4,
    device: Optional[torch.device] = None,
    page_size: int = 16,
) -> AttnPlan:
    """Split (request, kv head, query tile) units into key ranges and place them
    on persistent CTAs (``optimus_attn_plan``)."""
    cu = np.ascontiguousarray(cu_seqlens_q, dtype=np.int32)
    ke = np.ascontiguousarray(key_end, dtype=np.int32)
    n_req = len(ke)
    if grid is None:
        grid = sm_count() if torch.cuda.is_available() else 148
    mw, mg = C.c_int(0), C.c_int(0)
    _lib.check(
        _lib.call(
            "optimus_attn_plan_bounds", n_req, cu.ctypes.data, ke.ctypes.data,
            num_q_heads, num_kv_heads, min_split_tiles, page_size, C.byref(mw), C.byref(mg),
        ),
        "optimus_attn_plan_bounds",
    )
    work = np.zeros((max(mw.value, 1), 8), dtype=np.int32)
    groups = np.zeros((max(mg.value, 1), 8), dtype=np.int32)
    cta_off = np.zeros(grid + 1, dtype=np.int32)
    ng, npart = C.c_int(0), C.c_int(0)
    n = _lib.call(
        "optimus_attn_plan", n_req, cu.ctypes.data, ke.ctypes.data, num_q_heads, num_kv_heads,
        grid, min_split_tiles, page_size, work.ctypes.data, work.shape[0], cta_off.ctypes.data,
        groups.ctypes.data, groups.shape[0], C.byref(ng), C.byref(npart),
    )
    if n < 0:
        _lib.check(n, "optimus_attn_plan")
    work = work[:n]
    groups = groups[: ng.value]
    if device is None:
        dev_work = torch.from_numpy(work.copy())
        dev_off = torch.from_numpy(cta_off.copy())
        dev_groups = torch.from_numpy(groups.copy())
    else:
        dev_work = torch.from_numpy(work).to(device)
        dev_off = torch.from_numpy(cta_off).to(device)
        dev_groups = torch.from_numpy(groups).to(device)
    return AttnPlan(grid, n, ng.value, npart.value, dev_work, dev_off, dev_groups, work, cta_off, groups,
                    single_query_tile(cu, num_q_heads, num_kv_heads))


# --------------------------------------------------------------------------- K2
def paged_attention(
    q: torch.Tensor,
    k_cache: torch.Tensor,
    v_cache: torch.Tensor,
    q_pos: torch.Tensor,
    prompt_len: torch.Tensor,
    vis_base: torch.Tensor,
    vis_off: torch.Tensor,
    vis_words: torch.Tensor,
    block_tables: torch.Tensor,
    plan: AttnPlan,
    block_size: int,
    sm_scale: Optional[float] = None,
    out: Optional[torch.Tensor] = None,
    ws_o: Optional[torch.Tensor] = None,
    ws_ml: Optional[torch.Tensor] = None,
    stream=None,
) -> torch.Tensor:
    """Varlen paged attention with the streaming-decode visibility rule.

    ``q``: ``[n_tok, Hq, d]`` bf16; caches ``[num_pages, Hkv, P, d]`` bf16.
    Returns ``out`` ``[n_tok, Hq, d]`` bf16.
    """
    _cuda(q, k_cache, v_cache, q_pos, prompt_len, vis_base, vis_off, vis_words, block_tables, out)
    n_tok, hq, d = q.shape
    num_pages, hkv, page, d2 = k_cache.shape
    if d2 != d:
        raise ConfigError("paged_attention: head_dim mismatch between q and cache")
    if q.stride(-1) != 1 or q.stride(-2) != d:
        raise ConfigError("paged_attention: q must be [n_tok, Hq, d] with unit inner strides")
    if out is None:
        out = torch.empty((n_tok, hq, d), dtype=torch.bfloat16, device=q.device)
    if plan.n_partials > 0:
        need_o = plan.n_partials * 128 * d
        need_ml = plan.n_partials * 128 * 2
        if ws_o is None or ws_o.numel() < need_o:
            ws_o = torch.empty(need_o, dtype=torch.float32, device=q.device)
        if ws_ml is None or ws_ml.numel() < need_ml:
            ws_ml = torch.empty(need_ml, dtype=torch.float32, device=q.device)
    scale = float(sm_scale) if sm_scale is not None else 1.0 / float(d) ** 0.5
    st = _lib.call(
        "optimus_paged_attn",
        _ptr(q), q.stride(0), n_tok,
        _ptr(k_cache), _ptr(v_cache), num_pages,
        _ptr(q_pos), _ptr(prompt_len), _ptr(vis_base), _ptr(vis_off), _ptr(vis_words),
        _ptr(block_tables), block_tables.shape[1],
        _ptr(plan.work), _ptr(plan.cta_off), plan.grid if plan.n_work else 0,
        _ptr(plan.groups), plan.n_groups,
        block_size, hq, hkv, d, page, scale,
        _ptr(out), out.stride(0),
        _ptr(ws_o) if plan.n_partials else None, _ptr(ws_ml) if plan.n_partials else None,
        _v_dtype(v_cache), _stream(stream),
    )
    _lib.check(st, "optimus_paged_attn")
    return out


def paged_attention_append(
    q: torch.Tensor,
    k_new: torch.Tensor,
    v_new: torch.Tensor,
    k_cache: torch.Tensor,
    v_cache: torch.Tensor,
    q_pos: torch.Tensor,
    prompt_len: torch.Tensor,
    vis_base: torch.Tensor,
    vis_off: torch.Tensor,
    vis_words: torch.Tensor,
    block_tables: torch.Tensor,
    plan: AttnPlan,
    block_size: int,
    sm_scale: Optional[float] = None,
    out: Optional[torch.Tensor] = None,
    ws_o: Optional[torch.Tensor] = None,
    ws_ml: Optional[torch.Tensor] = None,
    slot_mapping_out: Optional[torch.Tensor] = None,
    slot_abs: Optional[torch.Tensor] = None,
    stream=None,
) -> torch.Tensor:
    """K1 folded into K2 (``optimus_paged_attn_append``): append ``k_new``/``v_new``
    ``[n_tok, Hkv, d]`` into the pages (rule S) and attend, in one launch.  Same
    result as :func:`kv_append` followed by :func:`paged_attention`; requires
    ``plan.single_tile`` (no request's query tokens span two MMA tiles).  ``slot_abs``:
    the step's :func:`slot_mapping` (else every launch re-derives the slots)."""
    _cuda(q, k_new, v_new, k_cache, v_cache, q_pos, prompt_len, vis_base, vis_off, vis_words,
          block_tables, out, slot_mapping_out)
    if not plan.single_tile:
        raise ConfigError("paged_attention_append: a request's query tokens span two query tiles "
                          "(chunk x Hq/Hkv > 128); use kv_append + paged_attention")
    n_tok, hq, d = q.shape
    num_pages, hkv, page, d2 = k_cache.shape
    if d2 != d or k_new.shape[-1] != d or k_new.shape[-2] != hkv:
        raise ConfigError("paged_attention_append: head_dim / kv-head mismatch")
    if q.stride(-1) != 1 or q.stride(-2) != d:
        raise ConfigError("paged_attention_append: q must be [n_tok, Hq, d] with unit inner strides")
    if k_new.stride() != v_new.stride() or k_new.stride(-1) != 1 or k_new.stride(-2) != d:
        raise ConfigError("paged_attention_append: k_new/v_new must be [n_tok, Hkv, d] with equal strides")
    if k_new.dtype != torch.bfloat16 or v_new.dtype != torch.bfloat16:
        raise ConfigError("paged_attention_append: k_new/v_new must be bf16")
    if slot_mapping_out is not None and (slot_mapping_out.dtype != torch.int64 or slot_mapping_out.numel() < n_tok):
        raise ConfigError("paged_attention_append: slot_mapping_out must be int64 [n_tok]")
    if out is None:
        out = torch.empty((n_tok, hq, d), dtype=torch.bfloat16, device=q.device)
    if plan.n_partials > 0:
        need_o = plan.n_partials * 128 * d
        need_ml = plan.n_partials * 128 * 2
        if ws_o is None or ws_o.numel() < need_o:
            ws_o = torch.empty(need_o, dtype=torch.float32, device=q.device)
        if ws_ml is None or ws_ml.numel() < need_ml:
            ws_ml = torch.empty(need_ml, dtype=torch.float32, device=q.device)
    scale = float(sm_scale) if sm_scale is not None else 1.0 / float(d) ** 0.5
    st = _lib.call(
        "optimus_paged_attn_append",
        _ptr(q), q.stride(0), n_tok,
        _ptr(k_new), _ptr(v_new), k_new.stride(0),
        _ptr(k_cache), _ptr(v_cache), num_pages,
        _ptr(q_pos), _ptr(prompt_len), _ptr(vis_base), _ptr(vis_off), _ptr(vis_words),
        _ptr(block_tables), block_tables.shape[1],
        _ptr(plan.work), _ptr(plan.cta_off), plan.grid if plan.n_work else 0,
        _ptr(plan.groups), plan.n_groups,
        block_size, hq, hkv, d, page, scale,
        _ptr(out), out.stride(0),
        _ptr(ws_o) if plan.n_partials else None, _ptr(ws_ml) if plan.n_partials else None,
        _v_dtype(v_cache), _ptr(slot_mapping_out) if slot_mapping_out is not None else None,
        _ptr(slot_abs), _stream(stream),
    )
    _lib.check(st, "optimus_paged_attn_append")
    return out


# --------------------------------------------------------------------------- K3
@dataclass
class UnmaskResult:
    commit_mask: torch.Tensor  # uint8 [n_rows]
    tokens: torch.Tensor       # int32 [n_rows]
    conf: torch.Tensor         # float32 [n_rows]


class VRangeGate:
    """fp16 V-cache range gate (``optimus_v_saturated``).  K1 stores bf16 V rows as
    fp16 (clamping |v| > 65504) and flags any clamp on the device; ``issue`` queues
    a copy of the flags into pinned memory (and clears them) on the stream, ``check``
    (after that stream synchronized) raises ``ConfigError`` if a value was clamped.
    The device flags are per process (a decoder clears them when it is created)."""

    def __init__(self):
        self.buf = torch.zeros(2, dtype=torch.int32, pin_memory=torch.cuda.is_available())

    def issue(self, stream=None) -> None:
        _lib.check(_lib.call("optimus_v_saturated", self.buf.data_ptr(), 1, _stream(stream)), "optimus_v_saturated")

    def check(self) -> None:
        if int(self.buf[0]) or int(self.buf[1]):
            self.buf.zero_()
            raise ConfigError("fp16 V cache: V values beyond +-65504 were clamped (cvt.satfinite); this model's "
                              "V range needs a bf16 V cache (DecodeConfig(v_dtype=torch.bfloat16))")


def unmask_splits(n_rows: int, vocab: int) -> int:
    return int(_lib.call("optimus_unmask_splits", n_rows, vocab))


def unmask_partials(
    logits: torch.Tensor,
    row_src: Optional[torch.Tensor],
    n_rows: int,
    n_vsplit: int,
    vocab_offset: int = 0,
    part: Optional[torch.Tensor] = None,
    stream=None,
) -> torch.Tensor:
    """Phase (a): per (row, vocab split) ``{max, sumexp, argmax}`` records."""
    _cuda(logits, row_src, part)
    if logits.dtype == torch.bfloat16:
        dt = 0
    elif logits.dtype == torch.float32:
        dt = 1
    else:
        raise ConfigError("unmask: logits must be bf16 or fp32")
    if logits.stride(-1) != 1:
        raise ConfigError("unmask: logits rows must be contiguous")
    vocab = logits.shape[-1]
    if part is None:
        part = torch.empty((max(n_rows, 1), n_vsplit, 3), dtype=torch.float32, device=logits.device)
    st = _lib.call(
        "optimus_unmask_partials", _ptr(logits), dt, logits.stride(0), _ptr(row_src),
        n_rows, vocab, vocab_offset, n_vsplit, _ptr(part), _stream(stream),
    )
    _lib.check(st, "optimus_unmask_partials")
    return part


def lmhead_unmask_partials(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    vocab_offset: int = 0,
    part: Optional[torch.Tensor] = None,
    stream=None,
    merge: bool = False,
    merged: Optional[torch.Tensor] = None,
) -> torch.Tensor:
    """f3: the LM head ``hidden @ weight.T`` reduced straight to the unmask partials
    (``optimus_lmhead_unmask_partials``); the logits are never materialised.
    Returns part ``[n_rows, optimus_lmhead_splits(vocab), 3]`` for ``unmask_finalize``,
    or with ``merge`` the per-row merge of the vocab tiles, ``[n_rows, 1, 3]``."""
    _cuda(hidden, weight, part)
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise ConfigError("lmhead: hidden and weight must be bf16")
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise ConfigError("lmhead: hidden [rows, K] and weight [vocab, K] must share K")
    if hidden.stride(-1) != 1 or weight.stride(-1) != 1:
        raise ConfigError("lmhead: rows must be contiguous")
    n_rows, k = hidden.shape
    vocab = weight.shape[0]
    n_vt = int(_lib.call("optimus_lmhead_splits", vocab))
    if part is None:
        part = torch.empty((max(n_rows, 1), n_vt, 3), dtype=torch.float32, device=hidden.device)
    st = _lib.call("optimus_lmhead_unmask_partials", _ptr(hidden), hidden.stride(0), n_rows, _ptr(weight),
                   weight.stride(0), vocab, k, vocab_offset, _ptr(part), _stream(stream))
    _lib.check(st, "optimus_lmhead_unmask_partials")
    if not merge:
        return part
    if merged is None:
        merged = torch.empty((max(n_rows, 1), 1, 3), dtype=torch.float32, device=hidden.device)
    st = _lib.call("optimus_unmask_merge_splits", _ptr(part), n_rows, n_vt, _ptr(merged), _stream(stream))
    _lib.check(st, "optimus_unmask_merge_splits")
    return merged


def lmhead_unmask_commit(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    cu_rows: torch.Tensor,
    tau: float = 0.9,
    fallback: str = "earliest",
    row_pos: Optional[torch.Tensor] = None,
    state: Optional[torch.Tensor] = None,
    token_buf: Optional[torch.Tensor] = None,
    stream=None,
) -> "UnmaskResult":
    """K3 from hidden states (f3): fused LM head -> per-row merge -> threshold and
    progress rule.  Same result contract as ``unmask_commit`` on the logits
    ``hidden @ weight.T`` (computed here in fp32, never stored)."""
    n_rows = hidden.shape[0]
    merged = lmhead_unmask_partials(hidden, weight, merge=True, stream=stream)
    return unmask_finalize(merged, 1, n_rows, 1, cu_rows, tau, fallback, row_pos=row_pos, state=state,
                           token_buf=token_buf, stream=stream)


def unmask_finalize(
    part: torch.Tensor,
    n_outer: int,
    n_rows: int,
    n_vsplit: int,
    cu_rows: torch.Tensor,
    tau: float,
    fallback: str = "earliest",
    row_pos: Optional[torch.Tensor] = None,
    state: Optional[torch.Tensor] = None,
    token_buf: Optional[torch.Tensor] = None,
    result: Optional[UnmaskResult] = None,
    stream=None,
) -> UnmaskResult:
    """Phase (b): merge partials, threshold at ``tau``, apply the progress rule."""
    _cuda(part, cu_rows, row_pos, state, token_buf)
    if fallback not in FALLBACK_MODES:
        raise ConfigError(f"unknown fallback mode {fallback!r}")
    dev = part.device
    if result is None:
        result = UnmaskResult(
            torch.empty(max(n_rows, 1), dtype=torch.uint8, device=dev),
            torch.empty(max(n_rows, 1), dtype=torch.int32, device=dev),
            torch.empty(max(n_rows, 1), dtype=torch.float32, device=dev),
        )
    n_req = cu_rows.shape[0] - 1
    st = _lib.call(
        "optimus_unmask_finalize", _ptr(part), n_outer, n_rows, n_vsplit, _ptr(cu_rows), n_req,
        float(tau), FALLBACK_MODES[fallback], _ptr(result.commit_mask), _ptr(result.tokens),
        _ptr(result.conf), _ptr(row_pos), _ptr(state), _ptr(token_buf),
        (state if state is not None else token_buf).stride(0) if (state is not None or token_buf is not None) else 0, _stream(stream),
    )
    _lib.check(st, "optimus_unmask_finalize")
    return result


def unmask_fused(
    logits: torch.Tensor,
    row_src: Optional[torch.Tensor],
    n_rows: int,
    n_vsplit: int,
    cu_rows: torch.Tensor,
    row_req: torch.Tensor,
    counters: torch.Tensor,
    tau: float,
    fallback: str = "earliest",
    row_pos: Optional[torch.Tensor] = None,
    state: Optional[torch.Tensor] = None,
    token_buf: Optional[torch.Tensor] = None,
    result: Optional[UnmaskResult] = None,
    part: Optional[torch.Tensor] = None,
    n_rows_dev: Optional[torch.Tensor] = None,
    stream=None,
) -> UnmaskResult:
    """K3 in one launch (``optimus_unmask_commit``): phases (a) and (b) fused on one
    vocab shard.  ``counters`` is an int32 [n_req] workspace, zero between calls."""
    _cuda(logits, row_src, cu_rows, row_req, counters, row_pos, state, token_buf, part, n_rows_dev)
    if logits.dtype == torch.bfloat16:
        dt = 0
    elif logits.dtype == torch.float32:
        dt = 1
    else:
        raise ConfigError("unmask: logits must be bf16 or fp32")
    if logits.stride(-1) != 1:
        raise ConfigError("unmask: logits rows must be contiguous")
    if fallback not in FALLBACK_MODES:
        raise ConfigError(f"unknown fallback mode {fallback!r}")
    n_req = cu_rows.shape[0] - 1
    if counters.dtype != torch.int32 or counters.numel() < n_req:
        raise ConfigError("unmask: counters must be int32 with >= n_req entries")
    dev = logits.device
    rows = max(n_rows, 1)
    if part is None:
        part = torch.empty((rows, n_vsplit, 3), dtype=torch.float32, device=dev)
    if result is None:
        result = UnmaskResult(torch.empty(rows, dtype=torch.uint8, device=dev),
                              torch.empty(rows, dtype=torch.int32, device=dev),
                              torch.empty(rows, dtype=torch.float32, device=dev))
    st = _lib.call(
        "optimus_unmask_commit", _ptr(logits), dt, logits.stride(0), _ptr(row_src), n_rows, _ptr(n_rows_dev),
        logits.shape[-1], n_vsplit, _ptr(part), _ptr(cu_rows), _ptr(row_req), n_req, _ptr(counters), float(tau),
        FALLBACK_MODES[fallback], _ptr(result.commit_mask), _ptr(result.tokens), _ptr(result.conf), _ptr(row_pos),
        _ptr(state), _ptr(token_buf), (state if state is not None else token_buf).stride(0) if (state is not None or token_buf is not None) else 0, _stream(stream),
    )
    _lib.check(st, "optimus_unmask_commit")
    return result


def unmask_commit(
    logits: torch.Tensor,
    cu_rows: torch.Tensor,
    tau: float = 0.9,
    fallback: str = "earliest",
    row_src: Optional[torch.Tensor] = None,
    n_rows: Optional[int] = None,
    n_vsplit: Optional[int] = None,
    stream=None,
) -> UnmaskResult:
    """Single-GPU K3 over the whole vocabulary, one launch (``unmask_fused``)."""
    if n_rows is None:
        n_rows = logits.shape[0] if row_src is None else row_src.shape[0]
    if n_vsplit is None:
        n_vsplit = unmask_splits(n_rows, logits.shape[-1])
    n_req = cu_rows.shape[0] - 1
    counts = (cu_rows[1:] - cu_rows[:-1]).long()
    row_req = torch.repeat_interleave(torch.arange(n_req, dtype=torch.int32, device=cu_rows.device), counts,
                                      output_size=n_rows)
    counters = torch.zeros(max(n_req, 1), dtype=torch.int32, device=cu_rows.device)
    return unmask_fused(logits, row_src, n_rows, n_vsplit, cu_rows, row_req, counters, tau, fallback,
                        stream=stream)
