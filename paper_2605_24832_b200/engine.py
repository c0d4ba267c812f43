"""Chunk planning and commit application — the control half of the hot path.

``plan_chunk`` / ``apply_chunk`` keep the reference's signatures and error
behaviour (``pkg/src/dllmsim/engine.py:45-95``):

* a plan retires the *oldest* ``min(|backlog|, c)`` decoded-but-uncached
  positions first (``engine.py:58``), then fills the leftover capacity with the
  earliest MASKED positions of the current block (IN_BLOCK, ``:60-62``) or of
  the whole output capped at ``block_size`` (OUT_BLOCK, ``:63-66``);
* applying a plan validates commits against the window (``:70-76``), moves the
  planned KV positions to DECODED_CACHED in FIFO order (``:84-88``), moves the
  commits (ascending) to DECODED_UNCACHED and appends them to the backlog
  (``:89-91``), bumps the counters and advances the block (``:92-94``).

``plan_batch`` / ``apply_batch`` are the batched twins used by the B200
decode step: they produce exactly the per-request plans (same tuples, same
order) but do the masked-position search with one vectorised pass per request
and skip the Python-level ``islice``/``nonzero`` round trips — the host side of
SURVEY §8f-1.  They are checked against ``plan_chunk`` in the tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from .core import TokenState, advance_blocks, rule_value
from .errors import ChunkTooSmall, EmptyWindow, IllegalCommit


@dataclass(frozen=True)
class StepSummary:
    """Outcome of one step of one request (reference ``engine.py:20-25``)."""

    computed: int
    commits: frozenset = field(default_factory=frozenset)


@dataclass(frozen=True)
class ChunkPlan:
    """Query tokens of one request for one step (reference ``engine.py:28-37``).

    ``kv_positions`` are recomputed with their committed token ids (they
    produce final KV); ``window`` positions are fed the MASK token and are the
    rows the unmask kernel scores.  Query order is kv first, then window.
    """

    kv_positions: tuple
    window: tuple

    @property
    def computed(self) -> int:
        return len(self.kv_positions) + len(self.window)


def _masked_positions(states: np.ndarray, lo: int, hi: int, limit: int) -> tuple:
    if limit <= 0 or hi <= lo:
        return ()
    idx = np.flatnonzero(states[lo:hi] == TokenState.MASKED)
    if idx.size > limit:
        idx = idx[:limit]
    return tuple((idx + lo).tolist())


def plan_chunk(request, chunk_size: int, block_size: int, window_rule="in_block") -> ChunkPlan:
    """Backlog first, then earliest masked positions (``engine.py:45-67``)."""
    if chunk_size < 2:
        raise ChunkTooSmall(f"chunk_size must be >= 2, got {chunk_size}")
    queue = request.uncached_queue
    n_kv = min(len(queue), chunk_size)
    kv = tuple(queue[i] for i in range(n_kv)) if n_kv else ()
    room = chunk_size - n_kv
    if rule_value(window_rule) == "in_block":
        lo = request.block_index * block_size
        hi = min(lo + block_size, request.output_tokens)
        window = _masked_positions(request.states, lo, hi, room)
    else:
        window = _masked_positions(
            request.states, 0, request.output_tokens, min(room, block_size)
        )
    return ChunkPlan(kv_positions=kv, window=window)


def check_commits(request, window: Sequence[int], commits: Iterable[int]) -> None:
    """Reject commits outside the window or of decoded positions (``:70-76``)."""
    allowed = set(window)
    states = request.states
    for p in commits:
        if p not in allowed:
            raise IllegalCommit(f"position {p} not in the decode window")
        if states[p] != TokenState.MASKED:
            raise IllegalCommit(f"position {p} already decoded")


def apply_chunk(request, plan: ChunkPlan, commits, block_size: int) -> StepSummary:
    """Retire the planned KV backlog, then apply commits (``engine.py:79-95``)."""
    check_commits(request, plan.window, commits)
    queue = request.uncached_queue
    states = request.states
    for p in plan.kv_positions:
        head = queue.popleft()
        if head != p:
            raise IllegalCommit(f"KV plan out of order: {head} != {p}")
        states[p] = TokenState.DECODED_CACHED
    ordered = sorted(commits)
    for p in ordered:
        states[p] = TokenState.DECODED_UNCACHED
    queue.extend(ordered)
    request.committed += len(ordered)
    request.steps_taken += 1
    advance_blocks(request, block_size)
    return StepSummary(computed=plan.computed, commits=frozenset(ordered))


def plan_batch(requests, chunk_size, block_size: int, window_rule="in_block") -> list:
    """``plan_chunk`` for every request of a batch (identical plans).

    ``chunk_size`` is one size for the batch (the reference's global chunk,
    sim.py:270-274) or a sequence with one size per request (mixed chunks)."""
    sizes = list(chunk_size) if np.ndim(chunk_size) else [chunk_size] * len(requests)
    if any(c < 2 for c in sizes):
        raise ChunkTooSmall(f"chunk_size must be >= 2, got {min(sizes)}")
    in_block = rule_value(window_rule) == "in_block"
    plans = []
    for req, chunk_size in zip(requests, sizes):
        queue = req.uncached_queue
        n_kv = min(len(queue), chunk_size)
        kv = tuple(queue[i] for i in range(n_kv)) if n_kv else ()
        room = chunk_size - n_kv
        if in_block:
            lo = req.block_index * block_size
            hi = min(lo + block_size, req.output_tokens)
            window = _masked_positions(req.states, lo, hi, room)
        else:
            window = _masked_positions(req.states, 0, req.output_tokens, min(room, block_size))
        plans.append(ChunkPlan(kv, window))
    return plans


def apply_batch(requests, plans, commit_sets, block_size: int) -> list:
    """``apply_chunk`` for every request of a batch, same validation."""
    return [
        apply_chunk(req, plan, commits, block_size)
        for req, plan, commits in zip(requests, plans, commit_sets)
    ]


# --------------------------------------------------------------------------- baselines
# The paper's comparison modes on the same kernels: a whole-block
# denoise step (BD), a prefix-cached block step and an autoregressive step, with the
# reference's state rules and computed counts (engine.py:98-157).  ``plan_block``
# gives the device step's query tokens (kv = positions recomputed with their
# committed ids, window = the MASK rows the unmask scores); ``apply_block`` applies
# the device's commits exactly as the reference step applies its oracle's.
BASELINE_MODES = ("bd", "prefix", "ar")


def plan_block(request, block_size: int, mode: str) -> ChunkPlan:
    """Query tokens of one baseline step.

    ``bd``: the whole block extent — every decoded position of the block is
    recomputed, the masked ones are the window (engine.py:98-102).
    ``prefix``: cached positions are reused; the block's uncached positions are
    recomputed and its masked positions are the window (engine.py:120-131).
    ``ar``: one row, the next position (engine.py:148-151)."""
    if mode == "ar":
        p = request.committed
        if p >= request.output_tokens:
            raise EmptyWindow(f"request {request.id} is already finished")
        return ChunkPlan(kv_positions=(), window=(p,))
    if mode not in ("bd", "prefix"):
        raise ValueError(f"unknown baseline mode {mode!r}")
    lo = request.block_index * block_size
    hi = min(lo + block_size, request.output_tokens)
    span = request.states[lo:hi]
    window = tuple((np.flatnonzero(span == TokenState.MASKED) + lo).tolist())
    if not window:
        raise EmptyWindow(f"request {request.id} has no masked token in its block")
    if mode == "bd":
        kv = tuple((np.flatnonzero(span != TokenState.MASKED) + lo).tolist())
    else:
        kv = tuple((np.flatnonzero(span == TokenState.DECODED_UNCACHED) + lo).tolist())
    return ChunkPlan(kv_positions=kv, window=window)


def apply_block(request, plan: ChunkPlan, commits, block_size: int, mode: str) -> StepSummary:
    """The reference baseline step's state update for the given commits."""
    states = request.states
    if mode == "ar":
        p = plan.window[0]
        states[p] = TokenState.DECODED_CACHED
        request.committed += 1
        request.steps_taken += 1
        advance_blocks(request, 1)
        return StepSummary(computed=1, commits=frozenset({p}))
    lo = request.block_index * block_size
    hi = min(lo + block_size, request.output_tokens)
    check_commits(request, plan.window, commits)
    if mode == "bd":
        extent = hi - lo
        for p in commits:
            states[p] = TokenState.DECODED_UNCACHED
        request.committed += len(commits)
        request.steps_taken += 1
        while np.all(states[lo:hi] != TokenState.MASKED):
            states[lo:hi] = TokenState.DECODED_CACHED
            advance_blocks(request, block_size)
            if request.finished:
                break
            lo = request.block_index * block_size
            hi = min(lo + block_size, request.output_tokens)
        return StepSummary(computed=extent, commits=frozenset(commits))
    span = states[lo:hi]
    cached = int(np.count_nonzero(span == TokenState.DECODED_CACHED))
    uncached = int(np.count_nonzero(span == TokenState.DECODED_UNCACHED))
    computed = (hi - lo) - cached + uncached
    for p in commits:
        states[p] = TokenState.DECODED_CACHED
    request.committed += len(commits)
    request.steps_taken += 1
    advance_blocks(request, block_size)
    return StepSummary(computed=computed, commits=frozenset(commits))


def block_diffusion_step(request, oracle, block_size: int) -> StepSummary:
    """Reference signature (engine.py:98): one full-block denoise step."""
    plan = plan_block(request, block_size, "bd")
    commits = oracle.commits(request, list(plan.window))
    summary = apply_block(request, plan, commits, block_size, "bd")
    if hasattr(oracle, "consume"):
        oracle.consume(request, commits)
    return summary


def prefix_cached_step(request, oracle, block_size: int) -> StepSummary:
    """Reference signature (engine.py:120): block step reusing cached positions."""
    plan = plan_block(request, block_size, "prefix")
    commits = oracle.commits(request, list(plan.window))
    summary = apply_block(request, plan, commits, block_size, "prefix")
    if hasattr(oracle, "consume"):
        oracle.consume(request, commits)
    return summary


def ar_step(request) -> StepSummary:
    """Reference signature (engine.py:148): the next position commits and caches."""
    return apply_block(request, plan_block(request, 1, "ar"), None, 1, "ar")


__all__ = [
    "BASELINE_MODES",
    "plan_block",
    "apply_block",
    "block_diffusion_step",
    "prefix_cached_step",
    "ar_step",
    "StepSummary",
    "ChunkPlan",
    "plan_chunk",
    "apply_chunk",
    "check_commits",
    "plan_batch",
    "apply_batch",
]
