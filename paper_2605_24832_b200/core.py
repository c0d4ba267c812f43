"""Per-request decode state: the host objects the B200 path keeps in sync.

These mirror the reference's value types so a caller written against
``dllmsim`` can hand its own objects to this package unchanged:

* ``TokenState`` — ``core.py:21-31`` (MASKED=0 -> DECODED_UNCACHED=1 ->
  DECODED_CACHED=2, monotone).
* ``WindowRule`` — ``core.py:34-38`` (``in_block`` / ``out_block``).
* ``Request`` — ``core.py:72-116``: per-request ``states`` (int8 per output
  position), FIFO ``uncached_queue`` of decoded-but-not-recomputed positions,
  ``block_index``, ``committed``, ``steps_taken``.

Positions are output-relative (``core.py:3-4``): position ``p`` is the p-th
generated token; its absolute sequence position in the KV cache is
``prompt_tokens + p`` (SURVEY §8c rule S).

Every function in this package that takes a request is duck-typed on these
attribute names, so ``dllmsim.Request`` objects work as well.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from enum import Enum, IntEnum
from typing import Optional

import numpy as np

from .errors import ConfigError


class TokenState(IntEnum):
    """Lifecycle of one generated position (reference ``core.py:21-31``)."""

    MASKED = 0
    DECODED_UNCACHED = 1
    DECODED_CACHED = 2


class WindowRule(Enum):
    """Where the decode window draws masked positions (``core.py:34-38``)."""

    IN_BLOCK = "in_block"
    OUT_BLOCK = "out_block"


def rule_value(rule) -> str:
    """Normalise a window rule (ours, dllmsim's, or a string) to its value."""
    if isinstance(rule, str):
        v = rule
    else:
        v = getattr(rule, "value", None)
    if v not in ("in_block", "out_block"):
        raise ConfigError(f"unknown window rule {rule!r}")
    return v


@dataclass
class Request:
    """One request's mutable decode state (reference ``core.py:72-116``)."""

    id: int
    arrival_time: float
    prompt_tokens: int
    output_tokens: int
    rng: Optional[np.random.Generator] = None
    rate_multiplier: float = 1.0
    committed: int = 0
    block_index: int = 0
    states: np.ndarray = field(default=None, repr=False)  # type: ignore[assignment]
    uncached_queue: deque = field(default_factory=deque, repr=False)
    steps_taken: int = 0
    prefill_done_time: Optional[float] = None
    first_token_time: Optional[float] = None
    finish_time: Optional[float] = None

    def __post_init__(self) -> None:
        if self.prompt_tokens < 1:
            raise ConfigError(f"prompt_tokens must be >= 1, got {self.prompt_tokens}")
        if self.output_tokens < 1:
            raise ConfigError(f"output_tokens must be >= 1, got {self.output_tokens}")
        if self.states is None:
            self.states = np.zeros(self.output_tokens, dtype=np.int8)
        if self.rng is None:
            self.rng = np.random.default_rng(self.id)

    @property
    def finished(self) -> bool:
        return self.committed >= self.output_tokens

    def block_span(self, block_size: int) -> tuple[int, int]:
        return block_span(self, block_size)

    def advance_blocks(self, block_size: int) -> None:
        advance_blocks(self, block_size)


def block_span(request, block_size: int) -> tuple[int, int]:
    """Half-open current block ``[kB, min(kB+B, out))`` (``core.py:103-107``)."""
    start = request.block_index * block_size
    return start, min(start + block_size, request.output_tokens)


def advance_blocks(request, block_size: int) -> None:
    """Skip every block that holds no MASKED position (``core.py:109-116``).

    A block counts as done once all its positions are decoded — cached or
    not; the loop stops at a finished request.
    """
    states = request.states
    out = request.output_tokens
    while request.committed < out:
        lo = request.block_index * block_size
        hi = min(lo + block_size, out)
        if (states[lo:hi] == TokenState.MASKED).any():
            return
        request.block_index += 1


__all__ = [
    "TokenState",
    "WindowRule",
    "Request",
    "rule_value",
    "block_span",
    "advance_blocks",
]
