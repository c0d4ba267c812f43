"""Packed per-slot decode state shared by Python request objects and native code.

The reference keeps each request's decode state on its ``Request`` object
(``core.py:72-116``): ``states`` (int8 per output position), the FIFO
``uncached_queue`` deque, and the ``block_index`` / ``committed`` /
``steps_taken`` counters.  For the native batched step (csrc/host_step.cu) the
same state lives in packed arrays indexed by batch slot.  A request admitted
into a ``BatchState`` is *rebound*: its class is swapped for a subclass whose
fields are properties over the arrays (``states`` becomes a row view, the queue a
deque-compatible ``RingQueue``).  So the reference functions (``plan_chunk`` /
``apply_chunk``, ours or dllmsim's) and the native planner see and mutate one
state, with no per-step copy.  ``release`` copies the state back onto the
object and restores its class.
"""

from __future__ import annotations

from typing import Dict, Iterable

import numpy as np

from .core import TokenState
from .errors import ConfigError


class RingQueue:
    """deque-compatible view of one slot's FIFO ring (popleft/append/extend/iter)."""

    __slots__ = ("_bs", "_slot")

    def __init__(self, bs: "BatchState", slot: int):
        self._bs = bs
        self._slot = slot

    def __len__(self) -> int:
        return int(self._bs.q_len[self._slot])

    def __iter__(self):
        bs, s = self._bs, self._slot
        h, n, cap = int(bs.q_head[s]), int(bs.q_len[s]), bs.qcap
        row = bs.queue[s]
        for i in range(n):
            yield int(row[(h + i) % cap])

    def __getitem__(self, i: int) -> int:
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("deque index out of range")
        bs, s = self._bs, self._slot
        return int(bs.queue[s][(int(bs.q_head[s]) + i) % bs.qcap])

    def popleft(self) -> int:
        bs, s = self._bs, self._slot
        if bs.q_len[s] == 0:
            raise IndexError("pop from an empty deque")
        v = int(bs.queue[s][bs.q_head[s]])
        bs.q_head[s] = (bs.q_head[s] + 1) % bs.qcap
        bs.q_len[s] -= 1
        return v

    def append(self, p: int) -> None:
        bs, s = self._bs, self._slot
        if bs.q_len[s] >= bs.qcap:
            raise ConfigError("uncached queue capacity exceeded")
        bs.queue[s][(bs.q_head[s] + bs.q_len[s]) % bs.qcap] = int(p)
        bs.q_len[s] += 1

    def extend(self, it: Iterable[int]) -> None:
        for p in it:
            self.append(p)

    def clear(self) -> None:
        self._bs.q_len[self._slot] = 0

    def __eq__(self, other) -> bool:
        return list(self) == list(other)

    def __repr__(self) -> str:
        return f"RingQueue({list(self)!r})"


def _int_field(name: str):
    def get(self):
        return int(getattr(self._bs, name)[self._slot])

    def set_(self, v):
        getattr(self._bs, name)[self._slot] = int(v)

    return property(get, set_)


class _Bound:
    """Mixin: request fields backed by a BatchState slot."""

    block_index = _int_field("block_index")
    committed = _int_field("committed")
    steps_taken = _int_field("steps_taken")

    @property
    def states(self):
        return self._bs.states[self._slot, : self._out]

    @states.setter
    def states(self, v):
        self._bs.states[self._slot, : self._out] = np.asarray(v, dtype=np.int8)

    @property
    def uncached_queue(self):
        return RingQueue(self._bs, self._slot)

    @uncached_queue.setter
    def uncached_queue(self, v):
        q = RingQueue(self._bs, self._slot)
        q.clear()
        q.extend(v)


_BOUND_CLASSES: Dict[type, type] = {}


def _bound_class(cls: type) -> type:
    sub = _BOUND_CLASSES.get(cls)
    if sub is None:
        sub = type(f"Slot{cls.__name__}", (_Bound, cls), {})
        _BOUND_CLASSES[cls] = sub
    return sub


class BatchState:
    """Packed state for up to ``max_slots`` requests of at most ``max_out`` tokens."""

    FIELDS = ("q_head", "q_len", "block_index", "committed", "steps_taken", "cached_prefix",
              "prompt", "out_len")

    def __init__(self, max_slots: int, max_out: int, qcap: int = 256):
        self.max_slots = max_slots
        self.max_out = max_out
        self.qcap = qcap
        # rows padded to 16 bytes: the device planner stages a row with 16-byte loads
        self.states = np.zeros((max_slots, (max_out + 15) // 16 * 16), dtype=np.int8)
        self.queue = np.zeros((max_slots, qcap), dtype=np.int32)
        for f in self.FIELDS:
            setattr(self, f, np.zeros(max_slots, dtype=np.int32))
        self._req: Dict[int, object] = {}

    def bind(self, req, slot: int) -> None:
        out = int(req.output_tokens)
        if out > self.max_out:
            raise ConfigError(f"output_tokens {out} > BatchState max_out {self.max_out}")
        q = list(req.uncached_queue)
        if len(q) > self.qcap:
            raise ConfigError("uncached queue longer than the ring capacity")
        st = np.asarray(req.states, dtype=np.int8)
        self.states[slot, :out] = st
        self.states[slot, out:] = 0
        self.queue[slot, : len(q)] = q
        self.q_head[slot] = 0
        self.q_len[slot] = len(q)
        self.block_index[slot] = req.block_index
        self.committed[slot] = req.committed
        self.steps_taken[slot] = req.steps_taken
        self.prompt[slot] = req.prompt_tokens
        self.out_len[slot] = out
        cp = np.flatnonzero(st != TokenState.DECODED_CACHED)
        self.cached_prefix[slot] = int(cp[0]) if cp.size else out
        d = req.__dict__
        for name in ("states", "uncached_queue", "block_index", "committed", "steps_taken"):
            d.pop(name, None)
        d["_bs"], d["_slot"], d["_out"] = self, slot, out
        req.__class__ = _bound_class(type(req))
        self._req[slot] = req

    def unbind(self, slot: int):
        req = self._req.pop(slot)
        base = type(req).__mro__[2]  # SlotX -> (_Bound, X)
        states = self.states[slot, : req._out].copy()
        queue = list(RingQueue(self, slot))
        counters = (int(self.block_index[slot]), int(self.committed[slot]), int(self.steps_taken[slot]))
        req.__class__ = base
        d = req.__dict__
        for name in ("_bs", "_slot", "_out"):
            d.pop(name, None)
        from collections import deque

        d["states"] = states
        d["uncached_queue"] = deque(queue)
        d["block_index"], d["committed"], d["steps_taken"] = counters
        return req
