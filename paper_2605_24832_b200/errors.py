"""Error hierarchy of the B200 decode path.

Mirrors the reference's exception tree (``pkg/src/dllmsim/errors.py:4-57``) so
code written against ``dllmsim`` keeps its ``except`` clauses: every error is a
``SimulatorError``; ``ConfigError`` is a bad knob or shape; ``IllegalCommit`` /
``ChunkTooSmall`` / ``EmptyWindow`` keep their meaning from the decode engine
(``engine.py:56-57,70-76,84-88``).  ``DeviceError`` is new: a CUDA entry point
of the C-ABI library returned a non-zero status.

When ``dllmsim`` itself is importable, its classes are reused so that an
``except dllmsim.IllegalCommit`` clause catches errors raised here too.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on whether the reference package is installed
    from dllmsim.errors import (  # type: ignore
        ChunkTooSmall,
        ConfigError,
        DegenerateIteration,
        EmptyWindow,
        IllegalCommit,
        RequestComplete,
        SimulatorError,
        TraceExhausted,
    )
except Exception:  # the reference is not installed (e.g. on the GPU box)

    class SimulatorError(Exception):
        """Root of every package error (reference ``errors.py:4``)."""

    class ConfigError(SimulatorError):
        """Malformed knob, shape or configuration (``errors.py:8``)."""

    class EmptyWindow(SimulatorError):
        """A commit decision was requested for an empty window (``errors.py:12``)."""

    class TraceExhausted(SimulatorError):
        """A replay trace has no entry for the requested step (``errors.py:20``)."""

    class RequestComplete(SimulatorError):
        """A step was planned for a finished request (``errors.py:24``)."""

    class IllegalCommit(SimulatorError):
        """Commit outside the window, double commit, or KV plan out of order."""

    class ChunkTooSmall(SimulatorError):
        """Chunk sizes below 2 cannot make progress (``errors.py:36``)."""

    class DegenerateIteration(SimulatorError):
        """The decode loop stopped making progress (``errors.py:44``)."""


class DeviceError(SimulatorError):
    """A B200 kernel entry point reported a CUDA or argument error."""

    def __init__(self, entry: str, status: int, detail: str = ""):
        self.entry = entry
        self.status = status
        msg = f"{entry} failed with status {status}"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)


class ExtensionMissing(SimulatorError):
    """The sm_100a C-ABI library is not built or could not be loaded.

    Raised instead of falling back to any CPU path: the product has none.
    """


__all__ = [
    "SimulatorError",
    "ConfigError",
    "EmptyWindow",
    "TraceExhausted",
    "RequestComplete",
    "IllegalCommit",
    "ChunkTooSmall",
    "DegenerateIteration",
    "DeviceError",
    "ExtensionMissing",
]
