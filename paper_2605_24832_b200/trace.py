"""Record the commits of batched B200 steps as the reference's commit trace
("record/replay GPU commit traces via CommitTrace JSONL").

The trace format, its validation and the replaying oracle are the reference's own
classes (``dllmsim.commit.CommitTrace`` / ``ReplayOracle``, commit.py:205-312); this
module only adds the recorder that feeds them from ``StreamingDecoder.step`` /
``DeviceLoop.step``, so a trace of the K3 decisions of a real or synthetic model on
the B200 replays the decode in the simulator exactly (``tests/test_trace.py``,
``tests/test_device_loop_gpu.py``).
"""

from __future__ import annotations

from typing import Dict, Optional

from .errors import ConfigError


def commit_trace_cls():
    """``dllmsim.commit.CommitTrace``; the reference package must be importable."""
    try:
        from dllmsim.commit import CommitTrace
    except ImportError as e:  # pragma: no cover - depends on the install
        raise ConfigError("commit traces need the reference package dllmsim "
                          "(pip install --target baseline/_ref /root/reference/pkg)") from e
    return CommitTrace


class TraceRecorder:
    """Records the commits of batched B200 steps into a ``CommitTrace``.

    Call ``before(requests)`` ahead of a step and ``after(requests, summaries)``
    with the step's ``StepSummary`` list (``StreamingDecoder.step`` order, or the
    ``DeviceLoop`` positions): step k of request r is r.steps_taken before the
    step, exactly the index the reference's loop records (``sim.py:269-305``).
    Requests that did not take a step (no computed tokens) are skipped."""

    def __init__(self, trace=None):
        self.trace = trace if trace is not None else commit_trace_cls()()
        self._k: Dict[int, int] = {}

    def before(self, requests) -> None:
        self._k = {r.id: int(r.steps_taken) for r in requests}

    def after(self, requests, summaries) -> None:
        for r, s in zip(requests, summaries):
            k: Optional[int] = self._k.get(r.id)
            if k is None or int(r.steps_taken) == k:
                continue  # not stepped (finished, or a position admitted mid-flight)
            self.trace.record(r.id, k, s.commits)
