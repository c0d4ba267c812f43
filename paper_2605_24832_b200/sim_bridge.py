"""dllmsim's own simulation loop with ONE B200 device step per decode iteration.

The reference loop asks the commit oracle one request at a time
(``_Loop.run_decode``, sim.py:269-291: plan_chunk -> oracle.commits -> apply_chunk
per request).  With the B200 oracle behind ``Scenario.oracle_factory`` that is one
device step per request.  ``BatchedLoop`` is the reference loop itself (subclass,
nothing re-implemented) with one addition at the top of each chunked decode
iteration: it plans the whole batch with the reference's ``plan_chunk`` and the
chunk the loop is about to choose (``_choose_chunk`` / ``FixedChunk.chunk_size``,
both pure functions of the loop state), hands the plans to
``oracle.commits_batch`` — one device step (K1 -> K2 per layer -> K3) for the
batch, kv-only plans included — and then lets the reference's per-request loop
run unchanged: each of its ``oracle.commits(req, window)`` calls is answered from
the batch result.  Every request's plan and commit set is therefore exactly what
the per-request loop would compute; only the number of device launches changes.

Policies without a chunked streaming branch (AR, FixedBlock, BlockLevelBatch) run
the reference loop as is.
"""

from __future__ import annotations

from .errors import ConfigError

try:
    from dllmsim import sim as _sim
    from dllmsim.engine import plan_chunk as _plan_chunk
    from dllmsim.scheduler import ElasticChunk, FixedChunk
except ImportError as e:  # pragma: no cover - depends on the install
    raise ConfigError("sim_bridge needs the reference package dllmsim "
                      "(pip install --target baseline/_ref /root/reference/pkg)") from e


class BatchedLoop(_sim._Loop):
    """``dllmsim.sim._Loop`` with the batch's commits computed in one device step."""

    def run_decode(self) -> None:
        policy = self.policy
        batch_fn = getattr(self.oracle, "commits_batch", None)
        if batch_fn is not None and isinstance(policy, (FixedChunk, ElasticChunk)) and self.active:
            batch = list(self.active)
            chunk = self._choose_chunk(len(batch)) if isinstance(policy, ElasticChunk) else policy.chunk_size
            plans = [_plan_chunk(r, chunk, policy.block_size, policy.window_rule) for r in batch]
            batch_fn(batch, plans)
        super().run_decode()


def run(scenario):
    """``dllmsim.sim.run`` with one device step per decode iteration."""
    return BatchedLoop(scenario).run()
