"""The B200 oracle's seam into dllmsim (Scenario.oracle_factory, sim.py:64,128-132),
run inside the reference's own loop on CPU with the device step replaced by a
recording stub.  What is checked is the host half of the seam:

* rule K through the loop: every committed position is recomputed as a kv row
  exactly once, after its commit and before its request finishes — including the
  positions whose kv-only step never reached the oracle (sim.py:278 skips the
  oracle when the backlog fills the chunk, engine.py:58-59, yet apply_chunk marks
  them DECODED_CACHED);
* the schedule is the reference's: the records are byte-identical to a run with the
  inner oracle alone (per-request seam and the batched loop alike);
* pages are released when a request finishes.
"""

import dataclasses

import numpy as np
import pytest

sim = pytest.importorskip("dllmsim.sim")
from dllmsim.commit import CommitProfile, StochasticOracle  # noqa: E402
from dllmsim.core import records_to_csv  # noqa: E402
from dllmsim.scheduler import ElasticChunk, FixedChunk  # noqa: E402
from dllmsim.costmodel import default_cost_model  # noqa: E402
from dllmsim.sim import ClosedLoop, OpenLoop  # noqa: E402
from dllmsim.workload import PROFILES  # noqa: E402

from paper_2605_24832_b200.decode import B200Oracle  # noqa: E402
from paper_2605_24832_b200 import sim_bridge  # noqa: E402


class _Tables:
    def __init__(self):
        self.live = set()

    def slot(self, rid):
        return 0 if rid in self.live else None


class StubDecoder:
    """Stands in for StreamingDecoder: records every device plan and answers the
    window rows with an inner reference oracle (what ReferenceOracleForward's
    logits make K3 decide on the GPU)."""

    def __init__(self, inner, block):
        self.inner = inner
        self.cfg = type("Cfg", (), {"block_size": block})()
        self.tables = _Tables()
        self.forward = self
        self.steps = []      # [(request id, kv positions, window)]
        self.released = []
        self.committed_at = {}  # (rid, pos) -> device step index of its commit
        self.recomputed_at = {}  # (rid, pos) -> device step index of its kv recompute

    def prepare(self, reqs, plans):
        for r in reqs:
            self.tables.live.add(r.id)
        return (list(reqs), list(plans))

    def device_step(self, dm):
        return None

    def fetch_commits(self, dm, res):
        reqs, plans = dm
        k = len(self.steps)
        out = []
        for r, p in zip(reqs, plans):
            for pos in p.kv_positions:
                assert (r.id, pos) in self.committed_at, "recomputed before it was committed"
                assert (r.id, pos) not in self.recomputed_at, "recomputed twice"
                self.recomputed_at[(r.id, pos)] = k
            c = self.inner.commits(r, list(p.window)) if p.window else set()
            for pos in c:
                self.committed_at[(r.id, pos)] = k
            out.append(c)
        self.steps.append([(r.id, tuple(p.kv_positions), tuple(p.window)) for r, p in zip(reqs, plans)])
        return out

    def release(self, req):
        self.tables.live.discard(req.id)
        self.released.append(req.id)

    def consume(self, req, committed):
        fn = getattr(self.inner, "consume", None)
        if fn:
            fn(req, committed)


def _steep():
    """Flat to 64 computed tokens, then steep: a lone request runs chunk 32, a full
    batch chunk 2, so arrivals switch an elastic chunk 32 -> 2 (kv-only steps)."""
    from dllmsim.costmodel import CostModel, Segment

    return CostModel(segments=(Segment(0.0, 0.0, 1e-3), Segment(64.0, 1.25e-4, 1e-3),
                               Segment(128.0, 2.5e-4, 9e-3)))


def _scenario(policy, seed, n=14, profile=PROFILES["sharegpt"], q=0.75):
    mode = (ClosedLoop(concurrency=6, total_requests=n) if seed % 2
            else OpenLoop(arrival_rate=300.0, num_requests=n))
    cost = _steep() if seed % 2 == 0 else default_cost_model()
    return sim.Scenario(mode=mode, policy=policy, commit_profile=CommitProfile(q=q, rate_jitter_sigma=0.75),
                        cost_model=cost, dataset=profile, seed=seed)


POLICIES = [
    FixedChunk(chunk_size=8, block_size=32),
    FixedChunk(chunk_size=2, block_size=16),
    ElasticChunk(block_size=32, candidates=(2, 32), warmup_observations=0, hysteresis=0.0),
    ElasticChunk(block_size=16, candidates=tuple(range(2, 17, 2)), warmup_observations=2),
]


@pytest.mark.parametrize("batched", [False, True])
@pytest.mark.parametrize("k", range(len(POLICIES)))
def test_seam_keeps_reference_schedule_and_rule_k(k, batched):
    policy = POLICIES[k]
    sc = _scenario(policy, 10 + k)
    ref = sim.run(sc)
    holder = {}

    def factory():
        dec = StubDecoder(StochasticOracle(sc.commit_profile), policy.block_size)
        holder["dec"] = dec
        return B200Oracle(dec)

    got = (sim_bridge.run if batched else sim.run)(dataclasses.replace(sc, oracle_factory=factory))
    assert records_to_csv(got.records) == records_to_csv(ref.records)
    dec = holder["dec"]
    # rule K: every committed position is recomputed once, after its commit ...
    last = {}
    for (rid, pos), k_c in dec.committed_at.items():
        last[rid] = max(last.get(rid, -1), k_c)
    missing = []
    for (rid, pos), k_c in dec.committed_at.items():
        k_r = dec.recomputed_at.get((rid, pos))
        if k_r is None:
            missing.append((rid, pos, k_c))
        else:
            assert k_r > k_c
    # ... except the commits of a request's final step (it leaves the batch, sim.py:309-313)
    assert all(k_c == last[rid] for rid, _, k_c in missing)
    # every request finished and released its pages exactly once
    assert sorted(dec.released) == sorted(r.id for r in got.request_log)
    if batched:  # one device step per decode iteration (none for an all-kv-only batch)
        its = sum(1 for r in got.records if r.kind.name == "DECODE")
        assert len(dec.steps) <= its


def test_kv_only_steps_are_folded_into_the_next_device_step():
    """ElasticChunk switching 32 -> 2 leaves backlogs >= 2: those plans are kv-only,
    the reference never calls the oracle for them, and the next device step of the
    request recomputes them first."""
    policy = POLICIES[2]
    sc = _scenario(policy, 4, n=12, q=0.85)
    holder = {}

    def factory():
        dec = StubDecoder(StochasticOracle(sc.commit_profile), policy.block_size)
        holder["dec"] = dec
        return B200Oracle(dec)

    res = sim.run(dataclasses.replace(sc, oracle_factory=factory))
    chunks = {r.chunk_size for r in res.records if r.kind.name == "DECODE"}
    assert {2, 32} <= chunks
    dec = holder["dec"]
    # some device step carried more kv rows than the chunk allowed: folded backlog
    assert any(len(kv) + len(win) > 2 and len(win) >= 1 and len(kv) >= 2
               for step in dec.steps for _, kv, win in step)
