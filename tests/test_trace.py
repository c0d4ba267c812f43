"""Commit-trace record / replay.  The trace and the replaying oracle
are the reference's own classes (dllmsim.commit, commit.py:205-312); what is tested
here is this package's side of it: the engine mirror replays the reference's
recorded traces step for step (goldens from tests/golden/make_golden.py), and
TraceRecorder produces a trace the reference loads and validates."""

import json

import pytest

from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.core import Request
from paper_2605_24832_b200.errors import TraceExhausted
from paper_2605_24832_b200.trace import TraceRecorder

commit = pytest.importorskip("dllmsim.commit")


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.loads((golden_dir / "trace.json").read_text())


def test_engine_mirror_replays_reference_traces(golden):
    """dllmsim's ReplayOracle driving this package's plan_chunk / apply_chunk
    reproduces the windows, commits and final states the reference recorded."""
    for case in golden["cases"]:
        for run in case["replays"]:
            ro = commit.ReplayOracle(commit.CommitTrace.from_jsonl(case["jsonl"]), carryover=run["carryover"])
            for i, (out, want) in enumerate(zip(case["outs"], run["requests"])):
                req = Request(id=case["seed"] * 100 + i, arrival_time=0.0, prompt_tokens=5, output_tokens=out)
                steps = []
                exhausted = False
                while not req.finished and len(steps) < 10 * out + 50:
                    plan = pe.plan_chunk(req, run["chunk"], case["block"], "in_block")
                    try:
                        commits = ro.commits(req, list(plan.window)) if plan.window else set()
                    except TraceExhausted:
                        exhausted = True
                        break
                    pe.apply_chunk(req, plan, commits, case["block"])
                    ro.consume(req, commits)
                    steps.append({"window": list(plan.window), "commits": sorted(commits)})
                assert steps == want["steps"], (case["seed"], run["chunk"], run["carryover"], i)
                assert exhausted == want["exhausted"] and req.finished == want["finished"]
                assert req.states.tolist() == want["final_states"]


def test_recorder_skips_requests_that_did_not_step():
    class R:
        def __init__(self, i):
            self.id, self.steps_taken = i, 0

    class S:
        def __init__(self, c):
            self.commits = frozenset(c)

    a, b = R(1), R(2)
    rec = TraceRecorder()
    assert isinstance(rec.trace, commit.CommitTrace)
    rec.before([a, b])
    a.steps_taken = 1  # b did not step
    rec.after([a, b], [S([0, 3]), S([])])
    assert rec.trace.steps == {1: [{0, 3}]}


def test_recorded_decode_round_trips_through_reference_jsonl():
    """Record a batched decode (engine mirror + the reference's stochastic oracle),
    serialise with the reference's JSONL, validate coverage, replay strictly."""
    prof = commit.CommitProfile(q=0.8)
    oracle = commit.StochasticOracle(prof)
    import numpy as np

    reqs = [Request(id=i, arrival_time=0.0, prompt_tokens=7, output_tokens=40 + 9 * i,
                    rng=np.random.default_rng(i)) for i in range(4)]
    rec = TraceRecorder()
    while not all(r.finished for r in reqs):
        live = [r for r in reqs if not r.finished]
        plans = pe.plan_batch(live, 8, 32, "in_block")
        cs = [oracle.commits(r, list(p.window)) if p.window else set() for r, p in zip(live, plans)]
        rec.before(live)
        sums = pe.apply_batch(live, plans, cs, 32)
        rec.after(live, sums)
    text = rec.trace.to_jsonl()
    tr = commit.CommitTrace.from_jsonl(text)
    tr.validate({r.id: r.output_tokens for r in reqs})
    assert tr.to_jsonl() == text
