"""Commit-trace record / replay: the package's CommitTrace JSONL and
ReplayOracle against goldens recorded and replayed by the reference itself
(tests/golden/make_golden.py: commit.py:206-312 driven through engine.py:45-95)."""

import json

import numpy as np
import pytest

from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.core import Request
from paper_2605_24832_b200.errors import TraceExhausted
from paper_2605_24832_b200.trace import CommitTrace, ReplayOracle, TraceRecorder, replay_oracle


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.loads((golden_dir / "trace.json").read_text())


def test_jsonl_round_trip_is_byte_identical(golden):
    for case in golden["cases"]:
        t = CommitTrace.from_jsonl(case["jsonl"])
        assert t.to_jsonl() == case["jsonl"]
        t.validate({case["seed"] * 100 + i: out for i, out in enumerate(case["outs"])})
        # lines in any order load the same trace
        lines = case["jsonl"].strip().split("\n")
        assert CommitTrace.from_jsonl("\n".join(reversed(lines))).to_jsonl() == case["jsonl"]


def test_record_and_validate_errors():
    t = CommitTrace()
    t.record(1, 0, [0, 2])
    with pytest.raises(ValueError):
        t.record(1, 2, [1])  # out of order
    t.record(1, 1, [2])
    with pytest.raises(ValueError):
        t.validate({})  # position 2 twice
    t2 = CommitTrace()
    t2.record(3, 0, [0])
    with pytest.raises(ValueError):
        t2.validate({3: 2})  # does not cover position 1
    assert CommitTrace().to_jsonl() == "\n"


def test_replays_match_reference(golden):
    for case in golden["cases"]:
        for run in case["replays"]:
            ro = ReplayOracle(CommitTrace.from_jsonl(case["jsonl"]), carryover=run["carryover"])
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


def test_strict_replay_past_the_end_raises():
    t = CommitTrace()
    t.record(5, 0, [0, 1])
    assert replay_oracle(t, 5, 0, [1, 2]) == {1}
    with pytest.raises(TraceExhausted):
        replay_oracle(t, 5, 1, [2])
    with pytest.raises(TraceExhausted):
        replay_oracle(t, 6, 0, [0])


def test_recorder_skips_requests_that_did_not_step():
    class R:
        def __init__(self, i):
            self.id, self.steps_taken = i, 0

    class S:
        def __init__(self, c):
            self.commits = frozenset(c)

    a, b = R(1), R(2)
    rec = TraceRecorder()
    rec.before([a, b])
    a.steps_taken = 1  # b did not step
    rec.after([a, b], [S([0, 3]), S([])])
    assert rec.trace.steps == {1: [{0, 3}]}
