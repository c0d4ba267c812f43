"""Control half: oracle restatement and the package's host mirror vs golden
vectors produced by the reference itself (tests/golden/make_golden.py)."""

import json
from collections import deque

import numpy as np
import pytest

from oracle import control as oc
from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.core import Request, TokenState, WindowRule
from paper_2605_24832_b200.errors import ChunkTooSmall, IllegalCommit


@pytest.fixture(scope="module")
def control(golden_dir):
    return json.loads((golden_dir / "control.json").read_text())


@pytest.fixture(scope="module")
def commits_golden(golden_dir):
    return json.loads((golden_dir / "commits.json").read_text())


def _oracle_req(out, before):
    return {"out": out, "states": list(before["states"]), "queue": list(before["queue"]),
            "block": before["block"], "committed": before["committed"], "steps": 0}


def _pkg_req(out, before):
    r = Request(id=0, arrival_time=0.0, prompt_tokens=1, output_tokens=out)
    r.states[:] = np.asarray(before["states"], dtype=np.int8)
    r.uncached_queue = deque(before["queue"])
    r.block_index = before["block"]
    r.committed = before["committed"]
    return r


def test_oracle_replays_match_reference(control):
    n_steps = 0
    for case in control["replays"]:
        req = oc.new_request(case["out"])
        for st in case["steps"]:
            assert req["states"] == st["before"]["states"]
            assert req["queue"] == st["before"]["queue"]
            assert req["block"] == st["before"]["block"]
            kv, win = oc.plan_chunk(req, st["chunk"], case["block"], case["rule"])
            assert kv == st["kv"] and win == st["window"]
            oc.apply_chunk(req, kv, win, set(st["commits"]), case["block"])
            assert req["block"] == st["after_block"]
            n_steps += 1
        assert req["states"] == case["final_states"]
    assert n_steps > 1000


def test_package_plan_apply_match_reference(control):
    for case in control["replays"]:
        rule = WindowRule(case["rule"])
        for st in case["steps"]:
            r = _pkg_req(case["out"], st["before"])
            plan = pe.plan_chunk(r, st["chunk"], case["block"], rule)
            assert list(plan.kv_positions) == st["kv"]
            assert list(plan.window) == st["window"]
            [bplan] = pe.plan_batch([r], st["chunk"], case["block"], rule)
            assert bplan == plan
            summary = pe.apply_chunk(r, plan, set(st["commits"]), case["block"])
            assert summary.computed == len(st["kv"]) + len(st["window"])
            assert r.block_index == st["after_block"]


def test_reference_engine_cases(control):
    for c in control["engine_cases"]:
        req = oc.new_request(c["out"])
        req["states"] = list(c["states"])
        req["queue"] = list(c["queue"])
        req["block"] = c["block"]
        kv, win = oc.plan_chunk(req, c["chunk"], c["bs"], c["rule"])
        assert (kv, win) == (c["kv"], c["window"]), c["name"]
        r = _pkg_req(c["out"], {"states": c["states"], "queue": c["queue"], "block": c["block"], "committed": 0})
        plan = pe.plan_chunk(r, c["chunk"], c["bs"], c["rule"])
        assert (list(plan.kv_positions), list(plan.window)) == (c["kv"], c["window"]), c["name"]


def test_commit_step_draws_match_reference(commits_golden):
    for d in commits_golden["draws"]:
        rng = np.random.default_rng(d["seed"])
        n = len(d["window"])
        u = rng.random(n - 1) if n > 1 else []
        dec = oc.commit_step_decisions(d["q"], d["m"], n, u)
        got = sorted(p for p, c in zip(d["window"], dec) if c)
        assert got == d["commits"]


def test_calibration_goldens_pinned(commits_golden):
    # test_commit.py:54-57 of the reference
    assert commits_golden["q"]["calibrate_32_5.29"] == pytest.approx(0.8111977515578267, abs=1e-7)
    assert commits_golden["q"]["calibrate_32_2.51"] == pytest.approx(0.6015936600147661, abs=1e-7)


def test_engine_errors_mirror_reference():
    r = Request(id=0, arrival_time=0.0, prompt_tokens=1, output_tokens=8)
    with pytest.raises(ChunkTooSmall):
        pe.plan_chunk(r, 1, 8)
    plan = pe.plan_chunk(r, 4, 8)
    with pytest.raises(IllegalCommit):
        pe.apply_chunk(r, plan, {5}, 8)
    r2 = Request(id=0, arrival_time=0.0, prompt_tokens=1, output_tokens=8)
    r2.states[0] = TokenState.DECODED_CACHED
    with pytest.raises(IllegalCommit):
        pe.apply_chunk(r2, pe.ChunkPlan((), (0, 1)), {0}, 8)
    r3 = Request(id=0, arrival_time=0.0, prompt_tokens=1, output_tokens=8)
    r3.uncached_queue.append(0)
    with pytest.raises(IllegalCommit):
        pe.apply_chunk(r3, pe.ChunkPlan((1,), ()), set(), 8)


def test_apply_advances_block():
    r = Request(id=0, arrival_time=0.0, prompt_tokens=1, output_tokens=8)
    plan = pe.plan_chunk(r, 4, 4)
    pe.apply_chunk(r, plan, {0, 1, 2, 3}, 4)
    assert r.block_index == 1


def _baselines():
    from pathlib import Path
    return json.loads((Path(__file__).resolve().parent / "golden" / "control.json").read_text())["baselines"]


@pytest.mark.parametrize("k", range(12))
def test_baseline_steps_match_reference(k):
    """BD / prefix-cached / AR steps (reference engine.py:98-157): the
    oracle restatement and the product host mirror (plan_block / apply_block)
    reproduce dllmsim's traces step for step given its commits."""
    case = _baselines()[k]
    mode, block, out = case["mode"], case["block"], case["out"]
    oreq = oc.new_request(out)
    req = Request(id=case["seed"], arrival_time=0.0, prompt_tokens=5, output_tokens=out)
    for st in case["steps"]:
        commits = set(st["commits"])
        if mode == "ar":
            comp_o = oc.ar_step(oreq)
        else:
            assert oc.block_step_window(oreq, block) == st["window"]
            comp_o = (oc.block_diffusion_step if mode == "bd" else oc.prefix_cached_step)(oreq, commits, block)
        assert comp_o == st["computed"] and oreq["states"] == st["states"]
        assert (oreq["block"], oreq["committed"]) == (st["block"], st["committed"])
        plan = pe.plan_block(req, block, mode)
        assert list(plan.window) == st["window"]
        summ = pe.apply_block(req, plan, commits if mode != "ar" else None, block, mode)
        assert summ.computed == st["computed"] and sorted(summ.commits) == st["commits"]
        assert req.states.tolist() == st["states"]
        assert (req.block_index, req.committed) == (st["block"], st["committed"])
    assert req.finished


def test_baseline_bd_plan_recomputes_the_whole_block():
    req = Request(id=0, arrival_time=0.0, prompt_tokens=3, output_tokens=20)
    req.states[[1, 4]] = TokenState.DECODED_UNCACHED
    plan = pe.plan_block(req, 8, "bd")
    assert plan.kv_positions == (1, 4) and plan.window == (0, 2, 3, 5, 6, 7)
    assert plan.computed == 8
    pplan = pe.plan_block(req, 8, "prefix")
    assert pplan.kv_positions == (1, 4)
    from paper_2605_24832_b200.errors import EmptyWindow
    req.states[:8] = TokenState.DECODED_CACHED
    req.block_index = 0
    with pytest.raises(EmptyWindow):
        pe.plan_block(req, 8, "bd")
