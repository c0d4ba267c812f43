"""Generate golden vectors by running the reference package ``dllmsim`` itself.

Run in the build container (the reference is not available on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes (small, committed):
  control.json  step-by-step replays of plan_chunk / apply_chunk under the
                StochasticOracle (engine.py:45-95, commit.py:86-112) plus the
                hand-written cases of the reference's test_engine.py:50-157.
  commits.json  commit_step decisions for seeded windows (commit.py:86-112) and
                calibrate_q goldens (test_commit.py:54-57).
  trace.json    CommitTrace JSONL recorded from stochastic decodes
                (commit.py:206-251) and ReplayOracle replays of it, strict and
                carry-over, under other chunk sizes (commit.py:254-312).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from dllmsim.commit import (CommitProfile, CommitTrace, ReplayOracle, StochasticOracle,  # noqa: E402
                            TraceExhausted, calibrate_q, commit_step)
from dllmsim.core import Request, TokenState, WindowRule  # noqa: E402
from dllmsim.engine import apply_chunk, ar_step, block_diffusion_step, plan_chunk, prefix_cached_step  # noqa: E402
from dllmsim.workload import PROFILES, calibrated_profile  # noqa: E402

OUT = Path(__file__).resolve().parent


def replay_case(seed: int, out_tokens: int, chunk: int, block: int, rule: str, q: float, m: float,
                chunk_schedule=None) -> dict:
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1, seed)))
    req = Request(id=seed, arrival_time=0.0, prompt_tokens=7, output_tokens=out_tokens, rng=rng)
    req.rate_multiplier = m
    oracle = StochasticOracle(CommitProfile(q=q))
    wr = WindowRule.IN_BLOCK if rule == "in_block" else WindowRule.OUT_BLOCK
    steps = []
    guard = 0
    while not req.finished and guard < 10 * out_tokens + 50:
        c = chunk if chunk_schedule is None else chunk_schedule[guard % len(chunk_schedule)]
        plan = plan_chunk(req, c, block, wr)
        before = {
            "states": req.states.tolist(),
            "queue": list(req.uncached_queue),
            "block": req.block_index,
            "committed": req.committed,
        }
        commits = oracle.commits(req, plan.window) if plan.window else set()
        apply_chunk(req, plan, commits, block)
        steps.append({
            "chunk": c,
            "before": before,
            "kv": list(plan.kv_positions),
            "window": list(plan.window),
            "commits": sorted(commits),
            "after_block": req.block_index,
        })
        guard += 1
    return {
        "seed": seed, "out": out_tokens, "chunk": chunk, "block": block, "rule": rule,
        "q": q, "m": m, "schedule": chunk_schedule, "steps": steps,
        "final_states": req.states.tolist(), "final_queue": list(req.uncached_queue),
    }


def baseline_case(seed: int, out_tokens: int, block: int, mode: str, q: float, m: float) -> dict:
    """A whole request under one of the reference's baseline steps
    (engine.py:98-157) with StochasticOracle: per step the window (masked positions
    of the block), the commits, the computed count and the state after."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1, seed)))
    req = Request(id=seed, arrival_time=0.0, prompt_tokens=5, output_tokens=out_tokens, rng=rng)
    req.rate_multiplier = m
    oracle = StochasticOracle(CommitProfile(q=q))
    steps = []
    while not req.finished:
        lo, hi = req.block_span(block if mode != "ar" else 1)
        window = [int(p) for p in range(lo, hi) if req.states[p] == TokenState.MASKED]
        if mode == "bd":
            s = block_diffusion_step(req, oracle, block)
        elif mode == "prefix":
            s = prefix_cached_step(req, oracle, block)
        else:
            s = ar_step(req)
        steps.append({"window": window, "commits": sorted(int(p) for p in s.commits), "computed": int(s.computed),
                      "states": [int(x) for x in req.states], "block": int(req.block_index),
                      "committed": int(req.committed)})
    return {"seed": seed, "out": out_tokens, "block": block, "mode": mode, "steps": steps}


def engine_cases() -> list:
    """The reference's hand-written plan/apply cases (test_engine.py:50-157)."""
    cases = []

    def mk(n):
        return Request(id=0, arrival_time=0.0, prompt_tokens=1, output_tokens=n,
                       rng=np.random.default_rng(0))

    r = mk(8)
    p = plan_chunk(r, 4, 8)
    cases.append({"name": "fresh", "out": 8, "states": r.states.tolist(), "queue": [], "block": 0,
                  "chunk": 4, "bs": 8, "rule": "in_block", "kv": list(p.kv_positions), "window": list(p.window)})
    r = mk(8)
    r.states[0] = r.states[1] = TokenState.DECODED_UNCACHED
    r.uncached_queue.extend([0, 1])
    p = plan_chunk(r, 4, 8)
    cases.append({"name": "backlog_first", "out": 8, "states": r.states.tolist(), "queue": [0, 1], "block": 0,
                  "chunk": 4, "bs": 8, "rule": "in_block", "kv": list(p.kv_positions), "window": list(p.window)})
    r = mk(40)
    r.states[0:7] = TokenState.DECODED_CACHED
    r.committed = 7
    r.advance_blocks(8)
    for rule, wr in (("out_block", WindowRule.OUT_BLOCK), ("in_block", WindowRule.IN_BLOCK)):
        p = plan_chunk(r, 6, 8, wr)
        cases.append({"name": f"cross_{rule}", "out": 40, "states": r.states.tolist(), "queue": [],
                      "block": r.block_index, "chunk": 6, "bs": 8, "rule": rule,
                      "kv": list(p.kv_positions), "window": list(p.window)})
    return cases


def trace_case(seed: int, outs, rec_chunk: int, replays, block: int = 32) -> dict:
    """Record a CommitTrace from stochastic decodes of len(outs) requests, then
    replay it through plan_chunk / apply_chunk with ReplayOracle."""
    trace = CommitTrace()
    oracle = StochasticOracle(CommitProfile(q=0.8))
    for i, out in enumerate(outs):
        rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1, i)))
        req = Request(id=seed * 100 + i, arrival_time=0.0, prompt_tokens=5, output_tokens=out, rng=rng)
        step = 0
        while not req.finished:
            plan = plan_chunk(req, rec_chunk, block, WindowRule.IN_BLOCK)
            commits = oracle.commits(req, plan.window) if plan.window else set()
            apply_chunk(req, plan, commits, block)
            trace.record(req.id, step, commits)
            step += 1
    trace.validate({seed * 100 + i: out for i, out in enumerate(outs)})
    jsonl = trace.to_jsonl()
    runs = []
    for chunk, carry in replays:
        ro = ReplayOracle(CommitTrace.from_jsonl(jsonl), carryover=carry)
        per_req = []
        for i, out in enumerate(outs):
            req = Request(id=seed * 100 + i, arrival_time=0.0, prompt_tokens=5, output_tokens=out,
                          rng=np.random.default_rng(0))
            steps = []
            exhausted = False
            while not req.finished and len(steps) < 10 * out + 50:
                plan = plan_chunk(req, chunk, block, WindowRule.IN_BLOCK)
                try:
                    commits = ro.commits(req, plan.window) if plan.window else set()
                except TraceExhausted:
                    exhausted = True
                    break
                apply_chunk(req, plan, commits, block)
                ro.consume(req, commits)
                steps.append({"window": list(plan.window), "commits": sorted(commits)})
            per_req.append({"steps": steps, "final_states": req.states.tolist(), "exhausted": exhausted,
                            "finished": bool(req.finished)})
        runs.append({"chunk": chunk, "carryover": carry, "requests": per_req})
    return {"seed": seed, "outs": list(outs), "rec_chunk": rec_chunk, "block": block, "jsonl": jsonl,
            "replays": runs}


def main() -> None:
    sharegpt = calibrated_profile(PROFILES["sharegpt"], "dense-8b")
    cases = []
    k = 0
    for rule in ("in_block", "out_block"):
        for chunk in (2, 4, 8, 16, 32):
            for out_tokens in (5, 33, 70, 97):
                cases.append(replay_case(1000 + k, out_tokens, chunk, 32, rule, sharegpt.q, 1.0))
                k += 1
    # alternating chunk sizes (the elastic scheduler switches chunk every step)
    for sched in ([32, 2], [2, 8, 16], [6, 32, 4]):
        cases.append(replay_case(2000 + k, 90, 0, 32, "in_block", sharegpt.q, 1.3, sched))
        k += 1
    # small blocks
    for bs in (4, 8):
        cases.append(replay_case(3000 + k, 41, 6, bs, "in_block", 0.7, 0.8))
        k += 1
    baselines = []
    for mode in ("bd", "prefix", "ar"):
        for j, (out_tokens, block) in enumerate(((40, 32), (97, 32), (33, 8), (64, 16))):
            baselines.append(baseline_case(4000 + 10 * j + len(baselines), out_tokens, block, mode, sharegpt.q, 1.0))
    (OUT / "control.json").write_text(json.dumps({"replays": cases, "engine_cases": engine_cases(),
                                                  "baselines": baselines}))

    draws = []
    for seed in range(40):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(1, 33))
        q = float(rng.uniform(0.3, 0.95))
        m = float(rng.uniform(0.5, 2.0))
        start = int(rng.integers(0, 50))
        window = list(range(start, start + n))
        rr = np.random.default_rng(10_000 + seed)
        commits = commit_step(CommitProfile(q=q), m, window, rr)
        draws.append({"seed": 10_000 + seed, "q": q, "m": m, "window": window, "commits": sorted(commits)})
    golden_q = {
        "calibrate_32_5.29": calibrate_q(32, 5.29),
        "calibrate_32_2.51": calibrate_q(32, 2.51),
        "sharegpt_dense8b_q": sharegpt.q,
        "sharegpt_dense8b_sigma": sharegpt.rate_jitter_sigma,
    }
    (OUT / "commits.json").write_text(json.dumps({"draws": draws, "q": golden_q}))
    traces = [trace_case(7, (40, 70, 33), 32, ((32, False), (32, True), (8, True), (4, True), (8, False))),
              trace_case(8, (97, 12), 16, ((16, False), (6, True), (32, True)))]
    (OUT / "trace.json").write_text(json.dumps({"cases": traces}))
    print("wrote", OUT / "control.json", OUT / "commits.json", OUT / "trace.json",
          len(cases), "replays")


if __name__ == "__main__":
    main()
