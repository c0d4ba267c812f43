"""End-to-end parity of the B200 decode step with the reference schedule.

The device step (K1 append, K2 attention, K3 unmask over logits that encode the
reference's commit_step draws) must reproduce, step for step, the request states
that the reference control loop produces with StochasticOracle on the same rng
streams (sim.py:269-305 streaming branch; engine.py:45-95; commit.py:86-112).
The host reference here is the oracle restatement pinned to dllmsim by
tests/golden.
"""

import copy

import numpy as np
import pytest
import torch

from oracle import control as oc
from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.core import Request
from paper_2605_24832_b200.decode import B200Oracle, DecodeConfig, StreamingDecoder, run_decode_batched
from paper_2605_24832_b200.synthetic import OracleDrivenForward

pytestmark = pytest.mark.gpu

Q = 0.7758267092770552  # calibrated sharegpt/dense-8b q


def _requests(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        r = Request(id=i, arrival_time=0.0, prompt_tokens=int(rng.integers(3, 90)),
                    output_tokens=int(rng.integers(20, 75)),
                    rng=np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1, i))))
        r.rate_multiplier = float(rng.choice([1.0, 0.6, 1.7]))
        out.append(r)
    return out


def _reference_step(batch, chunk, block, rule):
    """sim.py:276-291 with StochasticOracle: plan -> commit_step -> apply."""
    for req in batch:
        plan = pe.plan_chunk(req, chunk, block, rule)
        commits = set()
        if plan.window:
            n = len(plan.window)
            u = req.rng.random(n - 1) if n > 1 else []
            dec = oc.commit_step_decisions(Q, req.rate_multiplier, n, u)
            commits = {p for p, d in zip(plan.window, dec) if d}
        pe.apply_chunk(req, plan, commits, block)


def _cfg(block, page, rule):
    return DecodeConfig(num_layers=2, num_q_heads=8, num_kv_heads=2, head_dim=64, vocab=2048,
                        block_size=block, page_size=page, window_rule=rule, max_batch=8,
                        max_pages_per_req=64, num_pages=512)


@pytest.mark.parametrize("rule,chunk", [("in_block", 8), ("in_block", 16), ("out_block", 8)])
def test_batched_decode_reproduces_reference_schedule(rule, chunk):
    block, page = 16, 16
    ref = _requests(5, 6)
    dev = _requests(5, 6)
    cfg = _cfg(block, page, rule)
    dec = StreamingDecoder(cfg, OracleDrivenForward(cfg, 8 * chunk, Q, seed=1))
    steps = 0
    while not all(r.finished for r in ref):
        active_ref = [r for r in ref if not r.finished]
        active_dev = [r for r in dev if not r.finished]
        _reference_step(active_ref, chunk, block, rule)
        computed, committed, _ = run_decode_batched(dec, active_dev, chunk)
        for a, b in zip(ref, dev):
            assert np.array_equal(a.states, b.states), (steps, a.id)
            assert list(a.uncached_queue) == list(b.uncached_queue)
            assert (a.block_index, a.committed, a.steps_taken) == (b.block_index, b.committed, b.steps_taken)
        steps += 1
        assert steps < 400
    assert all(r.finished for r in dev)


def test_oracle_protocol_per_request_calls():
    """B200Oracle behind the reference's per-request protocol (sim.py:278-280)."""
    block, page, chunk, rule = 16, 16, 8, "in_block"
    ref = _requests(9, 4)
    dev = _requests(9, 4)
    cfg = _cfg(block, page, rule)
    decoder = StreamingDecoder(cfg, OracleDrivenForward(cfg, 8 * chunk, Q, seed=2))
    oracle = B200Oracle(decoder)
    for _ in range(6):
        _reference_step([r for r in ref if not r.finished], chunk, block, rule)
        for req in [r for r in dev if not r.finished]:
            plan = pe.plan_chunk(req, chunk, block, rule)
            commits = oracle.commits(req, plan.window) if plan.window else set()
            oracle.consume(req, commits)
            pe.apply_chunk(req, plan, commits, block)
        for a, b in zip(ref, dev):
            assert np.array_equal(a.states, b.states)


def _reference_baseline_step(batch, block, mode):
    """sim.py:253-267 with StochasticOracle: the reference's block / AR steps."""
    for req in batch:
        if mode == "ar":
            pe.ar_step(req)
            continue
        plan = pe.plan_block(req, block, mode)
        n = len(plan.window)
        u = req.rng.random(n - 1) if n > 1 else []
        dec = oc.commit_step_decisions(Q, req.rate_multiplier, n, u)
        commits = {p for p, d in zip(plan.window, dec) if d}
        pe.apply_block(req, plan, commits, block, mode)


@pytest.mark.parametrize("mode", ["bd", "prefix", "ar"])
def test_baseline_modes_reproduce_reference_schedule(mode):
    """BD / prefix-cached / AR on the B200 kernels: the device step's
    commits reproduce the reference baseline schedule step for step."""
    block, page = 16, 16
    ref = _requests(13, 5)
    dev = _requests(13, 5)
    cfg = _cfg(block, page, "in_block")
    dec = StreamingDecoder(cfg, OracleDrivenForward(cfg, 8 * block, Q, seed=3))
    steps = 0
    while not all(r.finished for r in ref):
        _reference_baseline_step([r for r in ref if not r.finished], block, mode)
        summ = dec.step_baseline([r for r in dev if not r.finished], mode)
        assert all(s.computed >= 1 for s in summ)
        for a, b in zip(ref, dev):
            assert np.array_equal(a.states, b.states), (mode, steps, a.id)
            assert (a.block_index, a.committed, a.steps_taken) == (b.block_index, b.committed, b.steps_taken)
        steps += 1
        assert steps < 500
    assert all(r.finished for r in dev)


def test_bd_oracle_inside_reference_block_step():
    """B200Oracle(mode="bd") behind the reference-signature block_diffusion_step."""
    block, page = 16, 16
    ref = _requests(17, 3)
    dev = _requests(17, 3)
    cfg = _cfg(block, page, "in_block")
    oracle = B200Oracle(StreamingDecoder(cfg, OracleDrivenForward(cfg, 8 * block, Q, seed=4)), mode="bd")
    for _ in range(5):
        _reference_baseline_step([r for r in ref if not r.finished], block, "bd")
        for req in [r for r in dev if not r.finished]:
            pe.block_diffusion_step(req, oracle, block)
        for a, b in zip(ref, dev):
            assert np.array_equal(a.states, b.states)
