"""The B200 oracle inside dllmsim's own simulation loop, on the GPU.

``Scenario.oracle_factory`` (sim.py:64,128-132) builds a ``B200Oracle`` whose
device step (K1 append, K2 paged attention, K3 unmask) decides every commit: the
window rows' logits encode a reference oracle's decisions
(``ReferenceOracleForward``), and the K3 threshold must turn them back into the
same sets.  Checked here against the reference's own acceptance criteria:

* #10 (test_acceptance.py:494-522): the hand-derived toy schedules, exactly
  (34 s / 18 s / 10 s, first token 3 s / 4 s / 3 s, elastic chunk 8 throughout);
* #9 (test_acceptance.py:427-455), a slice of randomized scenarios: token
  conservation, monotone clocks, and records byte-identical to the run with the
  reference oracle alone (per-request seam, and ``sim_bridge.BatchedLoop``);
* rule K under elastic 32 <-> 2 switching: after every device step, each
  position's KV in the pages equals a fresh recompute of its committed-token KV —
  including positions whose kv-only step never reached the oracle (sim.py:278).
"""

import dataclasses

import numpy as np
import pytest
import torch

sim = pytest.importorskip("dllmsim.sim")
from dllmsim.commit import CommitProfile, CommitTrace, ReplayOracle, StochasticOracle  # noqa: E402
from dllmsim.core import IterationKind, records_to_csv  # noqa: E402
from dllmsim.costmodel import CostModel, Segment, default_cost_model  # noqa: E402
from dllmsim.scheduler import (AutoregressivePolicy, BlockLevelBatch, ElasticChunk, FixedBlock,  # noqa: E402
                               FixedChunk)
from dllmsim.sim import ClosedLoop, OpenLoop, Scenario  # noqa: E402
from dllmsim.workload import PROFILES, DatasetProfile, TraceEntry  # noqa: E402

from paper_2605_24832_b200 import sim_bridge  # noqa: E402
from paper_2605_24832_b200.decode import B200Oracle, DecodeConfig, StreamingDecoder  # noqa: E402
from paper_2605_24832_b200.synthetic import ReferenceOracleForward  # noqa: E402

pytestmark = pytest.mark.gpu


def _cfg(block, page=64, max_pages=320, num_pages=8192, layers=1, max_batch=32):
    return DecodeConfig(num_layers=layers, num_q_heads=8, num_kv_heads=2, head_dim=128, vocab=4096,
                        block_size=block, page_size=page, fallback="none", max_batch=max_batch,
                        max_pages_per_req=max_pages, num_pages=num_pages)


def _b200_factory(inner_factory, block, policy, holder=None, oracle_cls=B200Oracle, **kw):
    mode = "bd" if isinstance(policy, (FixedBlock, BlockLevelBatch)) else "stream"

    def factory():
        cfg = _cfg(block, **kw)
        fwd = ReferenceOracleForward(cfg, inner_factory(), max_tokens=64 * 32)
        oracle = oracle_cls(StreamingDecoder(cfg, fwd), mode=mode)
        if holder is not None:
            holder["oracle"] = oracle
        return oracle
    return factory


# --------------------------------------------------------------------------- #10
def _toy_cost_model():  # flat 1 s through 16 tokens, 2 s at 32 (acceptance #10's toy)
    return CostModel(segments=(Segment(0.0, 0.0, 1.0), Segment(16.0, 1.0 / 16.0, 1.0),
                               Segment(32.0, 1.0 / 8.0, 2.0)))


def _four_per_step():
    t = CommitTrace()
    for rid in (0, 1):
        for step in range(8):
            t.record(rid, step, {4 * step + i for i in range(4)})
    return t


def _toy(policy, b200: bool):
    inner = lambda: ReplayOracle(_four_per_step(), carryover=True)
    return Scenario(
        mode=OpenLoop(arrival_rate=1.0, num_requests=2), policy=policy, commit_profile=CommitProfile(q=0.75),
        cost_model=_toy_cost_model(), dataset=DatasetProfile("toy", 8, 0, 32, 0, {"custom": (4.0, 0.0)}),
        requests=(TraceEntry(0, 0.0, 8, 32), TraceEntry(1, 0.0, 8, 32)),
        oracle_factory=_b200_factory(inner, 16, policy, max_pages=8, num_pages=64) if b200 else inner,
        seed=0)


@pytest.mark.parametrize("runner", ["sim", "batched"])
def test_acceptance_10_toy_schedules_with_b200_oracle(runner):
    run = sim.run if runner == "sim" else sim_bridge.run
    ar = run(_toy(AutoregressivePolicy(), True))
    assert [r.finish_time for r in ar.request_log] == [34.0, 34.0]
    assert [r.first_token_time for r in ar.request_log] == [3.0, 3.0]
    block = run(_toy(FixedBlock(block_size=16), True))
    assert [r.finish_time for r in block.request_log] == [18.0, 18.0]
    assert [r.first_token_time for r in block.request_log] == [4.0, 4.0]
    elastic_policy = ElasticChunk(block_size=16, candidates=(2, 4, 6, 8, 10, 12, 14, 16), warmup_observations=0,
                                  alpha=0.5, min_observations=8)
    elastic = run(_toy(elastic_policy, True))
    assert [r.finish_time for r in elastic.request_log] == [10.0, 10.0]
    assert [r.first_token_time for r in elastic.request_log] == [3.0, 3.0]
    decode = [r for r in elastic.records if r.kind is IterationKind.DECODE]
    assert all(r.chunk_size == 8 for r in decode)
    # and identical to the reference oracle's own run
    assert records_to_csv(elastic.records) == records_to_csv(sim.run(_toy(elastic_policy, False)).records)


# --------------------------------------------------------------------------- #9
def _random_scenario(rng, idx):
    """Randomized scenario in the shape of acceptance #9's generator (policies AR /
    FixedBlock / BlockLevelBatch / FixedChunk / ElasticChunk, random profiles,
    open and closed loops)."""
    ds = PROFILES[list(PROFILES)[rng.integers(len(PROFILES))]]
    block = int(rng.choice([8, 16, 32]))
    kind = int(rng.integers(5))
    policy = [lambda: AutoregressivePolicy(), lambda: FixedBlock(block_size=block),
              lambda: BlockLevelBatch(block_size=block),
              lambda: FixedChunk(chunk_size=int(rng.choice([2, 4, block])), block_size=block),
              lambda: ElasticChunk(block_size=block, candidates=tuple(range(2, block + 1, 2)),
                                   warmup_observations=int(rng.integers(0, 9)))][kind]()
    profile = CommitProfile(q=float(rng.uniform(0.0, 0.9)), rate_jitter_sigma=float(rng.choice([0.0, 0.75])))
    n = int(rng.integers(8, 17))
    mode = (OpenLoop(arrival_rate=float(rng.uniform(0.5, 12.0)), num_requests=n) if rng.random() < 0.5
            else ClosedLoop(concurrency=int(rng.integers(1, 9)), total_requests=n))
    return Scenario(mode=mode, policy=policy, commit_profile=profile, cost_model=default_cost_model(),
                    dataset=ds, seed=idx), block


@pytest.mark.parametrize("idx", [1, 2, 3, 5, 7, 8, 12, 14])
def test_acceptance_9_slice_with_b200_oracle(idx):
    rng = np.random.default_rng(7000 + idx)
    sc, block = _random_scenario(rng, idx)
    ref = sim.run(sc)
    inner = lambda: StochasticOracle(sc.commit_profile)
    runners = [sim.run] + ([sim_bridge.run] if isinstance(sc.policy, (FixedChunk, ElasticChunk)) else [])
    for run in runners:
        got = run(dataclasses.replace(sc, oracle_factory=_b200_factory(inner, block, sc.policy)))
        assert records_to_csv(got.records) == records_to_csv(ref.records), run
        n = sc.mode.num_requests if isinstance(sc.mode, OpenLoop) else sc.mode.total_requests
        assert len(got.request_log) == n
        dec = [r for r in got.records if r.kind is IterationKind.DECODE]
        assert sum(r.committed_tokens for r in dec) == sum(r.output_tokens for r in got.request_log)
        for req in got.request_log:
            assert req.finished and req.committed == req.output_tokens and not (req.states == 0).any()
            assert req.arrival_time <= req.prefill_done_time <= req.first_token_time <= req.finish_time
        for a, b in zip(got.records, got.records[1:]):
            assert b.clock_start >= a.clock_start + a.latency - 1e-9


# --------------------------------------------------------------------------- rule K
class PositionalForward(ReferenceOracleForward):
    """K/V of a query row are a fixed function of (request, position, whether the
    row is a window row with the MASK input or a kv row with its committed token),
    so the final KV of every position is known: what a fresh recompute writes."""

    def __init__(self, cfg, inner, **kw):
        super().__init__(cfg, inner, max_tokens=2048, **kw)
        self.resident_layers = False  # qkv() per layer, from the step's metadata

    @staticmethod
    def kv_value(rid, pos, window: bool, layer, cfg, device):
        rid = torch.as_tensor(rid, device=device, dtype=torch.float32).reshape(-1, 1, 1)
        pos = torch.as_tensor(pos, device=device, dtype=torch.float32).reshape(-1, 1, 1)
        win = torch.as_tensor(window, device=device, dtype=torch.float32).reshape(-1, 1, 1)
        h = torch.arange(cfg.num_kv_heads, device=device, dtype=torch.float32).reshape(1, -1, 1)
        d = torch.arange(cfg.head_dim, device=device, dtype=torch.float32).reshape(1, 1, -1)
        x = 0.37 * rid + 0.011 * pos + 0.5 * layer + 0.13 * h + 0.07 * d + 1.7 * win
        return torch.sin(x).to(torch.bfloat16), torch.cos(x).to(torch.bfloat16)

    def qkv(self, layer, dm):
        m = dm.host
        n = max(m.n_tok, 1)
        ids = np.asarray([r.id for r in dm.__dict__["requests"]], dtype=np.int64)
        rid = ids[m.tok_req] if m.n_tok else np.zeros(1)
        pos = np.asarray(m.tok_pos[: m.n_tok] if m.n_tok else [0])
        win = np.zeros(n, dtype=bool)
        win[np.asarray(m.row_tok[: m.n_rows], dtype=np.int64)] = True
        k, v = self.kv_value(rid, pos, win, layer, self.cfg, self.device)
        q = self.qkv_buf[layer][:n, : self.cfg.num_q_heads]
        return q, k, v


class CheckingOracle(B200Oracle):
    """After every device step: each request's DECODED_CACHED positions and the
    step's kv rows hold their final KV in the pages (all layers, all KV heads)."""

    checks = 0
    folded = 0

    def commits_batch(self, requests, plans):
        before = {r.id: list(self.recomputed.get(r.id, [])) for r in requests}
        queue = {r.id: list(r.uncached_queue) for r in requests}
        res = super().commits_batch(requests, plans)
        torch.cuda.synchronize()
        dec = self.decoder
        cfg = dec.cfg
        for req, plan in zip(requests, plans):
            s = dec.tables.slot(req.id)
            if s is None:  # finished: released
                continue
            now = self.recomputed[req.id][len(before[req.id]):]
            CheckingOracle.folded += len(now) - len(plan.kv_positions)
            assert list(now[len(now) - len(plan.kv_positions):]) == list(plan.kv_positions)
            assert set(now) >= set(queue[req.id][: len(plan.kv_positions)])
            pos = sorted(set(np.flatnonzero(req.states == 2).tolist()) | set(now))
            if not pos:
                continue
            a = req.prompt_tokens + np.asarray(pos)
            pages = torch.as_tensor(dec.tables.table[s][a // cfg.page_size], device=dec.device, dtype=torch.long)
            rows = torch.as_tensor(a % cfg.page_size, device=dec.device, dtype=torch.long)
            for layer in range(cfg.num_layers):
                kc, vc = dec.cache.layer(layer)
                k_want, v_want = PositionalForward.kv_value(req.id, pos, False, layer, cfg, dec.device)
                assert torch.equal(kc[pages, :, rows, :], k_want), (req.id, layer)
                assert torch.equal(vc[pages, :, rows, :].to(torch.bfloat16), v_want), (req.id, layer)
            CheckingOracle.checks += 1
        return res


def _elastic_scenario():
    steep = CostModel(segments=(Segment(0.0, 0.0, 1e-3), Segment(64.0, 1.25e-4, 1e-3),
                                Segment(128.0, 2.5e-4, 9e-3)))
    policy = ElasticChunk(block_size=32, candidates=(2, 32), warmup_observations=0, hysteresis=0.0)
    return Scenario(mode=OpenLoop(arrival_rate=300.0, num_requests=10), policy=policy,
                    commit_profile=CommitProfile(q=0.85, rate_jitter_sigma=0.75), cost_model=steep,
                    dataset=PROFILES["sharegpt"], seed=4), policy


def _positional_factory(sc, policy, holder, layers=2):
    def factory():
        cfg = _cfg(32, layers=layers)
        fwd = PositionalForward(cfg, StochasticOracle(sc.commit_profile))
        oracle = CheckingOracle(StreamingDecoder(cfg, fwd))
        holder["oracle"] = oracle
        return oracle
    return factory


@pytest.mark.parametrize("runner", ["sim", "batched"])
def test_elastic_32_2_pages_hold_fresh_recompute(runner):
    sc, policy = _elastic_scenario()
    holder = {}
    CheckingOracle.checks = CheckingOracle.folded = 0
    run = sim.run if runner == "sim" else sim_bridge.run
    got = run(dataclasses.replace(sc, oracle_factory=_positional_factory(sc, policy, holder)))
    assert records_to_csv(got.records) == records_to_csv(sim.run(sc).records)
    chunks = {r.chunk_size for r in got.records if r.kind is IterationKind.DECODE}
    assert {2, 32} <= chunks
    assert CheckingOracle.checks > 50
    if runner == "sim":  # kv-only steps skipped the oracle and were folded in later
        assert CheckingOracle.folded > 0


def test_without_folding_the_check_catches_stale_kv(monkeypatch):
    """Negative control: an oracle that recomputes only the plan's kv positions
    (the round-1 behaviour) leaves stale MASK-input KV behind kv-only steps."""
    def plan_kv_only(self, req, plan):
        self._track(req)
        kv = tuple(int(p) for p in plan.kv_positions)
        return kv, self._sent[req.id]

    monkeypatch.setattr(B200Oracle, "_device_plan", plan_kv_only)
    sc, policy = _elastic_scenario()
    with pytest.raises(AssertionError):
        sim.run(dataclasses.replace(sc, oracle_factory=_positional_factory(sc, policy, {})))
