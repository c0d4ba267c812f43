"""Synthetic inputs of BASELINE.json's configs (no network: no weights, no data).

* ``sample_length`` — lognormal lengths matched to (mean, std) by the method of
  moments, as the reference's workload generator does (workload.py:95-107).
* ``make_batch`` — a decode batch at SDAR-8B shape: ShareGPT-like prompt/output
  lengths (213/508 in, 321/214 out; reference workload.py:44-48) and a random
  decode progress per request, reached by replaying streaming steps with
  commit_step-style draws (commit.py:86-112) under the calibrated
  sharegpt/dense-8b profile (q = 0.7758, rate jitter sigma 1.5).
* ``SyntheticForward`` — stand-in for the model around the path: per-layer
  random Q/K/V rows and peaked logits whose max-softmax confidence is 0.97 for
  positions the commit profile would commit and 0.80 otherwise (the oracle-driven
  logits recipe), so K3 sees a realistic commit pattern.
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np
import torch

from .core import Request
from .decode import DecodeConfig, Forward
from .engine import apply_chunk, plan_chunk
from .meta import DeviceMeta

SHAREGPT = dict(prompt_mean=213.0, prompt_std=508.0, output_mean=321.0, output_std=214.0)
LONGBENCH = dict(prompt_mean=4015.0, prompt_std=2057.0, output_mean=116.0, output_std=138.0)
SHAREGPT_DENSE8B_Q = 0.7758267092770552  # calibrated_profile(sharegpt, dense-8b) (tests/golden)
SHAREGPT_DENSE8B_SIGMA = 1.5
RATE_MIN, RATE_MAX = 0.25, 4.0  # commit.py:22-23


def sample_length(mean: float, std: float, rng: np.random.Generator) -> int:
    if std == 0:
        return max(1, round(mean))
    s2 = math.log(1.0 + (std / mean) ** 2)
    mu = math.log(mean) - s2 / 2.0
    return max(1, round(rng.lognormal(mean=mu, sigma=math.sqrt(s2))))


def rate_multiplier(rng: np.random.Generator, sigma: float) -> float:
    if sigma == 0.0:
        return 1.0
    return min(RATE_MAX, max(RATE_MIN, math.exp(sigma * rng.standard_normal())))


def draw_commits(rng: np.random.Generator, window, q: float, m: float) -> set:
    """commit_step's rule (commit.py:103-111): rank 0 always, rank j w.p. min(1, m q^j)."""
    if not window:
        return set()
    out = {window[0]}
    if len(window) > 1:
        u = rng.random(len(window) - 1)
        for j, (p, uj) in enumerate(zip(window[1:], u), start=1):
            if uj < min(1.0, m * q ** j):
                out.add(p)
    return out


def make_batch(seed: int, batch: int, chunk: int, block: int = 32, rule: str = "in_block",
               lengths: dict = SHAREGPT, q: float = SHAREGPT_DENSE8B_Q,
               sigma: float = SHAREGPT_DENSE8B_SIGMA, fixed_prompt: Optional[int] = None,
               prompt_clip: Optional[tuple] = None, first_id: int = 0):
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(0,)))
    reqs = []
    for i in range(batch):
        rid = first_id + i
        prompt = fixed_prompt if fixed_prompt is not None else sample_length(
            lengths["prompt_mean"], lengths["prompt_std"], rng)
        if prompt_clip is not None:
            prompt = int(min(max(prompt, prompt_clip[0]), prompt_clip[1]))
        out = sample_length(lengths["output_mean"], lengths["output_std"], rng)
        out = max(out, 2)
        rrng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1, rid)))
        req = Request(id=rid, arrival_time=0.0, prompt_tokens=int(prompt), output_tokens=int(out), rng=rrng)
        req.rate_multiplier = rate_multiplier(rrng, sigma)
        target = int(rng.uniform(0.0, 1.0) * out)
        guard = 0
        while req.committed < target and guard < 10 * out:
            plan = plan_chunk(req, max(chunk, 2), block, rule)
            commits = draw_commits(rrng, list(plan.window), q, req.rate_multiplier)
            apply_chunk(req, plan, commits, block)
            guard += 1
        if req.finished:  # keep every request in flight
            req = Request(id=rid, arrival_time=0.0, prompt_tokens=int(prompt), output_tokens=int(out), rng=rrng)
            req.rate_multiplier = rate_multiplier(rrng, sigma)
        reqs.append(req)
    return reqs


def logit_recipe(seed: int, n_versions: int, max_slots: int, rows_per_slot: int, vocab: int, q: float,
                 sigma: float, t_hi: float = 0.97, t_lo: float = 0.80):
    """The logit table's decisions (SURVEY §8c recipe): per (version, slot, window
    rank) whether the row commits (rank 0 always; rank j w.p. min(1, m q^j), m the
    slot's rate multiplier — commit_step's rule, commit.py:103-111), its peak's
    max-softmax confidence (t_hi / t_lo around tau = 0.9) and its peak token.
    Shared by the GPU table (SyntheticForward) and the CPU reference arm (bench.py),
    which therefore take the same decisions on the same rows."""
    rng = np.random.default_rng(seed + 17)
    mult = np.array([rate_multiplier(rng, sigma) for _ in range(max_slots)])
    rank = np.arange(rows_per_slot)
    p = np.minimum(1.0, mult[None, :, None] * q ** rank[None, None, :])
    commit = rng.random((n_versions, max_slots, rows_per_slot)) < p
    commit[..., 0] = True
    conf = np.where(commit, t_hi, t_lo)
    tok = rng.integers(0, vocab, n_versions * max_slots * rows_per_slot).reshape(commit.shape)
    return commit, conf, tok


class SyntheticForward(Forward):
    """Random activations at the decode shape plus oracle-driven logits."""

    def __init__(self, cfg: DecodeConfig, max_tokens: int, max_slots: int, device="cuda", seed: int = 0,
                 n_versions: int = 2, q: float = SHAREGPT_DENSE8B_Q, sigma: float = SHAREGPT_DENSE8B_SIGMA,
                 conf_commit: float = 0.97, conf_hold: float = 0.80, vocab_shard: Optional[tuple] = None,
                 per_layer_qkv: bool = True):
        self.cfg = cfg
        self.device = torch.device(device)
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        H = cfg.num_q_heads + 2 * cfg.num_kv_heads
        n_buf = cfg.num_layers if per_layer_qkv else 1
        self.qkv_buf = [torch.randn((max_tokens, H, cfg.head_dim), generator=g, device=self.device,
                                    dtype=torch.float32).to(torch.bfloat16) for _ in range(n_buf)]
        # per-layer activations are resident: the decoder may enqueue every layer's
        # K1/K2 in one native call (no model work between the layers)
        self.resident_layers = True
        self.qkv_capacity = max_tokens
        self.max_slots = max_slots
        self.rows_per_slot = cfg.block_size
        self.n_versions = n_versions
        self.version = 0
        v0, v1 = vocab_shard if vocab_shard is not None else (0, cfg.vocab)
        self.vocab_offset = v0
        self.logit_table = self._make_logits(g, seed, q, sigma, conf_commit, conf_hold, v0, v1)
        self._row_src_pinned = None
        self._row_src_dev = None

    def _make_logits(self, g, seed, q, sigma, t_hi, t_lo, v0, v1):
        cfg = self.cfg
        n = self.n_versions * self.max_slots * self.rows_per_slot
        width = v1 - v0
        out = torch.empty((n, width), dtype=cfg.logits_dtype, device=self.device)
        commit, conf, tok = logit_recipe(seed, self.n_versions, self.max_slots, self.rows_per_slot, cfg.vocab, q,
                                         sigma, t_hi, t_lo)
        conf = conf.reshape(-1)
        chunk = 256
        V = cfg.vocab
        lg = torch.Generator(device=self.device)
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            lg.manual_seed(seed * 1000003 + a)
            x = torch.randn((b - a, V), generator=lg, device=self.device, dtype=torch.float32)
            t = torch.as_tensor(tok.reshape(-1)[a:b], device=self.device)
            x.scatter_(1, t[:, None], -float("inf"))
            lse = torch.logsumexp(x, dim=1)
            c = torch.as_tensor(conf[a:b], device=self.device, dtype=torch.float32)
            peak = lse + torch.log(c / (1 - c))
            x.scatter_(1, t[:, None], peak[:, None])
            out[a:b] = x[:, v0:v1].to(cfg.logits_dtype)
        self.expected_commit = commit
        return out

    def qkv(self, layer: int, dm: DeviceMeta):
        cfg = self.cfg
        n = max(dm.host.n_tok, 1)
        buf = self.qkv_buf[layer % len(self.qkv_buf)][:n]
        hq, hkv = cfg.num_q_heads, cfg.num_kv_heads
        return buf[:, :hq], buf[:, hq:hq + hkv], buf[:, hq + hkv:]

    def row_src_host(self, dm: DeviceMeta, slots: Optional[np.ndarray] = None) -> np.ndarray:
        m = dm.host
        rank = np.arange(m.n_rows, dtype=np.int32) - m.cu_rows[m.row_req]
        slot = m.row_req if slots is None else slots[m.row_req]
        base = self.version * self.max_slots * self.rows_per_slot
        return (base + slot * self.rows_per_slot + np.minimum(rank, self.rows_per_slot - 1)).astype(np.int32)

    def fill_row_src(self, dm) -> None:
        """Native path: write the logits-row map into the step arena before its H2D."""
        src = self.row_src_host(dm, dm.__dict__.get("slots"))
        dm.__dict__["row_src_host"][: src.size] = src
        dm.__dict__["row_src_dev"] = dm.row_src[: max(src.size, 1)]
        dm.__dict__["row_src_version"] = self.version

    def logits(self, dm: DeviceMeta):
        cached = dm.__dict__.get("row_src_dev")
        if cached is not None and dm.__dict__.get("row_src_version") == self.version:
            return self.logit_table, cached
        src = self.row_src_host(dm, dm.__dict__.get("slots"))
        n = max(src.size, 1)
        if self._row_src_pinned is None or self._row_src_pinned.numel() < n:
            self._row_src_pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
            self._row_src_dev = torch.empty(n, dtype=torch.int32, device=self.device)
        self._row_src_pinned.numpy()[: src.size] = src
        self._row_src_dev[: src.size].copy_(self._row_src_pinned[: src.size], non_blocking=True)
        dm.__dict__["extra_h2d"] = src.nbytes
        dm.__dict__["row_src_dev"] = self._row_src_dev[: max(src.size, 1)]
        dm.__dict__["row_src_version"] = self.version
        return self.logit_table, self._row_src_dev[: max(src.size, 1)]

    def next_version(self):
        self.version = (self.version + 1) % self.n_versions


class OracleDrivenForward(Forward):
    """Stand-in model whose logits encode the reference's commit draw.

    For every request with a non-empty window it consumes the request's rng exactly
    like ``commit_step`` (commit.py:104-111: ``rng.random(n - 1)`` when n > 1) and
    synthesizes each window row's logits with max-softmax confidence 0.97 (rank 0,
    and rank j >= 1 when u_j < min(1, m q^j)) or 0.80 otherwise.  With tau = 0.9 the
    B200 unmask kernel must then reproduce StochasticOracle's commit sets exactly,
    which makes the whole device step comparable with the reference schedule.
    """

    def __init__(self, cfg: DecodeConfig, max_tokens: int, q: float, device="cuda", seed: int = 0,
                 conf_commit: float = 0.97, conf_hold: float = 0.80):
        self.cfg = cfg
        self.q = q
        self.device = torch.device(device)
        self.t_hi, self.t_lo = conf_commit, conf_hold
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        H = cfg.num_q_heads + 2 * cfg.num_kv_heads
        self.qkv_buf = [torch.randn((max_tokens, H, cfg.head_dim), generator=g, device=self.device,
                                    dtype=torch.float32).to(torch.bfloat16) for _ in range(cfg.num_layers)]
        self.resident_layers = True
        self.qkv_capacity = max_tokens
        self.gen = torch.Generator(device=self.device)
        self.gen.manual_seed(seed + 1)
        self.tok_rng = np.random.default_rng(seed + 2)

    def qkv(self, layer: int, dm: DeviceMeta):
        n = max(dm.host.n_tok, 1)
        buf = self.qkv_buf[layer][:n]
        hq, hkv = self.cfg.num_q_heads, self.cfg.num_kv_heads
        return buf[:, :hq], buf[:, hq:hq + hkv], buf[:, hq + hkv:]

    def logits(self, dm: DeviceMeta):
        reqs = dm.__dict__["requests"]
        cu_rows = dm.host.cu_rows
        confs = []
        for r, req in enumerate(reqs):
            n = int(cu_rows[r + 1] - cu_rows[r])  # window rows of request r (ChunkPlan.window)
            if n == 0:
                continue
            m = float(getattr(req, "rate_multiplier", 1.0))
            dec = [True]
            if n > 1:
                u = req.rng.random(n - 1)
                dec += [bool(uj < min(1.0, m * self.q ** j)) for j, uj in enumerate(u, start=1)]
            confs += [self.t_hi if d else self.t_lo for d in dec]
        return self._peaked(confs), None

    def _peaked(self, confs):
        """Window-row logits with max-softmax confidence confs[i] (SURVEY §8c recipe)."""
        n_rows = len(confs)
        V = self.cfg.vocab
        x = torch.randn((max(n_rows, 1), V), generator=self.gen, device=self.device, dtype=torch.float32)
        if n_rows:
            tok = torch.as_tensor(self.tok_rng.integers(0, V, n_rows), device=self.device)
            x.scatter_(1, tok[:, None], -float("inf"))
            lse = torch.logsumexp(x, dim=1)
            c = torch.as_tensor(confs, device=self.device, dtype=torch.float32)
            x.scatter_(1, tok[:, None], (lse + torch.log(c / (1 - c)))[:, None])
        return x.to(self.cfg.logits_dtype)


class ReferenceOracleForward(OracleDrivenForward):
    """Stand-in model whose logits encode ANY reference commit oracle's decisions
    (``StochasticOracle``, ``ReplayOracle``, a test's custom oracle: the duck-typed
    protocol of engine.py:105-110).  For every request with window rows in the step,
    ``inner.commits(request, window)`` is asked once and each row's logits get
    confidence 0.97 (committed) or 0.80 (held); with tau = 0.9 and fallback "none"
    the B200 unmask reproduces the inner oracle's sets exactly.  ``consume`` is
    forwarded, so carry-over replay keeps working.  This is how the B200 oracle is
    driven inside dllmsim's own loop (``Scenario.oracle_factory``, sim.py:64,128-132)
    without a model checkpoint."""

    def __init__(self, cfg: DecodeConfig, inner, max_tokens: int, device="cuda", seed: int = 0, **kw):
        super().__init__(cfg, max_tokens, 0.0, device=device, seed=seed, **kw)
        self.inner = inner

    def logits(self, dm: DeviceMeta):
        reqs = dm.__dict__["requests"]
        cu_rows, row_pos = dm.host.cu_rows, dm.host.row_pos
        confs = []
        for r, req in enumerate(reqs):
            a, b = int(cu_rows[r]), int(cu_rows[r + 1])
            if b == a:
                continue
            window = [int(p) for p in row_pos[a:b]]
            got = self.inner.commits(req, window)
            confs += [self.t_hi if p in got else self.t_lo for p in window]
        return self._peaked(confs), None

    def consume(self, request, committed) -> None:
        fn = getattr(self.inner, "consume", None)
        if fn is not None:
            fn(request, committed)


class TPForward(SyntheticForward):
    """SyntheticForward plus the row-parallel o-proj + all-reduce after every
    layer's attention (BASELINE configs[4]: head-sharded attention, NCCL o-proj
    all-reduce).  Layers run one at a time (the o-proj sits between them)."""

    def __init__(self, cfg: DecodeConfig, max_tokens: int, max_slots: int, hidden: int, full_q_heads: int,
                 world: int = 1, rank: int = 0, group=None, **kw):
        super().__init__(cfg, max_tokens, max_slots, **kw)
        from .tp import RowParallelOProj
        self.resident_layers = False
        self.oproj = RowParallelOProj(cfg.num_layers, full_q_heads, cfg.head_dim, hidden, world, rank,
                                      device=self.device, seed=kw.get("seed", 0), group=group)
        self.last_hidden = None

    def post_attn(self, layer: int, attn_out, dm) -> None:
        n = dm.host.n_tok
        if n:
            self.last_hidden = self.oproj(layer, attn_out[:n])
