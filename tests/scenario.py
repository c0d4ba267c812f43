"""Seeded decode-step scenarios shared by the CPU and GPU tests.

Request states are produced by replaying the reference's own step rule
(plan_chunk / apply_chunk with commit_step-style draws) to a random progress, so
the visibility patterns are the ones real streaming decoding produces
(non-contiguous commits, KV backlog crossing block boundaries, ...).
"""

from __future__ import annotations

import numpy as np

from oracle import control as oc
from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.core import Request


def replay_to_progress(req: Request, rng, chunk: int, block: int, rule: str, q: float, frac: float):
    """Advance ``req`` through streaming steps until ~frac of it is committed."""
    target = int(frac * req.output_tokens)
    guard = 0
    while req.committed < target and not req.finished and guard < 10 * req.output_tokens:
        plan = pe.plan_chunk(req, chunk, block, rule)
        if plan.window:
            u = rng.random(len(plan.window) - 1) if len(plan.window) > 1 else []
            dec = oc.commit_step_decisions(q, 1.0, len(plan.window), u)
            commits = {p for p, c in zip(plan.window, dec) if c}
        else:
            commits = set()
        pe.apply_chunk(req, plan, commits, block)
        guard += 1


def make_requests(seed: int, n_req: int, prompt_range, out_range, chunk: int, block: int,
                  rule: str = "in_block", q: float = 0.78, fixed_prompt=None):
    rng = np.random.default_rng(seed)
    reqs = []
    for i in range(n_req):
        if fixed_prompt is None or isinstance(fixed_prompt, dict):
            prompt = int(rng.integers(*prompt_range))
            if fixed_prompt is not None:  # per-request overrides
                prompt = int(fixed_prompt.get(i, prompt))
        else:
            prompt = int(fixed_prompt)
        out = int(rng.integers(*out_range))
        r = Request(id=i, arrival_time=0.0, prompt_tokens=prompt, output_tokens=out,
                    rng=np.random.default_rng(seed * 1000 + i))
        replay_to_progress(r, rng, max(chunk, 2), block, rule, q, float(rng.uniform(0.0, 0.9)))
        if r.finished:  # keep every request decodable
            r = Request(id=i, arrival_time=0.0, prompt_tokens=prompt, output_tokens=out,
                        rng=np.random.default_rng(seed * 1000 + i))
        reqs.append(r)
    return reqs


def make_block_tables(rng, reqs, page_size: int, num_pages: int = None, max_pages: int = None):
    """Shuffled physical pages covering prompt + output of every request."""
    need = [(r.prompt_tokens + r.output_tokens + page_size - 1) // page_size for r in reqs]
    if max_pages is None:
        max_pages = max(need)
    total = sum(need)
    if num_pages is None:
        num_pages = total + 3
    perm = rng.permutation(num_pages)
    bt = np.zeros((len(reqs), max_pages), dtype=np.int32)
    k = 0
    for i, n in enumerate(need):
        bt[i, :n] = perm[k:k + n]
        k += n
    return bt, num_pages
