"""Literal CPU restatement of the reference control half (test infrastructure).

Each function follows the cited reference lines statement by statement, with
plain Python data (lists / dicts), so the golden vectors produced by running the
reference itself can pin it.  Requests are dicts:
``{"out": int, "states": list[int], "queue": list[int], "block": int,
"committed": int, "steps": int}``.
"""

from __future__ import annotations

MASKED, UNCACHED, CACHED = 0, 1, 2


class OracleIllegalCommit(Exception):
    """Mirrors ``IllegalCommit`` (reference errors.py:28)."""


class OracleChunkTooSmall(Exception):
    """Mirrors ``ChunkTooSmall`` (reference errors.py:36)."""


def new_request(output_tokens: int) -> dict:
    return {"out": output_tokens, "states": [MASKED] * output_tokens, "queue": [],
            "block": 0, "committed": 0, "steps": 0}


def block_span(req: dict, block_size: int) -> tuple[int, int]:
    """reference core.py:103-107."""
    lo = req["block"] * block_size
    return lo, min(lo + block_size, req["out"])


def advance_blocks(req: dict, block_size: int) -> None:
    """reference core.py:109-116: skip blocks without MASKED positions."""
    while req["committed"] < req["out"]:
        lo, hi = block_span(req, block_size)
        if all(s != MASKED for s in req["states"][lo:hi]):
            req["block"] += 1
        else:
            break


def plan_chunk(req: dict, chunk: int, block_size: int, rule: str = "in_block") -> tuple[list, list]:
    """reference engine.py:45-67 -> (kv_positions, window)."""
    if chunk < 2:
        raise OracleChunkTooSmall(chunk)
    kv = req["queue"][: min(len(req["queue"]), chunk)]
    cap = chunk - len(kv)
    if rule == "in_block":
        lo, hi = block_span(req, block_size)
        masked = [p for p in range(lo, hi) if req["states"][p] == MASKED]
        window = masked[:cap]
    else:
        masked = [p for p in range(req["out"]) if req["states"][p] == MASKED]
        window = masked[: min(cap, block_size)]
    return list(kv), window


def apply_chunk(req: dict, kv: list, window: list, commits, block_size: int) -> int:
    """reference engine.py:70-95; returns computed token count."""
    allowed = set(window)
    for p in commits:
        if p not in allowed or req["states"][p] != MASKED:
            raise OracleIllegalCommit(p)
    for p in kv:
        head = req["queue"].pop(0)
        if head != p:
            raise OracleIllegalCommit((head, p))
        req["states"][p] = CACHED
    for p in sorted(commits):
        req["states"][p] = UNCACHED
        req["queue"].append(p)
    req["committed"] += len(commits)
    req["steps"] += 1
    advance_blocks(req, block_size)
    return len(kv) + len(window)


def commit_step_decisions(q: float, rate_multiplier: float, window_len: int, uniforms) -> list[bool]:
    """reference commit.py:103-111: rank 0 always commits; rank j>=1 commits iff
    u_j < min(1, m q^j) with u = rng.random(n-1) drawn in rank order."""
    out = [True]
    for j in range(1, window_len):
        p = min(1.0, rate_multiplier * q ** j)
        out.append(bool(uniforms[j - 1] < p))
    return out


class OracleEmptyWindow(Exception):
    """Mirrors ``EmptyWindow`` (reference errors.py:12)."""


def block_step_window(req: dict, block_size: int) -> list:
    """Masked positions of the current block (reference engine.py:100-101 / 128-131)."""
    lo, hi = block_span(req, block_size)
    return [p for p in range(lo, hi) if req["states"][p] == MASKED]


def block_diffusion_step(req: dict, commits, block_size: int) -> int:
    """reference engine.py:98-117 with the oracle's answer ``commits``: returns the
    computed count (the whole block extent)."""
    lo, hi = block_span(req, block_size)
    extent = hi - lo
    window = block_step_window(req, block_size)
    if not window:
        raise OracleEmptyWindow(req)
    for p in commits:
        if p not in window or req["states"][p] != MASKED:
            raise OracleIllegalCommit(p)
    for p in commits:
        req["states"][p] = UNCACHED
    req["committed"] += len(commits)
    req["steps"] += 1
    while all(s != MASKED for s in req["states"][lo:hi]):
        for p in range(lo, hi):
            req["states"][p] = CACHED
        advance_blocks(req, block_size)
        if req["committed"] >= req["out"]:
            break
        lo, hi = block_span(req, block_size)
    return extent


def prefix_cached_step(req: dict, commits, block_size: int) -> int:
    """reference engine.py:120-145: commits are cached at once; computed =
    extent - cached + uncached of the block before the step."""
    lo, hi = block_span(req, block_size)
    span = req["states"][lo:hi]
    cached = sum(1 for s in span if s == CACHED)
    uncached = sum(1 for s in span if s == UNCACHED)
    window = block_step_window(req, block_size)
    if not window:
        raise OracleEmptyWindow(req)
    computed = (hi - lo) - cached + uncached
    for p in commits:
        if p not in window or req["states"][p] != MASKED:
            raise OracleIllegalCommit(p)
    for p in commits:
        req["states"][p] = CACHED
    req["committed"] += len(commits)
    req["steps"] += 1
    advance_blocks(req, block_size)
    return computed


def ar_step(req: dict) -> int:
    """reference engine.py:148-157: the next position commits and caches."""
    p = req["committed"]
    if p >= req["out"]:
        raise OracleEmptyWindow(req)
    req["states"][p] = CACHED
    req["committed"] += 1
    req["steps"] += 1
    advance_blocks(req, 1)
    return 1
