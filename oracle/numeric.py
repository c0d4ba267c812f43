"""CPU restatement of the numeric half of the decode step (test infrastructure).

Rules (the reference states them in prose only):

S  slot mapping (core.py:3-4): absolute position s = prompt + p,
   slot = block_table[s // P] * P + s % P.
K  KV append: every planned token (kv rows and window rows) writes its K/V row.
V  visibility (engine.py:58-66): a query at output position
   p_q sees key s iff s < prompt, or (p = s - prompt) satisfies
   p // B <= p_q // B (block-causal, bidirectional inside a block) and p was
   DECODED_CACHED before the step or is planned in this step.
U  unmask (commit.py:103): per window row
   conf = max softmax probability (float64 here), tok = argmax (lowest index on
   ties); commit iff conf >= tau; progress rule "earliest" always commits the
   first window row, "top1" commits the most confident row when none passes.

Everything is numpy; attention is computed per (request, kv head) with the G
query heads of a group folded into the row dimension (no repeat of K/V).
"""

from __future__ import annotations

import numpy as np

CACHED = 2


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even), returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = rounded.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(a), a, out).reshape(a.shape)


def v_storage(v: np.ndarray, dtype: str) -> np.ndarray:
    """V rows as the cache stores them, as int16 bit patterns: bf16 unchanged, or
    fp16 (round-to-nearest, saturating at +-65504 — exact for bf16 values in range)."""
    v = np.asarray(v, dtype=np.float32)
    if dtype == "fp16":
        return np.clip(v, -65504.0, 65504.0).astype(np.float16).view(np.int16)
    b = bf16_round(v).view(np.uint32) >> 16
    return b.astype(np.uint16).view(np.int16)


def slot_mapping(tok_req, tok_pos, prompt_len, block_tables, page_size: int) -> np.ndarray:
    """Rule S for every planned token."""
    tok_req = np.asarray(tok_req)
    s = np.asarray(prompt_len)[tok_req] + np.asarray(tok_pos)
    pages = np.asarray(block_tables)[tok_req, s // page_size]
    return pages.astype(np.int64) * page_size + s % page_size


def kv_append(k_cache: np.ndarray, v_cache: np.ndarray, k_new, v_new, slots, page_size: int) -> None:
    """Rule K: cache[page, h, off, :] = new[i, h, :] (caches [pages, Hkv, P, d])."""
    slots = np.asarray(slots)
    pages, offs = slots // page_size, slots % page_size
    k_cache[pages, :, offs, :] = np.asarray(k_new)
    v_cache[pages, :, offs, :] = np.asarray(v_new)


def visible_outputs(states_before: np.ndarray, planned) -> np.ndarray:
    """Output positions whose KV is valid in this step (rule V, state part)."""
    vis = np.asarray(states_before) == CACHED
    vis = vis.copy()
    vis[list(planned)] = True
    return vis


def key_mask(prompt: int, vis_out: np.ndarray, q_pos, block_size: int, n_keys: int) -> np.ndarray:
    """Boolean [n_q, n_keys]: which absolute keys each query sees (rule V)."""
    s = np.arange(n_keys)
    p = s - prompt
    q_pos = np.asarray(q_pos)
    out_ok = np.zeros(n_keys, dtype=bool)
    inside = (p >= 0) & (p < len(vis_out))
    out_ok[inside] = vis_out[p[inside]]
    base = (s < prompt) | out_ok
    causal = (p[None, :] // block_size) <= (q_pos[:, None] // block_size)
    return base[None, :] & ((s[None, :] < prompt) | causal)


def gather_keys(cache: np.ndarray, block_table, n_keys: int, page_size: int) -> np.ndarray:
    """[n_keys, Hkv, d] rows of one request, read through its block table."""
    s = np.arange(n_keys)
    pages = np.asarray(block_table)[s // page_size]
    return cache[pages, :, s % page_size, :]


def paged_attention(q, k_cache, v_cache, cu_seqlens, q_pos, prompt_len, vis_out_list,
                    block_tables, block_size: int, page_size: int, sm_scale=None,
                    dtype=np.float32, workers: int = 1) -> np.ndarray:
    """Reference output [n_tok, Hq, d] for the decode step.

    ``vis_out_list[r]`` is the boolean visibility of request r's output positions
    (``visible_outputs``).  Keys considered: [0, prompt + len(vis_out)).
    """
    q = np.asarray(q, dtype=dtype)
    n_tok, hq, d = q.shape
    hkv = k_cache.shape[1]
    G = hq // hkv
    scale = (1.0 / np.sqrt(d)) if sm_scale is None else sm_scale
    out = np.zeros((n_tok, hq, d), dtype=np.float32)

    def one(r):
        t0, t1 = int(cu_seqlens[r]), int(cu_seqlens[r + 1])
        if t1 == t0:
            return
        prompt = int(prompt_len[r])
        vis_out = vis_out_list[r]
        n_keys = prompt + len(vis_out)
        mask = key_mask(prompt, vis_out, q_pos[t0:t1], block_size, n_keys)  # [nq, n_keys]
        K = gather_keys(k_cache, block_tables[r], n_keys, page_size).astype(dtype)
        V = gather_keys(v_cache, block_tables[r], n_keys, page_size).astype(dtype)
        nq = t1 - t0
        for h in range(hkv):
            Q = q[t0:t1, h * G:(h + 1) * G, :].reshape(nq * G, d)        # row = t*G + g
            S = (Q @ K[:, h, :].T) * dtype(scale)
            m = np.repeat(mask, G, axis=0)
            S = np.where(m, S, -np.inf)
            S = S - S.max(axis=1, keepdims=True)
            P = np.exp(S)
            P /= P.sum(axis=1, keepdims=True)
            O = P @ V[:, h, :]
            out[t0:t1, h * G:(h + 1) * G, :] = O.reshape(nq, G, d)

    _for_each(one, range(len(cu_seqlens) - 1), workers)
    return out


def _for_each(fn, items, workers: int) -> None:
    """Run fn over items, on `workers` threads when > 1 (numpy releases the GIL in
    its array kernels; requests / row blocks are independent)."""
    items = list(items)
    if workers <= 1:
        for i in items:
            fn(i)
        return
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(workers) as ex:
        for _ in ex.map(fn, items):
            pass


def unmask(logits, cu_rows, tau: float = 0.9, fallback: str = "earliest", workers: int = 1):
    """Rule U -> (commit_mask bool[n], tok int64[n], conf float64[n])."""
    x = np.asarray(logits)
    n = x.shape[0]
    tok = np.zeros(n, dtype=np.int64)
    conf = np.zeros(n, dtype=np.float64)

    def rows(a):
        b = min(n, a + 16)
        xb = np.asarray(x[a:b], dtype=np.float64)
        tok[a:b] = np.argmax(xb, axis=1)
        conf[a:b] = 1.0 / np.exp(xb - xb.max(axis=1, keepdims=True)).sum(axis=1)

    _for_each(rows, range(0, n, 16), workers)
    commit = conf >= tau
    for r in range(len(cu_rows) - 1):
        a, b = int(cu_rows[r]), int(cu_rows[r + 1])
        if b <= a:
            continue
        if fallback == "earliest":
            commit[a] = True
        elif fallback == "top1" and not commit[a:b].any():
            commit[a + int(np.argmax(conf[a:b]))] = True
    return commit, tok, conf


def peaked_logits(rng: np.random.Generator, n_rows: int, vocab: int, tokens, confs) -> np.ndarray:
    """Oracle-driven logits recipe (SURVEY §8c parity harness): background N(0,1)
    plus one peak ``S + ln(t/(1-t))`` with S = logsumexp of the other columns, so
    the max softmax probability is t (before bf16 rounding)."""
    x = rng.standard_normal((n_rows, vocab)).astype(np.float32)
    for i in range(n_rows):
        t = float(confs[i])
        k = int(tokens[i])
        others = np.delete(x[i].astype(np.float64), k)
        mx = others.max()
        lse = mx + np.log(np.exp(others - mx).sum())
        x[i, k] = np.float32(lse + np.log(t / (1.0 - t)))
    return x


def unmask_partial_ref(logits_shard, vocab_offset: int = 0):
    """Per-row {max, sum exp(x - max), argmax + offset} of one vocabulary shard
    (the record the unmask partials kernel writes; float64 here)."""
    x = np.asarray(logits_shard, dtype=np.float64)
    m = x.max(axis=1)
    s = np.exp(x - m[:, None]).sum(axis=1)
    idx = np.argmax(x, axis=1) + vocab_offset
    return m, s, idx


def unmask_merge_ref(parts):
    """Merge shard records in the given (fixed) order: larger max wins, ties keep
    the lower index; sums are rescaled to the merged max."""
    M, S, I = [np.array(a, copy=True) for a in parts[0]]
    for m2, s2, i2 in parts[1:]:
        take = (m2 > M) | ((m2 == M) & (i2 < I))
        newM = np.maximum(M, m2)
        S = S * np.exp(M - newM) + s2 * np.exp(m2 - newM)
        I = np.where(take, i2, I)
        M = newM
    return M, S, I
