"""CPU tests of the host side of the device step: metadata packing (rule V
bitmaps) and the split-KV / persistent-CTA planner (pure host code inside the
C-ABI library, callable without a GPU)."""

import numpy as np
import pytest

from oracle import numeric as on
from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.meta import build_step_meta
from tests.scenario import make_block_tables, make_requests


def _expand_bits(meta, r):
    """Per-key visibility (before the block-causal cap) encoded by the bitmap."""
    ke = int(meta.key_end[r])
    vb = int(meta.vis_base[r])
    w0, w1 = int(meta.vis_off[r]), int(meta.vis_off[r + 1])
    words = meta.vis_words[w0:w1]
    vis = np.ones(ke, dtype=bool)
    for s in range(vb, ke):
        vis[s] = bool((int(words[(s - vb) >> 5]) >> ((s - vb) & 31)) & 1)
    return vis


@pytest.mark.parametrize("rule", ["in_block", "out_block"])
@pytest.mark.parametrize("chunk", [2, 8, 32])
def test_bitmaps_match_oracle_rule_v(rule, chunk):
    rng = np.random.default_rng(chunk)
    block = 32
    reqs = make_requests(7 + chunk, 12, (1, 90), (2, 140), chunk, block, rule)
    plans = pe.plan_batch(reqs, chunk, block, rule)
    bt, _ = make_block_tables(rng, reqs, 16)
    meta = build_step_meta(reqs, plans, block, bt)
    assert meta.vis_base.min() >= 0 and (meta.vis_base % 32 == 0).all()
    for r, (req, plan) in enumerate(zip(reqs, plans)):
        t0, t1 = int(meta.cu_seqlens[r]), int(meta.cu_seqlens[r + 1])
        assert list(meta.tok_pos[t0:t1]) == list(plan.kv_positions) + list(plan.window)
        if t1 == t0:
            continue
        vis_out = on.visible_outputs(req.states, list(plan.kv_positions) + list(plan.window))
        n_keys = req.prompt_tokens + req.output_tokens
        ref = on.key_mask(req.prompt_tokens, vis_out, meta.tok_pos[t0:t1], block, n_keys)
        ke = int(meta.key_end[r])
        # nothing any query can see lies beyond key_end
        assert not ref[:, ke:].any()
        bits = _expand_bits(meta, r)
        for i, qp in enumerate(meta.tok_pos[t0:t1]):
            lim = min(req.prompt_tokens + (qp // block + 1) * block, ke)
            got = bits.copy()
            got[lim:] = False
            assert np.array_equal(got, ref[i, :ke]), (r, i)
        # window rows for the unmask kernel
        a, b = int(meta.cu_rows[r]), int(meta.cu_rows[r + 1])
        assert list(meta.row_pos[a:b]) == list(plan.window)
        assert list(meta.tok_pos[meta.row_tok[a:b]]) == list(plan.window)


def _plan(cu, ke, hq, hkv, grid, min_split=4, page_size=64):
    from paper_2605_24832_b200.ops import plan_attention
    return plan_attention(np.asarray(cu), np.asarray(ke), hq, hkv, grid=grid, min_split_tiles=min_split,
                          page_size=page_size)


@pytest.mark.parametrize("hq,hkv", [(32, 8), (4, 4), (4, 2), (32, 4)])
def test_planner_covers_every_key_tile_once(hq, hkv):
    rng = np.random.default_rng(hq + hkv)
    n = 37
    counts = rng.integers(0, 40, n)
    cu = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    ke = rng.integers(1, 9000, n).astype(np.int32)
    for grid in (1, 7, 148):
        plan = _plan(cu, ke, hq, hkv, grid, page_size=64)
        G = hq // hkv
        T = 128 // G
        w = plan.work_host
        off = plan.cta_off_host
        assert off[0] == 0 and off[-1] == plan.n_work and (np.diff(off) >= 0).all()
        cover = {}
        for it in w:
            req, head, tb, nt, kb, kend, slot, _ = it
            assert 0 <= head < hkv and kb % 64 == 0 and kend > kb and kend <= ke[req]
            assert cu[req] <= tb and tb + nt <= cu[req + 1] and 1 <= nt <= T
            cover.setdefault((req, head, tb), []).append((kb, kend, slot))
        for r in range(n):
            nq = counts[r]
            for h in range(hkv):
                for t0 in range(0, nq, T):
                    ranges = sorted(cover.pop((r, h, cu[r] + t0)))
                    assert ranges[0][0] == 0 and ranges[-1][1] == ke[r]
                    for a, b in zip(ranges, ranges[1:]):
                        assert a[1] == b[0]
                    if len(ranges) == 1:
                        assert ranges[0][2] == -1
                    else:
                        assert all(x[2] >= 0 for x in ranges)
        assert not cover
        # an item never spans more than 255 pages (kernel stages its page ids in smem)
        assert (((w[:, 5] - 1) // 64) - (w[:, 4] // 64) + 1 <= 255).all()
        slots = sorted(s for s in w[:, 6] if s >= 0)
        assert slots == list(range(plan.n_partials))
        for g in plan.groups_host:
            req, head, tb, nt, slot0, ns, _, _ = g
            assert ns >= 2


def test_planner_balances_uniform_long_contexts():
    # 64 requests x 4096 keys x 8 heads on 148 CTAs: LPT + splitting keeps the
    # busiest CTA within 10% of the mean load.
    n = 64
    cu = np.arange(0, 33 * (n + 1), 33)[: n + 1].astype(np.int32)
    ke = np.full(n, 4096 + 32, dtype=np.int32)
    plan = _plan(cu, ke, 32, 8, 148)
    tiles = (plan.work_host[:, 5] - plan.work_host[:, 4] + 63) // 64
    per_cta = [tiles[a:b].sum() + 2 * (b - a) for a, b in zip(plan.cta_off_host[:-1], plan.cta_off_host[1:])]
    assert max(per_cta) <= 1.12 * np.mean(per_cta)


@pytest.mark.parametrize("hq,hkv,maxq", [(32, 8, 33), (32, 8, 41), (64, 8, 20), (4, 4, 140), (12, 4, 50)])
def test_single_query_tile_matches_work_list(hq, hkv, maxq):
    """plan.single_tile (precondition of the fused append) holds exactly when every
    (request, KV head) is one query tile in the planner's work list."""
    rng = np.random.default_rng(hq * 7 + maxq)
    for _ in range(6):
        n = 23
        counts = rng.integers(0, maxq, n)
        cu = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        ke = rng.integers(1, 5000, n).astype(np.int32)
        plan = _plan(cu, ke, hq, hkv, 148, page_size=64)
        w = plan.work_host
        pairs = np.unique(w[:, [0, 2]], axis=0)
        one_group = len(pairs) == len(np.unique(pairs[:, 0]))
        assert plan.single_tile == one_group
