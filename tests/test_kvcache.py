"""Page pool and block tables (kvcache.py): pages are allocated when a request's
positions need them (prompt + first block at admission, later blocks as the plan
reaches them), freed at finish, and never shared between live requests; every
position a step plans has a page before K1 writes it (rule S)."""

import numpy as np
import pytest

from paper_2605_24832_b200.errors import ConfigError
from paper_2605_24832_b200.kvcache import BlockTables, PagePool


def test_pool_alloc_free_lifo_and_exhaustion():
    pool = PagePool(8)
    a = pool.alloc(3)
    assert a == [0, 1, 2] and pool.free_pages == 5
    b = pool.alloc(2)
    assert b == [3, 4]
    pool.free(a)
    assert pool.free_pages == 6
    assert pool.alloc(3) == a  # most recently freed first, same order
    with pytest.raises(ConfigError):
        pool.alloc(4)
    assert pool.alloc(0) == []


def test_admit_ensure_release():
    pool = PagePool(32)
    bt = BlockTables(pool, max_slots=4, max_pages=8, page_size=16)
    s0 = bt.admit(100, 40)          # 3 pages
    assert bt.n_pages[s0] == 3 and bt.slot(100) == s0
    bt.ensure(s0, 48)               # still 3
    assert bt.n_pages[s0] == 3
    bt.ensure(s0, 49)               # opens a 4th page
    assert bt.n_pages[s0] == 4
    s1 = bt.admit(101, 16)
    assert s1 != s0
    live = set(bt.table[s0, :4].tolist()) | set(bt.table[s1, :1].tolist())
    assert len(live) == 5           # no page shared between live requests
    with pytest.raises(ConfigError):
        bt.admit(100, 1)            # admitted twice
    with pytest.raises(ConfigError):
        bt.ensure(s1, 16 * 9)       # > max_pages
    free0 = pool.free_pages
    bt.release(100)
    assert pool.free_pages == free0 + 4 and bt.slot(100) is None
    assert not bt.table[s0].any() and bt.n_pages[s0] == 0  # row cleared
    s2 = bt.admit(102, 1, slot=s0)
    assert s2 == s0
    with pytest.raises(ConfigError):
        bt.admit(103, 1, slot=s1)   # taken


def test_random_admit_release_never_shares_pages():
    rng = np.random.default_rng(0)
    pool = PagePool(256)
    bt = BlockTables(pool, max_slots=16, max_pages=32, page_size=16)
    live = {}
    nid = 0
    for _ in range(2000):
        op = rng.random()
        if op < 0.35 and len(live) < 16:
            try:
                live[nid] = bt.admit(nid, int(rng.integers(1, 100)))
            except ConfigError:
                pass
            nid += 1
        elif op < 0.7 and live:
            rid = int(rng.choice(list(live)))
            try:
                bt.ensure(live[rid], int(rng.integers(1, 16 * 32)))
            except ConfigError:
                pass
        elif live:
            rid = int(rng.choice(list(live)))
            bt.release(rid)
            del live[rid]
        pages = [p for s in live.values() for p in bt.table[s, : bt.n_pages[s]].tolist()]
        assert len(pages) == len(set(pages))
        assert len(pages) + pool.free_pages == 256


@pytest.mark.gpu
@pytest.mark.parametrize("chunk,fallback", [(48, "earliest"), (64, "earliest"), (32, "top1")])
def test_out_block_plans_never_touch_unallocated_pages(chunk, fallback):
    """OUT_BLOCK windows take the earliest masked positions anywhere in the output,
    so a step can reach blocks past the current one.  Through the native step
    (StreamingDecoder.step), every planned position must have a page of its own
    request when K1 runs, and no page may belong to two live requests."""
    import torch

    from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
    from paper_2605_24832_b200.synthetic import OracleDrivenForward, make_batch

    block, page = 32, 64
    cfg = DecodeConfig(num_layers=1, num_q_heads=8, num_kv_heads=2, head_dim=128, vocab=2048, block_size=block,
                       page_size=page, window_rule="out_block", fallback=fallback, max_batch=16,
                       max_pages_per_req=32, num_pages=16 * 32)
    reqs = make_batch(3, 12, chunk, block, rule="out_block")
    for r in reqs:
        assert r.prompt_tokens + r.output_tokens <= 32 * page or pytest.skip("long request")
    dec = StreamingDecoder(cfg, OracleDrivenForward(cfg, 16 * chunk, 0.6, seed=5))
    nat = dec.native()
    plan0 = nat.plan
    seen = {"steps": 0, "beyond": 0}

    def checked_plan(requests, c):
        dm = plan0(requests, c)
        m = dm.host
        owner = {}
        for i, req in enumerate(requests):
            s = int(dm.slots[i])
            npg = int(dec.tables.n_pages[s])
            owned = dec.tables.table[s, :npg].tolist()
            for p in owned:
                assert owner.setdefault(p, req.id) == req.id, "page shared by two live requests"
            for t in range(int(m.cu_seqlens[i]), int(m.cu_seqlens[i + 1])):
                a = req.prompt_tokens + int(m.tok_pos[t])
                assert a // page < npg, (req.id, int(m.tok_pos[t]), npg)
                assert int(m.block_tables[i, a // page]) == owned[a // page]
                seen["beyond"] += int(m.tok_pos[t]) // block > req.block_index
        seen["steps"] += 1
        return dm

    nat.plan = checked_plan
    live = list(reqs)
    while live:
        dec.step(live, chunk)
        live = [r for r in live if not r.finished]
        assert seen["steps"] < 400
    torch.cuda.synchronize()
    assert seen["beyond"] > 0  # the case the check is about did occur
