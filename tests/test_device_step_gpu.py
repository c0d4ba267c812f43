"""Device twins of the native host step (csrc/device_step.cu, SURVEY §8f-1 device
half): optimus_device_plan / optimus_device_apply over device-resident packed state
produce the same step metadata and state transitions as optimus_host_plan /
optimus_host_apply (themselves pinned to the Python mirror and to dllmsim), bit for
bit, step by step over whole decodes."""

import copy

import numpy as np
import pytest
import torch

from paper_2605_24832_b200 import _lib
from paper_2605_24832_b200.batch_state import BatchState
from tests.scenario import make_requests
from tests.test_host_step import _native_apply, _native_plan

pytestmark = pytest.mark.gpu

CAPS = 4096


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _p(t):
    return t.data_ptr() if t is not None else None


@pytest.mark.parametrize("rule,chunk,block", [("in_block", 8, 32), ("in_block", 32, 32), ("out_block", 8, 16),
                                              ("in_block", 2, 8), ("in_block", "mixed", 32)])
def test_device_plan_and_apply_match_host(rule, chunk, block):
    rng = np.random.default_rng(40 + block + (7 if chunk == "mixed" else chunk))
    reqs = make_requests(21 + block, 12, (1, 300), (3, 200), 8, block, rule)
    bs = BatchState(16, 256, qcap=64)
    for i, r in enumerate(copy.deepcopy(reqs)):
        bs.bind(r, i)
    tables = np.arange(16 * 40, dtype=np.int32).reshape(16, 40)
    # device copy of the packed state
    D = {k: _dev(getattr(bs, k)) for k in ("states", "queue", "q_head", "q_len", "block_index", "committed",
                                            "steps_taken", "cached_prefix", "prompt", "out_len")}
    Dt = _dev(tables)
    L = _lib.load()
    stream = torch.cuda.current_stream().cuda_stream
    steps = 0
    while True:
        idx = [i for i in range(len(reqs)) if bs.committed[i] < bs.out_len[i]]
        if not idx:
            break
        n = len(idx)
        c = rng.choice([2, 4, 8, 16, 24, 32], n).astype(np.int32) if chunk == "mixed" else chunk
        out, counts = _native_plan(bs, idx, c, block, rule, tables, caps=CAPS)
        n_tok, n_rows, n_words = (int(x) for x in counts[:3])
        # device plan
        O = {k: torch.zeros(n + 1, dtype=torch.int32, device="cuda") for k in ("cu_seqlens", "vis_off", "cu_rows")}
        O.update({k: torch.zeros(n, dtype=torch.int32, device="cuda") for k in ("prompt_len", "key_end", "vis_base")})
        O.update({k: torch.zeros(CAPS, dtype=torch.int32, device="cuda")
                  for k in ("tok_req", "tok_pos", "row_tok", "row_pos", "row_req", "vis_words")})
        O["block_tables"] = torch.zeros((n, tables.shape[1]), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(4, dtype=torch.int32, device="cuda")
        sl = _dev(np.asarray(idx, dtype=np.int32))
        cpr = _dev(c) if chunk == "mixed" else None
        st = L.optimus_device_plan(
            n, _p(sl), 0 if chunk == "mixed" else chunk, _p(cpr), block, 0 if rule == "in_block" else 1,
            _p(D["states"]), D["states"].shape[1], _p(D["queue"]), bs.qcap, _p(D["q_head"]), _p(D["q_len"]),
            _p(D["block_index"]), _p(D["cached_prefix"]), _p(D["prompt"]), _p(D["out_len"]), _p(Dt),
            tables.shape[1], _p(O["cu_seqlens"]), _p(O["tok_req"]), _p(O["tok_pos"]), CAPS, _p(O["prompt_len"]),
            _p(O["key_end"]), _p(O["vis_base"]), _p(O["vis_off"]), _p(O["vis_words"]), CAPS, _p(O["cu_rows"]),
            _p(O["row_tok"]), _p(O["row_pos"]), _p(O["row_req"]), CAPS, _p(O["block_tables"]), _p(cnt), stream)
        assert st == 0
        torch.cuda.synchronize()
        assert cnt.cpu().tolist() == [n_tok, n_rows, n_words, 0], steps
        for k in ("cu_seqlens", "prompt_len", "key_end", "vis_base", "vis_off", "cu_rows"):
            assert np.array_equal(O[k].cpu().numpy(), out[k]), (k, steps)
        for k, m in (("tok_req", n_tok), ("tok_pos", n_tok), ("row_tok", n_rows), ("row_pos", n_rows),
                     ("row_req", n_rows)):
            assert np.array_equal(O[k].cpu().numpy()[:m], out[k][:m]), (k, steps)
        assert np.array_equal(O["vis_words"].cpu().numpy().view(np.uint32)[:n_words], out["vis_words"][:n_words])
        assert np.array_equal(O["block_tables"].cpu().numpy(), out["block_tables"])
        # commits: random, the first window row of each request always
        mask = rng.random(n_rows) < 0.35
        for r in range(n):
            a, b = out["cu_rows"][r], out["cu_rows"][r + 1]
            if b > a:
                mask[a] = True
        commits_h = _native_apply(bs, idx, block, out, mask)
        commits_d = torch.zeros(n, dtype=torch.int32, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        dm = _dev(mask.astype(np.uint8))
        st = L.optimus_device_apply(
            n, _p(sl), block, _p(O["cu_seqlens"]), _p(O["tok_pos"]), _p(O["cu_rows"]), _p(O["row_pos"]), _p(dm),
            _p(D["states"]), D["states"].shape[1], _p(D["queue"]), bs.qcap, _p(D["q_head"]), _p(D["q_len"]),
            _p(D["block_index"]), _p(D["committed"]), _p(D["steps_taken"]), _p(D["cached_prefix"]),
            _p(D["out_len"]), _p(commits_d), _p(status), stream)
        assert st == 0
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        assert commits_d.cpu().tolist() == list(commits_h)
        for k in ("states", "q_head", "q_len", "block_index", "committed", "steps_taken", "cached_prefix"):
            assert np.array_equal(D[k].cpu().numpy(), getattr(bs, k)), (k, steps)
        # the ring: compare the live entries
        for i in range(len(reqs)):
            h, ln = int(bs.q_head[i]), int(bs.q_len[i])
            live = [(h + j) % bs.qcap for j in range(ln)]
            assert np.array_equal(D["queue"].cpu().numpy()[i][live], bs.queue[i][live])
        steps += 1
        assert steps < 500
    assert steps > 5


def test_device_apply_rejects_out_of_order_kv():
    bs = BatchState(2, 64, qcap=8)
    reqs = make_requests(5, 1, (3, 10), (20, 30), 8, 16, "in_block")
    for i, r in enumerate(reqs):
        bs.bind(r, i)
    L = _lib.load()
    # a plan claiming a kv position the ring does not hold at its front
    cu = _dev(np.array([0, 1], np.int32))
    tok = _dev(np.array([5], np.int32))
    cur = _dev(np.array([0, 0], np.int32))
    rp = _dev(np.zeros(1, np.int32))
    D = {k: _dev(getattr(bs, k)) for k in ("states", "queue", "q_head", "q_len", "block_index", "committed",
                                            "steps_taken", "cached_prefix", "out_len")}
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    sl0, m0, c0 = _dev(np.array([0], np.int32)), _dev(np.zeros(1, np.uint8)), torch.zeros(1, dtype=torch.int32,
                                                                                           device="cuda")
    st = L.optimus_device_apply(
        1, _p(sl0), 16, _p(cu), _p(tok), _p(cur), _p(rp), _p(m0),
        _p(D["states"]), D["states"].shape[1], _p(D["queue"]), bs.qcap, _p(D["q_head"]), _p(D["q_len"]),
        _p(D["block_index"]), _p(D["committed"]), _p(D["steps_taken"]), _p(D["cached_prefix"]), _p(D["out_len"]),
        _p(c0), _p(status), torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    assert int(status.item()) == -1
    for k in ("states", "q_head", "q_len", "committed", "steps_taken"):  # nothing applied
        assert np.array_equal(D[k].cpu().numpy(), getattr(bs, k)), k


def test_device_apply_is_atomic_over_the_batch():
    """An illegal commit in the last request leaves every request unchanged
    (validation pass before the apply kernel; engine.py:70-83 checks first)."""
    bs = BatchState(3, 64, qcap=8)
    reqs = make_requests(6, 3, (3, 10), (20, 30), 8, 16, "in_block")
    for r in reqs:
        r.states[:] = 0
        r.uncached_queue.clear()
        r.committed = r.block_index = r.steps_taken = 0
    for i, r in enumerate(reqs):
        bs.bind(r, i)
    bs.states[2, 1] = 1  # request 2 position 1 is already decoded
    L = _lib.load()
    # each request: no kv, window rows (0, 1); all rows commit -> request 2 row 1 is illegal
    cu = _dev(np.array([0, 2, 4, 6], np.int32))
    tok = _dev(np.array([0, 1, 0, 1, 0, 1], np.int32))
    cur = _dev(np.array([0, 2, 4, 6], np.int32))
    rp = _dev(np.array([0, 1, 0, 1, 0, 1], np.int32))
    mask = _dev(np.ones(6, np.uint8))
    D = {k: _dev(getattr(bs, k)) for k in ("states", "queue", "q_head", "q_len", "block_index", "committed",
                                            "steps_taken", "cached_prefix", "out_len")}
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    sl = _dev(np.array([0, 1, 2], np.int32))
    c0 = torch.zeros(3, dtype=torch.int32, device="cuda")
    st = L.optimus_device_apply(
        3, _p(sl), 16, _p(cu), _p(tok), _p(cur), _p(rp), _p(mask),
        _p(D["states"]), D["states"].shape[1], _p(D["queue"]), bs.qcap, _p(D["q_head"]), _p(D["q_len"]),
        _p(D["block_index"]), _p(D["committed"]), _p(D["steps_taken"]), _p(D["cached_prefix"]), _p(D["out_len"]),
        _p(c0), _p(status), torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    assert int(status.item()) != 0
    for k in ("states", "q_head", "q_len", "committed", "steps_taken", "block_index"):
        assert np.array_equal(D[k].cpu().numpy(), getattr(bs, k)), k


@pytest.mark.parametrize("hq,hkv,page,maxq,ke_hi", [(32, 8, 64, 33, 3000), (32, 8, 16, 33, 9000), (64, 8, 16, 33, 800),
                                                    (16, 4, 64, 33, 600), (4, 4, 8, 9, 40000)])
def test_device_work_planner_matches_host_whole_unit_plan(hq, hkv, page, maxq, ke_hi, monkeypatch):
    """optimus_device_attn_plan == optimus_attn_plan's whole-unit placement (incl. the
    255-page cap cuts and their split groups at page 8 / 16 with long contexts)."""
    monkeypatch.setenv("OPTIMUS_PLAN_FORCE", "whole")
    from paper_2605_24832_b200 import ops
    rng = np.random.default_rng(hq * 31 + page + maxq)
    L = _lib.load()
    for _ in range(4):
        n = int(rng.integers(1, 65))
        counts = rng.integers(0, maxq, n)
        cu = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        ke = rng.integers(1, ke_hi, n).astype(np.int32)
        grid = 148
        plan = ops.plan_attention(cu, ke, hq, hkv, grid=grid, min_split_tiles=4, page_size=page)
        mw = 4096
        work = torch.zeros((mw, 8), dtype=torch.int32, device="cuda")
        off = torch.zeros(grid + 1, dtype=torch.int32, device="cuda")
        groups = torch.zeros((1024, 8), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(4, dtype=torch.int32, device="cuda")
        dcu, dke = _dev(cu), _dev(ke)  # keep the device copies alive across the launch
        st = L.optimus_device_attn_plan(n, _p(dcu), _p(dke), hq, hkv, grid, page, 0, _p(work), mw, _p(off),
                                        _p(groups), 1024, _p(cnt), torch.cuda.current_stream().cuda_stream)
        assert st == 0
        torch.cuda.synchronize()
        c = cnt.cpu().tolist()
        assert c[3] == 0 and c[0] == plan.n_work and c[1] == plan.n_groups and c[2] == plan.n_partials
        assert np.array_equal(off.cpu().numpy(), plan.cta_off_host)
        assert np.array_equal(work.cpu().numpy()[: c[0]], plan.work_host)
        assert np.array_equal(groups.cpu().numpy()[: c[1]], plan.groups_host)


@pytest.mark.parametrize("hq,hkv,page,maxq,ke_hi", [(32, 8, 64, 33, 3000), (32, 8, 16, 33, 9000), (64, 8, 16, 33, 800),
                                                    (16, 4, 64, 33, 600), (4, 4, 8, 9, 40000)])
def test_device_work_planner_cut_mode_invariants(hq, hkv, page, maxq, ke_hi):
    """allow_cut = 1: every unit's pieces tile [0, key_end) in key order with
    consecutive partial slots iff cut, groups describe exactly the cut units, the work
    list is in CTA order, and the planned makespan (half-tile costs) never exceeds the
    whole-unit plan's by more than the cut overhead, while a dominant long unit is cut."""
    rng = np.random.default_rng(hq * 7 + page + maxq)
    L = _lib.load()
    G = hq // hkv
    T = 128 // G
    for it in range(5):
        n = int(rng.integers(1, 65))
        counts = rng.integers(0, maxq, n)
        counts[0] = max(int(counts[0]), 1)
        cu = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        ke = rng.integers(1, ke_hi, n).astype(np.int32)
        if it == 0:
            ke[0] = ke_hi * 4  # one dominant request
        grid = 148
        res = {}
        for cut in (0, 1):
            mw, mg = 4096, 1024
            work = torch.zeros((mw, 8), dtype=torch.int32, device="cuda")
            off = torch.zeros(grid + 1, dtype=torch.int32, device="cuda")
            groups = torch.zeros((mg, 8), dtype=torch.int32, device="cuda")
            cnt = torch.zeros(4, dtype=torch.int32, device="cuda")
            dcu, dke = _dev(cu), _dev(ke)
            st = L.optimus_device_attn_plan(n, _p(dcu), _p(dke), hq, hkv, grid, page, cut, _p(work), mw, _p(off),
                                            _p(groups), mg, _p(cnt), torch.cuda.current_stream().cuda_stream)
            assert st == 0
            torch.cuda.synchronize()
            c = cnt.cpu().tolist()
            assert c[3] == 0
            res[cut] = (c, work.cpu().numpy()[: c[0]], off.cpu().numpy(), groups.cpu().numpy()[: c[1]])
        c, w, o, g = res[1]
        assert o[0] == 0 and o[-1] == c[0] and np.all(np.diff(o) >= 0)
        units = {}
        for x, r in enumerate(w):
            cta = int(np.searchsorted(o, x, side="right") - 1)
            units.setdefault((int(r[0]), int(r[1]), int(r[2])), []).append((int(r[4]), int(r[5]), int(r[6]), cta))
        n_units = sum(hkv * ((int(q) + T - 1) // T) for q in counts if q > 0)
        assert len(units) == n_units
        cut_units = 0
        loads = np.zeros(grid)
        for (req, head, tok), pcs in units.items():
            pcs.sort()
            assert pcs[0][0] == 0 and pcs[-1][1] == ke[req]
            assert all(pcs[i][1] == pcs[i + 1][0] for i in range(len(pcs) - 1))
            if len(pcs) > 1:
                cut_units += 1
                slots = [p[2] for p in pcs]
                assert slots == list(range(slots[0], slots[0] + len(pcs)))
            else:
                assert pcs[0][2] == -1
            for a, b, _, cta in pcs:
                loads[cta] += 2 * ((b - a + 63) // 64) + 3 + (3 if len(pcs) > 1 else 0)
        assert cut_units == c[1] and sum(int(x[5]) for x in g) == c[2]
        # makespan vs the whole-unit plan
        c0, w0, o0, _ = res[0]
        loads0 = np.zeros(grid)
        for x, r in enumerate(w0):
            cta = int(np.searchsorted(o0, x, side="right") - 1)
            loads0[cta] += 2 * ((r[5] - r[4] + 63) // 64) + 3 + (3 if r[6] >= 0 else 0)
        assert loads.max() <= loads0.max() + 8
        hard_cap = 255 * page // 64  # tiles per item (the page cap cuts longer units in both modes)
        if it == 0 and (ke[0] + 63) // 64 <= hard_cap and 2 * (ke[0] + 63) // 64 > 1.2 * loads0.mean() + 40:
            assert c[1] > 0 and loads.max() < loads0.max()
