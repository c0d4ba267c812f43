"""The native host planner/applier (csrc/host_step.cu) against the Python mirror
of plan_chunk / build_step_meta / apply_chunk (which tests/golden pin to the
reference), step by step over whole decodes, on CPU."""

import copy

import numpy as np
import pytest

from paper_2605_24832_b200 import _lib
from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.batch_state import BatchState
from paper_2605_24832_b200.meta import build_step_meta
from tests.scenario import make_requests


def _native_plan(bs, slots, chunk, block, rule, tables, caps=4096):
    n = len(slots)
    sl = np.asarray(slots, dtype=np.int32)
    out = {k: np.zeros(n + 1, np.int32) for k in ("cu_seqlens", "vis_off", "cu_rows")}
    out.update({k: np.zeros(n, np.int32) for k in ("prompt_len", "key_end", "vis_base")})
    out.update({k: np.zeros(caps, np.int32) for k in ("tok_req", "tok_pos", "row_tok", "row_pos", "row_req")})
    out["vis_words"] = np.zeros(caps, np.uint32)
    out["block_tables"] = np.zeros((n, tables.shape[1]), np.int32)
    counts = np.zeros(4, np.int32)
    L = _lib.load()
    st = L.optimus_host_plan(
        n, sl.ctypes.data, chunk if np.ndim(chunk) == 0 else 0,
        None if np.ndim(chunk) == 0 else np.ascontiguousarray(chunk, dtype=np.int32).ctypes.data,
        block, 0 if rule == "in_block" else 1,
        bs.states.ctypes.data, bs.states.shape[1], bs.queue.ctypes.data, bs.qcap,
        bs.q_head.ctypes.data, bs.q_len.ctypes.data, bs.block_index.ctypes.data,
        bs.cached_prefix.ctypes.data, bs.prompt.ctypes.data, bs.out_len.ctypes.data,
        tables.ctypes.data, tables.shape[1], out["cu_seqlens"].ctypes.data, out["tok_req"].ctypes.data,
        out["tok_pos"].ctypes.data, caps, out["prompt_len"].ctypes.data, out["key_end"].ctypes.data,
        out["vis_base"].ctypes.data, out["vis_off"].ctypes.data, out["vis_words"].ctypes.data, caps,
        out["cu_rows"].ctypes.data, out["row_tok"].ctypes.data, out["row_pos"].ctypes.data,
        out["row_req"].ctypes.data, caps, out["block_tables"].ctypes.data, counts.ctypes.data)
    assert st == 0
    return out, counts


def _native_apply(bs, slots, block, out, mask):
    n = len(slots)
    sl = np.asarray(slots, dtype=np.int32)
    commits = np.zeros(n, np.int32)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    st = _lib.load().optimus_host_apply(
        n, sl.ctypes.data, block, out["cu_seqlens"].ctypes.data, out["tok_pos"].ctypes.data,
        out["cu_rows"].ctypes.data, out["row_pos"].ctypes.data, m.ctypes.data, bs.states.ctypes.data,
        bs.states.shape[1], bs.queue.ctypes.data, bs.qcap, bs.q_head.ctypes.data, bs.q_len.ctypes.data,
        bs.block_index.ctypes.data, bs.committed.ctypes.data, bs.steps_taken.ctypes.data,
        bs.cached_prefix.ctypes.data, bs.out_len.ctypes.data, commits.ctypes.data)
    assert st == 0
    return commits


@pytest.mark.parametrize("rule,chunk,block", [("in_block", 8, 32), ("in_block", 32, 32), ("out_block", 8, 16),
                                              ("in_block", 2, 8), ("out_block", 16, 8), ("in_block", "mixed", 32)])
def test_native_plan_and_apply_match_python_over_whole_decodes(rule, chunk, block):
    rng = np.random.default_rng(block + (7 if chunk == "mixed" else chunk))
    ref = make_requests(11 + block, 10, (1, 200), (3, 120), 8, block, rule)
    nat = copy.deepcopy(ref)
    bs = BatchState(16, 256, qcap=64)
    for i, r in enumerate(nat):
        bs.bind(r, i)
    tables = np.arange(16 * 40, dtype=np.int32).reshape(16, 40)
    steps = 0
    while not all(r.finished for r in ref):
        idx = [i for i, r in enumerate(ref) if not r.finished]
        batch_ref = [ref[i] for i in idx]
        c = rng.choice([2, 4, 8, 16, 24, 32], len(idx)) if chunk == "mixed" else chunk
        plans = pe.plan_batch(batch_ref, c, block, rule)
        meta = build_step_meta(batch_ref, plans, block, tables[idx])
        out, counts = _native_plan(bs, idx, c, block, rule, tables)
        n_tok, n_rows, n_words = counts[:3]
        assert n_tok == meta.n_tok and n_rows == meta.n_rows
        for k in ("cu_seqlens", "prompt_len", "key_end", "vis_base", "vis_off", "cu_rows"):
            assert np.array_equal(out[k], getattr(meta, k)), k
        for k in ("tok_req", "tok_pos"):
            assert np.array_equal(out[k][:n_tok], getattr(meta, k)), k
        for k in ("row_tok", "row_pos", "row_req"):
            assert np.array_equal(out[k][:n_rows], getattr(meta, k)), k
        assert np.array_equal(out["vis_words"][:n_words], meta.vis_words[:n_words])
        assert np.array_equal(out["block_tables"], meta.block_tables)
        mask = rng.random(n_rows) < 0.3
        for r in range(len(idx)):  # progress rule: first window row commits
            a, b = meta.cu_rows[r], meta.cu_rows[r + 1]
            if b > a:
                mask[a] = True
        commit_sets = [set(meta.row_pos[meta.cu_rows[r]:meta.cu_rows[r + 1]][mask[meta.cu_rows[r]:meta.cu_rows[r + 1]]])
                       for r in range(len(idx))]
        pe.apply_batch(batch_ref, plans, commit_sets, block)
        counts_nat = _native_apply(bs, idx, block, out, mask)
        assert list(counts_nat) == [len(c) for c in commit_sets]
        for i in range(len(ref)):
            a, b = ref[i], nat[i]
            assert np.array_equal(a.states, b.states), (steps, i)
            assert list(a.uncached_queue) == list(b.uncached_queue)
            assert (a.block_index, a.committed, a.steps_taken) == (b.block_index, b.committed, b.steps_taken)
        steps += 1
        assert steps < 500


def test_bound_requests_work_with_reference_functions_and_unbind():
    reqs = make_requests(3, 3, (1, 50), (10, 60), 8, 16, "in_block")
    twin = copy.deepcopy(reqs)
    bs = BatchState(4, 128, qcap=32)
    for i, r in enumerate(reqs):
        bs.bind(r, i)
    for _ in range(5):
        for a, b in zip(reqs, twin):
            if b.finished:
                continue
            pa, pb = pe.plan_chunk(a, 8, 16), pe.plan_chunk(b, 8, 16)
            assert pa == pb
            c = set(pb.window[:2])
            pe.apply_chunk(a, pa, c, 16)
            pe.apply_chunk(b, pb, c, 16)
    for i, r in enumerate(reqs):
        back = bs.unbind(i)
        assert type(back).__name__ == "Request"
        assert np.array_equal(back.states, twin[i].states)
        assert list(back.uncached_queue) == list(twin[i].uncached_queue)
        assert back.committed == twin[i].committed and back.block_index == twin[i].block_index


def test_illegal_commit_leaves_every_request_unchanged():
    """optimus_host_apply validates the whole batch before it changes anything
    (the reference checks commits before mutating, engine.py:70-83): an illegal
    commit in the LAST request leaves the earlier requests' state untouched too."""
    reqs = make_requests(5, 3, (1, 50), (40, 60), 8, 32, "in_block")
    bs = BatchState(4, 128, qcap=32)
    for i, r in enumerate(reqs):
        bs.bind(r, i)
    tables = np.arange(4 * 8, dtype=np.int32).reshape(4, 8)
    idx = [0, 1, 2]
    out, counts = _native_plan(bs, idx, 8, 32, "in_block", tables)
    n_rows = int(counts[1])
    mask = np.ones(n_rows, np.uint8)
    before = {k: getattr(bs, k).copy() for k in ("states", "queue", "q_head", "q_len", "block_index", "committed",
                                                  "steps_taken", "cached_prefix")}
    # corrupt the last request's last row: point it at an already-decoded position
    last = int(out["cu_rows"][3]) - 1
    bs.states[2, 0] = 1
    before["states"][2, 0] = 1
    out["row_pos"][last] = 0
    commits = np.zeros(3, np.int32)
    m = np.ascontiguousarray(mask)
    sl = np.asarray(idx, dtype=np.int32)
    st = _lib.load().optimus_host_apply(
        3, sl.ctypes.data, 32, out["cu_seqlens"].ctypes.data, out["tok_pos"].ctypes.data,
        out["cu_rows"].ctypes.data, out["row_pos"].ctypes.data, m.ctypes.data, bs.states.ctypes.data,
        bs.states.shape[1], bs.queue.ctypes.data, bs.qcap, bs.q_head.ctypes.data, bs.q_len.ctypes.data,
        bs.block_index.ctypes.data, bs.committed.ctypes.data, bs.steps_taken.ctypes.data,
        bs.cached_prefix.ctypes.data, bs.out_len.ctypes.data, commits.ctypes.data)
    assert st != 0
    for k, v in before.items():
        assert np.array_equal(getattr(bs, k), v), k
