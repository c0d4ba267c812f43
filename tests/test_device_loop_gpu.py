"""The graph-captured device loop (device_loop.DeviceLoop: plan, work list, K1/K2,
unmask and apply all on the device) against the host native step
(NativeStepper: host planning, one H2D, device step, one D2H, host apply) on the
same requests and logits: identical Request states and commits, step by step,
through the end of every request."""

import copy

import numpy as np
import pytest
import torch

import bench
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.device_loop import DeviceLoop
from paper_2605_24832_b200.synthetic import SyntheticForward

pytestmark = pytest.mark.gpu


def _setup(seed, batch, chunk, page=64, layers=2, rule="in_block", block=32):
    class A:
        pass
    a = A()
    a.workload, a.chunk, a.page, a.batch, a.seed, a.steps = "sharegpt", chunk, page, batch, seed, 1
    reqs = bench.workload_requests(a)
    cfg = DecodeConfig(num_layers=layers, page_size=page, max_batch=batch, window_rule=rule, block_size=block,
                       num_pages=bench.pages_needed(reqs, page) + 2 * batch + 64,
                       max_pages_per_req=max((r.prompt_tokens + r.output_tokens + page - 1) // page for r in reqs) + 2)
    dev = torch.device("cuda")
    fwd = SyntheticForward(cfg, batch * chunk, batch, device=dev, seed=seed)
    dec = StreamingDecoder(cfg, fwd, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    for l in range(cfg.num_layers):
        dec.cache.k[l].normal_(generator=g)
        dec.cache.v[l].normal_(generator=g)
    return reqs, dec


@pytest.mark.parametrize("batch,chunk,rule,block", [(12, 32, "in_block", 32), (24, 8, "in_block", 32),
                                                    (10, 16, "out_block", 32), (8, 8, "in_block", 16)])
def test_device_loop_matches_host_native_step(batch, chunk, rule, block):
    reqs_h, dec_h = _setup(3, batch, chunk, rule=rule, block=block)
    reqs_d, dec_d = _setup(3, batch, chunk, rule=rule, block=block)
    loop = DeviceLoop(dec_d, reqs_d, chunk)
    steps = 0
    while not all(r.finished for r in reqs_h):
        active = [r for r in reqs_h if not r.finished]
        sh = dec_h.step(active, chunk)
        sd = loop.step()
        by_id = {r.id: s for r, s in zip(active, sh)}
        for r, s in zip(reqs_d, sd):
            if r.id in by_id:
                assert set(s.commits) == set(by_id[r.id].commits), (steps, r.id)
                assert s.computed == by_id[r.id].computed
            else:
                assert s.computed == 0 and not s.commits
        for a, b in zip(reqs_h, reqs_d):
            assert np.array_equal(a.states, b.states), (steps, a.id)
            assert list(a.uncached_queue) == list(b.uncached_queue)
            assert (a.block_index, a.committed, a.steps_taken) == (b.block_index, b.committed, b.steps_taken)
        steps += 1
        assert steps < 5000
    assert loop.finished()
    # the device state ended where the host mirror did
    for k in ("states", "block_index", "committed", "steps_taken"):
        assert np.array_equal(loop.D[k].cpu().numpy(), getattr(loop.bs, k)), k


@pytest.mark.parametrize("lookahead", [False, True])
def test_device_loop_continuous_batching_matches_host(lookahead):
    """DeviceLoop.replace admits a new request into a finished position (same batch
    slot, state and block-table rows copied into the captured graph's inputs); the
    closed loop matches the host native step run with the same admissions.  With
    lookahead the next iteration is already in flight when the host applies one, so
    an admission takes effect one iteration later: the host run admits with that lag."""
    batch, chunk = 10, 16
    reqs_h, dec_h = _setup(4, batch, chunk)
    reqs_d, dec_d = _setup(4, batch, chunk)

    def spares():
        class A:
            pass
        a = A()
        a.workload, a.chunk, a.page, a.batch, a.seed, a.steps = "sharegpt", chunk, 64, 6, 4, 1
        return [r for r in bench.workload_requests(a, seed_offset=5)
                if r.prompt_tokens + r.output_tokens <= dec_h.cfg.max_pages_per_req * 64]

    spare_h, spare_d = spares(), spares()
    assert len(spare_h) >= 3
    loop = DeviceLoop(dec_d, reqs_d, chunk, lookahead=lookahead)
    pos_h = {r.id: i for i, r in enumerate(reqs_h)}  # host: loop position of each live request
    for i, r in enumerate(reqs_h):  # the host batch takes the device loop's slots (logit rows follow slots)
        dec_h.native()._slot(r, int(loop.slots_h[i]))
    live_h = list(reqs_h)
    lagged = []  # host admissions waiting one iteration (lookahead)
    steps = admitted = 0
    while live_h or lagged or not loop.finished():
        sh = dec_h.step(live_h, chunk) if live_h else []
        sd = loop.step()
        by_id = {r.id: s for r, s in zip(live_h, sh)}
        for r, s in zip(loop.requests, sd):
            if r.id in by_id:
                assert set(s.commits) == set(by_id[r.id].commits), (steps, r.id)
                assert s.computed == by_id[r.id].computed, (steps, r.id)
            else:
                assert s.computed == 0 and not s.commits, (steps, r.id)
        for a in live_h:
            b = loop.requests[pos_h[a.id]]
            assert a.id == b.id and np.array_equal(a.states, b.states), (steps, a.id)
            assert (a.block_index, a.committed, a.steps_taken) == (b.block_index, b.committed, b.steps_taken)
        done = sorted(pos_h[r.id] for r in live_h if r.finished)
        live_h = [r for r in live_h if not r.finished]
        for i, nh in lagged:
            dec_h.native()._slot(nh, int(loop.slots_h[i]))
            live_h.append(nh)
        lagged = []
        assert set(done) <= loop.free
        for i in done:  # every finished position takes the next spare, in position order
            if not spare_h:
                break
            nh, nd = spare_h.pop(0), spare_d.pop(0)
            pos_h[nh.id] = i
            loop.replace(i, nd)
            if lookahead:
                lagged.append((i, nh))
            else:
                dec_h.native()._slot(nh, int(loop.slots_h[i]))
                live_h.append(nh)
            admitted += 1
        steps += 1
        assert steps < 5000
    loop.drain()
    assert admitted >= 3


@pytest.mark.parametrize("path", ["host_step", "device_loop"])
def test_recorded_gpu_trace_replays_exactly(path):
    """The B200 path's commit decisions (K3 on the synthetic logits), recorded as a
    CommitTrace in the reference's JSONL format, replay the same decode through
    the CPU engine with the strict ReplayOracle: identical windows and commits per
    step, identical final states."""
    from paper_2605_24832_b200 import engine as pe
    from paper_2605_24832_b200.core import Request
    from dllmsim.commit import CommitTrace, ReplayOracle

    from paper_2605_24832_b200.trace import TraceRecorder

    batch, chunk = 8, 16
    staged, dec = _setup(6, batch, chunk)
    block = dec.cfg.block_size
    fresh = lambda: [Request(id=r.id, arrival_time=0.0, prompt_tokens=r.prompt_tokens,
                             output_tokens=min(r.output_tokens, 300)) for r in staged]
    reqs = fresh()
    rec = TraceRecorder()
    loop = DeviceLoop(dec, reqs, chunk) if path == "device_loop" else None
    gpu_steps = {r.id: [] for r in reqs}
    n = 0
    while not all(r.finished for r in reqs):
        active = list(reqs) if loop is not None else [r for r in reqs if not r.finished]
        rec.before(active)
        summ = loop.step() if loop is not None else dec.step(active, chunk)
        rec.after(active, summ)
        for r, s in zip(active, summ):
            if s.computed:
                gpu_steps[r.id].append(sorted(s.commits))
        n += 1
        assert n < 5000
    text = rec.trace.to_jsonl()
    trace = CommitTrace.from_jsonl(text)
    trace.validate({r.id: r.output_tokens for r in reqs})
    ro = ReplayOracle(trace, carryover=False)
    for orig, r in zip(reqs, fresh()):
        replayed = []
        while not r.finished:
            plan = pe.plan_chunk(r, chunk, block, "in_block")
            commits = ro.commits(r, list(plan.window)) if plan.window else set()
            pe.apply_chunk(r, plan, commits, block)
            replayed.append(sorted(commits))
        assert replayed == gpu_steps[r.id], r.id
        assert np.array_equal(r.states, orig.states) and r.steps_taken == orig.steps_taken


def test_device_loop_mixed_chunks_matches_host():
    """Per-position chunk sizes (the elastic scheduler's per-request chunks, BASELINE
    configs[3]): the device plan reads them from device memory; same decode as the
    host native step given the same per-request chunks."""
    batch = 12
    rng = np.random.default_rng(9)
    chunks = [int(c) for c in rng.choice([8, 16, 24, 32], batch)]
    reqs_h, dec_h = _setup(7, batch, 32)
    reqs_d, dec_d = _setup(7, batch, 32)
    loop = DeviceLoop(dec_d, reqs_d, chunks)
    chunk_of = {r.id: c for r, c in zip(reqs_h, chunks)}
    for i, r in enumerate(reqs_h):
        dec_h.native()._slot(r, int(loop.slots_h[i]))
    steps = 0
    while not all(r.finished for r in reqs_h):
        active = [r for r in reqs_h if not r.finished]
        sh = dec_h.step(active, [chunk_of[r.id] for r in active])
        sd = loop.step()
        by_id = {r.id: s for r, s in zip(active, sh)}
        for r, s in zip(reqs_d, sd):
            if r.id in by_id:
                assert set(s.commits) == set(by_id[r.id].commits), (steps, r.id)
                assert s.computed == by_id[r.id].computed
        for a, b in zip(reqs_h, reqs_d):
            assert np.array_equal(a.states, b.states), (steps, a.id)
        steps += 1
        assert steps < 5000


def test_device_loop_elastic_chunk_matches_host():
    """ElasticChunk on the device loop: every iteration the reference's scheduler
    (dllmsim.scheduler.select_chunk over a CommitEstimator fed with each step's windows
    and commits, sim.py:219-232,270-293) picks the chunk for the batch, and
    DeviceLoop.step(chunk=c) runs it from the same captured graph.  Same decode as the
    host native step given the same chunk sequence, and the estimator fed from the
    loop's own window observations stays equal to the host one.  (The calibrated B200
    cost model makes select_chunk pick the largest candidate at this batch; a steeper
    model makes the chunk move, which is what this exercises.)"""
    sched = pytest.importorskip("dllmsim.scheduler")
    costmodel = pytest.importorskip("dllmsim.costmodel")
    from paper_2605_24832_b200 import engine as pe

    Seg = costmodel.Segment
    cost = costmodel.CostModel((Seg(0, 2e-6, 2e-4), Seg(64, 4e-6, 2e-4 + 64 * 2e-6),
                                Seg(256, 8e-6, 2e-4 + 64 * 2e-6 + 192 * 4e-6)))
    batch, block = 12, 32
    reqs_h, dec_h = _setup(11, batch, 32)
    reqs_d, dec_d = _setup(11, batch, 32)
    loop = DeviceLoop(dec_d, reqs_d, 32, max_chunk=32)
    for i, r in enumerate(reqs_h):
        dec_h.native()._slot(r, int(loop.slots_h[i]))
    mk = lambda: sched.CommitEstimator(window_size=block, alpha=0.95, prior_q=0.8, min_observations=8)
    est_h, est_d = mk(), mk()
    prev, seq, steps = None, [], 0
    while not all(r.finished for r in reqs_h):
        active = [r for r in reqs_h if not r.finished]
        c = 32 if est_h.observations < 32 else sched.select_chunk(est_h, cost, len(active),
                                                                 tuple(range(2, 33, 2)), prev, 0.05)
        prev = c
        seq.append(c)
        windows = [pe.plan_chunk(r, c, block, "in_block").window for r in active]
        sh = dec_h.step(active, c)
        sd = loop.step(chunk=c)
        by_id = {r.id: s for r, s in zip(active, sh)}
        for r, s in zip(reqs_d, sd):
            if r.id in by_id:
                assert set(s.commits) == set(by_id[r.id].commits), (steps, r.id, c)
                assert s.computed == by_id[r.id].computed
            else:
                assert s.computed == 0 and not s.commits
        for a, b in zip(reqs_h, reqs_d):
            assert np.array_equal(a.states, b.states), (steps, a.id)
        for w, s in zip(windows, sh):
            if w:
                rank = {p: i for i, p in enumerate(w)}
                est_h.observe(len(w), {rank[p] for p in s.commits})
        for n_w, ranks in loop.window_observations():
            est_d.observe(n_w, ranks)
        assert est_d.observations == est_h.observations and np.array_equal(est_d.hist, est_h.hist)
        steps += 1
        assert steps < 5000
    assert len(set(seq)) >= 3, seq  # the chunk really changed between iterations


def test_graph_captured_host_step_matches_eager(monkeypatch):
    """NativeStepper.device_step_graph (the host-planned step replayed as one CUDA
    graph, counts read on the device) == the eager step, commit for commit."""
    batch, chunk = 12, 16
    reqs_e, dec_e = _setup(8, batch, chunk)
    reqs_g, dec_g = _setup(8, batch, chunk)
    dec_g.append_mode = "k1"  # the graph-captured host step runs the k1 form of K1
    steps = 0
    while not all(r.finished for r in reqs_e):
        ae = [r for r in reqs_e if not r.finished]
        ag = [r for r in reqs_g if not r.finished]
        monkeypatch.setenv("OPTIMUS_STEP_GRAPH", "0")
        se = dec_e.step(ae, chunk)
        monkeypatch.setenv("OPTIMUS_STEP_GRAPH", "1")
        sg = dec_g.step(ag, chunk)
        assert [set(s.commits) for s in se] == [set(s.commits) for s in sg], steps
        for a, b in zip(reqs_e, reqs_g):
            assert np.array_equal(a.states, b.states), (steps, a.id)
        steps += 1
        assert steps < 5000
    assert dec_g.native()._graphs  # the graph path ran


def test_device_loop_rejects_what_the_device_planners_cannot_run():
    """Limits of csrc/device_step.cu are checked before capture (chunk <= 128,
    out_len <= 4096 / the packed state's capacity, <= 256 requests)."""
    from paper_2605_24832_b200.core import Request
    from paper_2605_24832_b200.errors import ConfigError

    reqs, dec = _setup(4, 4, 8)
    with pytest.raises(ConfigError):
        DeviceLoop(dec, reqs, 130)
    big = Request(id=999, arrival_time=0.0, prompt_tokens=10, output_tokens=5000)
    with pytest.raises(ConfigError):
        DeviceLoop(dec, reqs[:3] + [big], 8)


@pytest.mark.parametrize("backend", ["loop", "loop_lookahead"])
def test_streaming_decoder_step_on_the_device_loop(backend):
    """StreamingDecoder.step with DecodeConfig.step_backend = "loop" runs the
    graph-captured DeviceLoop behind the same per-step call: a closed loop that drops
    finished requests and brings new ones into the batch gives exactly the host
    step's commits and states (new requests take the freed positions' batch slots, so
    the host run admits them into the same slots).  With "loop_lookahead" the next
    iteration is already in flight when step() returns, so an admission takes effect
    one call later: the host run admits with that lag."""
    import dataclasses
    batch, chunk = 10, 16
    reqs_h, dec_h = _setup(12, batch, chunk)
    reqs_d, dec_d = _setup(12, batch, chunk)
    dec_d.cfg = dataclasses.replace(dec_d.cfg, step_backend=backend)
    look = backend == "loop_lookahead"

    def spares():
        class A:
            pass
        a = A()
        a.workload, a.chunk, a.page, a.batch, a.seed, a.steps = "sharegpt", chunk, 64, 6, 12, 1
        return [r for r in bench.workload_requests(a, seed_offset=9)
                if r.prompt_tokens + r.output_tokens <= dec_h.cfg.max_pages_per_req * 64]

    spare_h, spare_d = spares(), spares()
    live_h, live_d = list(reqs_h), list(reqs_d)
    sd = dec_d.step(live_d, chunk)  # builds the loop: its positions take the batch slots
    L = dec_d._loop
    for i, r in enumerate(reqs_h):
        dec_h.native()._slot(r, int(L.slots_h[i]))
    sh = dec_h.step(live_h, chunk)
    lagged, steps, admitted = [], 0, 0
    while True:
        by_id = {r.id: s for r, s in zip(live_h, sh)}
        for r, s in zip(live_d, sd):
            if r.id in by_id:
                assert set(s.commits) == set(by_id[r.id].commits), (steps, r.id)
                assert s.computed == by_id[r.id].computed, (steps, r.id)
            else:
                assert s.computed == 0 and not s.commits, (steps, r.id)
        for a in live_h:
            b = next(x for x in live_d if x.id == a.id)
            assert np.array_equal(a.states, b.states), (steps, a.id)
        live_h = [r for r in live_h if not r.finished]
        done_d = [r for r in live_d if r.finished]
        live_d = [r for r in live_d if not r.finished]
        for nh in lagged:
            live_h.append(nh)
        lagged = []
        for r in done_d:  # every finished request is replaced by the next spare
            if not spare_d:
                break
            nh, nd = spare_h.pop(0), spare_d.pop(0)
            slot = int(L.slots_h[[x.id for x in L.requests].index(r.id)])
            live_d.append(nd)
            dec_h.native()._slot(nh, slot)
            (lagged if look else live_h).append(nh)
            admitted += 1
        if not live_d and not live_h and not lagged:
            break
        sd = dec_d.step(live_d, chunk)
        sh = dec_h.step(live_h, chunk) if live_h else []
        steps += 1
        assert steps < 5000
    dec_d.release_all([])
    assert admitted >= 3


def test_streaming_decoder_loop_backend_mixed_chunks():
    """The loop backend takes the per-request chunk list of the mixed-chunk workload
    (BASELINE configs[3]) through the same StreamingDecoder.step call: each request's
    chunk lands at its loop position; same decode as the host backend."""
    import dataclasses
    batch = 12
    rng = np.random.default_rng(21)
    reqs_h, dec_h = _setup(21, batch, 32)
    reqs_d, dec_d = _setup(21, batch, 32)
    dec_d.cfg = dataclasses.replace(dec_d.cfg, step_backend="loop")
    chunk_of = {r.id: int(c) for r, c in zip(reqs_h, rng.choice([8, 16, 24, 32], batch))}
    # both paths decode in reverse order, so list order != loop position order
    live_d = list(reversed(reqs_d))
    sd = dec_d.step(live_d, [chunk_of[r.id] for r in live_d])
    L = dec_d._loop
    for r in reqs_h:
        dec_h.native()._slot(r, int(L.slots_h[[x.id for x in L.requests].index(r.id)]))
    live_h = list(reversed(reqs_h))
    sh = dec_h.step(live_h, [chunk_of[r.id] for r in live_h])
    steps = 0
    while True:
        assert [set(s.commits) for s in sd] == [set(s.commits) for s in sh], steps
        assert [s.computed for s in sd] == [s.computed for s in sh], steps
        for a, b in zip(live_h, live_d):
            assert a.id == b.id and np.array_equal(a.states, b.states), (steps, a.id)
        live_h = [r for r in live_h if not r.finished]
        live_d = [r for r in live_d if not r.finished]
        if not live_d:
            break
        sd = dec_d.step(live_d, [chunk_of[r.id] for r in live_d])
        sh = dec_h.step(live_h, [chunk_of[r.id] for r in live_h])
        steps += 1
        assert steps < 5000
    assert not live_h
    dec_d.release_all([])


@pytest.mark.gpu
def test_device_admit_writes_the_slot_rows():
    """optimus_device_admit (DeviceLoop.replace + flush_admissions): after admitting
    requests into finished positions, every field of their batch slots in the device
    state (scalars, state row, FIFO ring, block-table row) equals the host's packed rows,
    and the other slots are untouched."""
    batch, chunk = 6, 16
    reqs, dec = _setup(11, batch, chunk)
    loop = DeviceLoop(dec, reqs, chunk)
    while not any(r.finished for r in loop.requests):
        loop.step()
    free = sorted(loop.free)
    assert free

    class A:
        pass
    a = A()
    a.workload, a.chunk, a.page, a.batch, a.seed, a.steps = "sharegpt", chunk, 64, 8, 7, 1
    cand = [r for r in bench.workload_requests(a, seed_offset=9)
            if r.prompt_tokens + r.output_tokens <= dec.cfg.max_pages_per_req * 64]
    before = {k: v.clone() for k, v in loop.D.items()}
    tbl_before = loop.Dt.clone()
    admitted = []
    for i, r in zip(free, cand):
        loop.replace(i, r)
        admitted.append(int(loop.slots_h[i]))
    loop.flush_admissions()
    torch.cuda.synchronize()
    bs = loop.bs
    for k in loop.state_keys:
        dev = loop.D[k].cpu().numpy()
        host = getattr(bs, k)
        for s in admitted:
            assert np.array_equal(dev[s], host[s]), (k, s)
        others = [s for s in range(dev.shape[0]) if s not in admitted]
        assert np.array_equal(dev[others], before[k].cpu().numpy()[others]), k
    tbl = loop.Dt.cpu().numpy()
    for s in admitted:
        assert np.array_equal(tbl[s], dec.tables.table[s])
    others = [s for s in range(tbl.shape[0]) if s not in admitted]
    assert np.array_equal(tbl[others], tbl_before.cpu().numpy()[others])
