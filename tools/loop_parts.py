"""GPU time of the DeviceLoop iteration graph and of its parts (diagnostics): the whole
graph, the same graph captured without the per-layer split-KV combine launches (valid
only when the device plan has no split groups), and the two device planners timed
alone (they are pure: replayed back to back on the loop's live state).

    python tools/loop_parts.py [--workload sharegpt]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24832_b200 import _lib  # noqa: E402
from paper_2605_24832_b200.device_loop import DeviceLoop  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--seeds", default="1")
ap.add_argument("--ab-cut", action="store_true",
                help="only A/B the device planner's cutting (allow_cut 1 vs 0), interleaved, per seed")
a = ap.parse_args()
a.page, a.seed, a.steps, a.chunk = 64, 0, 1, 32
a.batch = 128 if a.workload == "llada" else 64
dev = torch.device("cuda")


def graph_us(g, reps=8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts[2:])


def make_loop(skip=(), seed=1, allow_cut=1):
    W = bench.build_decoder(a, dev, e2e_pools=False, reqs=bench.workload_requests(a, seed_offset=seed))
    real = _lib.call

    def call(name, *args):
        if name == "optimus_device_attn_plan":
            args = args[:7] + (allow_cut,) + args[8:]
        return 0 if name in skip else real(name, *args)
    _lib.call = call
    try:
        L = DeviceLoop(W.dec, W.reqs, 32)
        L.capture()
    finally:
        _lib.call = real
    return L


if a.ab_cut:
    for seed in [int(x) for x in a.seeds.split(",")]:
        Ls = {c: make_loop(seed=seed, allow_cut=c) for c in (1, 0)}
        for L in Ls.values():
            for _ in range(2):
                L.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = {c: [] for c in Ls}
        for rnd in range(8):
            for c, L in Ls.items():
                e0.record(); L.graphs[0].replay(); e1.record(); torch.cuda.synchronize()
                ts[c].append(e0.elapsed_time(e1) * 1e3)
        g = {c: int(L.Hs[0]["wcounts"][1]) for c, L in Ls.items()}
        print(f"{a.workload} seed {seed}: allow_cut=1 {np.median(ts[1][2:]):8.1f} us (groups {g[1]})   "
              f"allow_cut=0 {np.median(ts[0][2:]):8.1f} us (groups {g[0]})")
        del Ls
    sys.exit(0)
res = {}
for label, skip in (("graph", ()), ("graph without combine launches", ("optimus_paged_attn_combine_dev",))):
    L = make_loop(skip)
    for _ in range(2):
        L.step()
    torch.cuda.synchronize()
    groups = int(L.Hs[0]["wcounts"][1]) if hasattr(L, "Hs") else -1
    res[label] = graph_us(L.graphs[0])
    print(f"{label:34s} {res[label]:8.1f} us  (split groups {groups})")

# the planners alone, back to back on the last loop's state (pure functions)
cfg, D, M, n = L.cfg, L.D, L.M, L.n
ct, cr, cw = L.caps
p = lambda t: t.data_ptr()
rule = 0


def plan():
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.call(
        "optimus_device_plan", n, p(L.slots), L.chunk, p(L.chunks_d), cfg.block_size, rule, p(D["states"]),
        D["states"].shape[1], p(D["queue"]), L.bs.qcap, p(D["q_head"]), p(D["q_len"]), p(D["block_index"]),
        p(D["cached_prefix"]), p(D["prompt"]), p(D["out_len"]), p(L.Dt), L.Dt.shape[1],
        p(M["cu_seqlens"]), p(M["tok_req"]), p(M["tok_pos"]), ct, p(M["prompt_len"]), p(M["key_end"]),
        p(M["vis_base"]), p(M["vis_off"]), p(M["vis_words"]), cw, p(M["cu_rows"]), p(M["row_tok"]),
        p(M["row_pos"]), p(M["row_req"]), cr, p(M["block_tables"]), p(M["counts"]), s), "device_plan")


def wplan():
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.call(
        "optimus_device_attn_plan", n, p(M["cu_seqlens"]), p(M["key_end"]), cfg.num_q_heads, cfg.num_kv_heads,
        L.grid, cfg.page_size, 1, p(M["work"]), L.max_work, p(M["cta_off"]), p(M["groups"]),
        M["groups"].shape[0], p(M["wcounts"]), s), "device_attn_plan")


for label, fn in (("optimus_device_plan", plan), ("optimus_device_attn_plan", wplan)):
    g = torch.cuda.CUDAGraph()
    fn(); torch.cuda.synchronize()
    with torch.cuda.graph(g):  # (captures on its own stream: current_stream() inside)
        for _ in range(10):
            fn()
    print(f"{label:34s} {graph_us(g) / 10:8.1f} us per launch (10 in one graph)")
# apply mutates the state: time (restore + apply) minus (restore) graphs
snap = {k: v.clone() for k, v in D.items()}


def restore():
    for k, v in snap.items():
        D[k].copy_(v)


def apply():
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.call(
        "optimus_device_apply", n, p(L.slots), cfg.block_size, p(M["cu_seqlens"]), p(M["tok_pos"]),
        p(M["cu_rows"]), p(M["row_pos"]), p(L.res.commit_mask), p(D["states"]), D["states"].shape[1],
        p(D["queue"]), L.bs.qcap, p(D["q_head"]), p(D["q_len"]), p(D["block_index"]), p(D["committed"]),
        p(D["steps_taken"]), p(D["cached_prefix"]), p(D["out_len"]), p(M["commits"]), p(M["counts"][3:]),
        s), "device_apply")


gs = {}
for label, fns in (("restore", (restore,)), ("restore+apply", (restore, apply))):
    g = torch.cuda.CUDAGraph()
    for f in fns:
        f()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(10):
            for f in fns:
                f()
    gs[label] = graph_us(g) / 10
restore()
print(f"{'optimus_device_apply':34s} {gs['restore+apply'] - gs['restore']:8.1f} us per launch pair (validate + apply)")
print(f"n_tok {int(M['counts'][0])} rows {int(M['counts'][1])} work {int(M['wcounts'][0])}")
