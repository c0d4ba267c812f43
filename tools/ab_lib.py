"""Same-process A/B of K2 between two builds of the C-ABI library (clocks drift with
the power cap between processes; interleaved replays inside one process do not).

    python tools/ab_lib.py tools/_bin/lib_<sha>.so [--workload sharegpt] [--layers 8]

Variant A = the given library, B = the working tree's build.  Each variant plans
with its own library and replays its own CUDA graph of L back-to-back K2 launches.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24832_b200 import _lib, ops  # noqa: E402
from paper_2605_24832_b200.engine import plan_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib_a")
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--chunk", type=int, default=32)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--tp", type=int, default=1, help="rank 0's KV-head shard of tp ranks")
ap.add_argument("--rounds", type=int, default=12)
ap.add_argument("--step", action="store_true", help="also A/B the whole device step (L x (K1, K2) + K3)")
a = ap.parse_args()
a.page, a.seed, a.steps = 64, 0, 1
a.batch = a.batch or (128 if a.workload == "llada" else 64)
dev = torch.device("cuda")
lib_b = _lib.load()
lib_a = _lib.load(a.lib_a)
W = bench.build_decoder(a, dev, world=a.tp, rank=0, layers=a.layers, e2e_pools=False)
dec, fwd, cfg = W.dec, W.fwd, W.cfg
plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), cfg.block_size, cfg.window_rule)
dm = dec.prepare(W.reqs, plans)
m = dm.host
k2b = bench.algorithmic_bytes(dm, cfg)[0]
graphs = {}
steps = {}
for name, lib in (("A", lib_a), ("B", lib_b)):
    _lib._LIB = lib
    plan = ops.plan_attention(m.cu_seqlens, m.key_end, cfg.num_q_heads, cfg.num_kv_heads, grid=dec.grid,
                              min_split_tiles=cfg.min_split_tiles, device=dev, page_size=cfg.page_size)
    out = dec._workspaces(plan, m.n_tok)
    if plan.n_partials:
        dec._ws_o = torch.empty(plan.n_partials * 128 * cfg.head_dim, dtype=torch.float32, device=dev)
        dec._ws_ml = torch.empty(plan.n_partials * 256, dtype=torch.float32, device=dev)
    ws_o, ws_ml = dec._ws_o, dec._ws_ml

    def k2(l, plan=plan, out=out, ws_o=ws_o, ws_ml=ws_ml):
        q, k, v = fwd.qkv(l, dm)
        kc, vc = dec.cache.layer(l)
        ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off, dm.vis_words,
                            dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok], ws_o=ws_o, ws_ml=ws_ml)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        k2(0)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for l in range(cfg.num_layers):
                k2(l)
    torch.cuda.synchronize()
    ref = out[: m.n_tok].clone()
    graphs[name] = (g, plan, ref)
    if a.step:
        gs = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            dec.device_step(dm)
            s.synchronize()
            with torch.cuda.graph(gs, stream=s):
                dec.device_step(dm)
        torch.cuda.synchronize()
        steps[name] = gs
    print(f"{name}: work {plan.n_work} groups {plan.n_groups}", flush=True)
_lib._LIB = lib_b
d = (graphs["A"][2].float() - graphs["B"][2].float()).norm() / graphs["A"][2].float().norm()
print(f"outputs A vs B (last layer of the capture run): rel diff {d.item():.2e}")
res = {k: [] for k in graphs}
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
for _ in range(a.rounds):
    for name, (g, _, _) in graphs.items():
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) * 1e3 / cfg.num_layers)
st = {k: [] for k in steps}
for _ in range(a.rounds):
    for name, g in steps.items():
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        st[name].append(e0.elapsed_time(e1) * 1e3)
for name, v in st.items():
    v = np.array(v[2:])
    print(f"{name}: whole step us median {np.median(v):8.1f} min {v.min():8.1f}")
hbm, _ = bench.peaks()
for name, v in res.items():
    v = np.array(v[2:])
    med = float(np.median(v))
    print(f"{name}: K2 us/launch median {med:7.2f} min {v.min():7.2f}  -> {k2b / (med * 1e-6) / 1e9:7.0f} GB/s "
          f"({k2b / (med * 1e-6) / 1e9 / hbm:.3f} of HBM)")
