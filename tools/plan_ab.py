"""Interleaved A/B of the attention planner's candidates on rank 0's KV-head shard
(diagnostics): whole units, LPT cutting, flat stream.

    python tools/plan_ab.py --workload ctx4096 --tps 1,2,4,8 [--layers 36]

Per (tp, plan): a CUDA graph of L back-to-back K2 launches (+ the split-KV combine),
replayed in interleaved rounds; µs per layer and HBM fraction of the algorithmic bytes.
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24832_b200 import ops  # noqa: E402
from paper_2605_24832_b200.engine import plan_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ctx4096")
ap.add_argument("--tps", default="1,2,4,8")
ap.add_argument("--plans", default="auto,whole,cut,flat")
ap.add_argument("--layers", type=int, default=36)
ap.add_argument("--rounds", type=int, default=10)
ap.add_argument("--seed-offset", type=int, default=0, help="another batch of the workload (bench: 0)")
a = ap.parse_args()
a.page, a.seed, a.steps, a.chunk = 64, 0, 1, 32
a.batch = 128 if a.workload == "llada" else 64
dev = torch.device("cuda")
hbm, _ = bench.peaks()
for tp in [int(t) for t in a.tps.split(",")]:
    W = bench.build_decoder(a, dev, world=tp, rank=0, layers=a.layers, e2e_pools=False,
                            reqs=bench.workload_requests(a, seed_offset=a.seed_offset) if a.seed_offset else None)
    dec, fwd, cfg = W.dec, W.fwd, W.cfg
    plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), cfg.block_size, cfg.window_rule)
    dm = dec.prepare(W.reqs, plans)
    m = dm.host
    k2b = bench.algorithmic_bytes(dm, cfg)[0]
    graphs = {}
    for force in a.plans.split(","):
        if force == "auto":
            os.environ.pop("OPTIMUS_PLAN_FORCE", None)
        else:
            os.environ["OPTIMUS_PLAN_FORCE"] = force
        plan = ops.plan_attention(m.cu_seqlens, m.key_end, cfg.num_q_heads, cfg.num_kv_heads, grid=dec.grid,
                                  min_split_tiles=cfg.min_split_tiles, device=dev, page_size=cfg.page_size)
        os.environ.pop("OPTIMUS_PLAN_FORCE", None)
        out = torch.empty((m.n_tok, cfg.num_q_heads, cfg.head_dim), dtype=torch.bfloat16, device=dev)
        ws_o = torch.empty(max(plan.n_partials, 1) * 128 * cfg.head_dim, dtype=torch.float32, device=dev)
        ws_ml = torch.empty(max(plan.n_partials, 1) * 256, dtype=torch.float32, device=dev)

        def k2(l, plan=plan, out=out, ws_o=ws_o, ws_ml=ws_ml):
            q, _, _ = fwd.qkv(l, dm)
            kc, vc = dec.cache.layer(l)
            ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off, dm.vis_words,
                                dm.block_tables, plan, cfg.block_size, out=out, ws_o=ws_o, ws_ml=ws_ml)
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
        graphs[force] = (g, plan, out, ws_o, ws_ml)
    res = {k: [] for k in graphs}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(a.rounds):
        for k, (g, *_) in graphs.items():
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3 / cfg.num_layers)
    for k, (g, plan, *_) in graphs.items():
        us = float(np.median(res[k][2:]))
        print(f"{a.workload:9s} tp{tp} {k:6s} work {plan.n_work:4d} groups {plan.n_groups:4d}  {us:7.2f} us/layer "
              f"{k2b / (us * 1e-6) / 1e9 / hbm:.3f} of HBM", flush=True)
    W = graphs = None
    bench.free()
