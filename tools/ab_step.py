"""Interleaved A/B of the full device step under different decoder knobs (diagnostics).

usage: python tools/ab_step.py --workload sharegpt --modes slots,fused,k1
Each mode's step is captured as one CUDA graph; rounds replay the graphs in turn so
clock drift under the power cap hits every mode alike.
"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.engine import plan_batch
from paper_2605_24832_b200.synthetic import SyntheticForward

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--chunk", type=int, default=32)
ap.add_argument("--page", type=int, default=64)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--modes", default="slots,fused,k1")
ap.add_argument("--rounds", type=int, default=15)
a = ap.parse_args()
a.steps = 1
dev = torch.device("cuda")
reqs = bench.workload_requests(a)
P = a.page
cfg = DecodeConfig(page_size=P, max_batch=a.batch, num_pages=bench.pages_needed(reqs, P) + 64,
                   max_pages_per_req=max((r.prompt_tokens + r.output_tokens + P - 1) // P for r in reqs) + 1)
fwd = SyntheticForward(cfg, a.batch * a.chunk, a.batch, device=dev)
dec = StreamingDecoder(cfg, fwd, device=dev)
for l in range(cfg.num_layers):
    dec.cache.k[l].normal_(); dec.cache.v[l].normal_()
dm = dec.prepare(reqs, plan_batch(reqs, a.chunk, cfg.block_size, cfg.window_rule))
graphs = {}
dms = []
import os
for mode in a.modes.split(","):
    # "k1@43": append mode k1 with OPTIMUS_K2_RINGS=43 (K2 variant chosen at capture);
    # "slots:OPTIMUS_PLAN_KITEM=2.0": any environment knob, set while this mode is planned
    # and captured
    mode_, _, kv = mode.partition(":")
    for k in [k for k in os.environ if k.startswith("OPTIMUS_PLAN_")]:
        os.environ.pop(k)
    if kv:
        k, _, v = kv.partition("=")
        os.environ[k] = v
    am, _, rings = mode_.partition("@")
    if rings:
        os.environ["OPTIMUS_K2_RINGS"] = rings
    else:
        os.environ.pop("OPTIMUS_K2_RINGS", None)
    dec.append_mode = am
    dm = dec.prepare(reqs, plan_batch(reqs, a.chunk, cfg.block_size, cfg.window_rule))
    dms.append(dm)  # the graph reads its buffers
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        dec.device_step(dm); s.synchronize()
        with torch.cuda.graph(g, stream=s):
            dec.device_step(dm)
    torch.cuda.synchronize()
    graphs[mode] = g
res = {m: [] for m in graphs}
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for r in range(a.rounds):
    for m, g in graphs.items():
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        res[m].append(e0.elapsed_time(e1) * 1e3)
for m, v in res.items():
    v = np.array(v[3:])
    print(f"{a.workload:10s} {m:8s} step us median {np.median(v):8.1f}  min {v.min():8.1f}")
