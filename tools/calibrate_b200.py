"""Measure this path's device step latency on a B200 over a grid of batch sizes and
chunk sizes (SDAR-8B attention shape, ShareGPT-like lengths, 36 layers + unmask) and
fit the reference's cost model to it.

    python tools/calibrate_b200.py [--out profiles/b200]

Writes <out>_step_profile.csv (the reference's ``x,latency_ms`` profile format:
x = computed tokens of the step = sum of |kv_positions| + |window| over the batch,
as charged at sim.py:293) and <out>_cost_model.json (CostModel JSON; load with
``dllmsim.costmodel.CostModel.from_json`` or pass the CSV to ``dllmsim calibrate``).
"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2605_24832_b200  # noqa: F401  (puts baseline/_ref on sys.path)
from dllmsim.costmodel import fit, profile_to_csv
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.engine import plan_batch
from paper_2605_24832_b200.synthetic import SyntheticForward

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="profiles/b200")
ap.add_argument("--batches", default="1,2,4,8,16,24,32,48,64,96,128")
ap.add_argument("--chunks", default="2,4,8,16,32")
ap.add_argument("--page", type=int, default=64)
a = ap.parse_args()
dev = torch.device("cuda")
batches = [int(b) for b in a.batches.split(",")]
chunks = [int(c) for c in a.chunks.split(",")]


class Args:
    pass


P = a.page
bmax = max(batches)
ar = Args()
ar.workload, ar.chunk, ar.page, ar.batch, ar.seed, ar.steps = "sharegpt", 32, P, bmax, 0, 1
pool = bench.workload_requests(ar)
cfg = DecodeConfig(page_size=P, max_batch=bmax, num_pages=bench.pages_needed(pool, P) + 64,
                   max_pages_per_req=max((r.prompt_tokens + r.output_tokens + P - 1) // P for r in pool) + 1)
fwd = SyntheticForward(cfg, bmax * max(chunks), bmax, device=dev)
dec = StreamingDecoder(cfg, fwd, device=dev)
g = torch.Generator(device=dev)
g.manual_seed(7)
for l in range(cfg.num_layers):
    dec.cache.k[l].normal_(generator=g)
    dec.cache.v[l].normal_(generator=g)
samples = []
t0 = time.time()
for b in batches:
    for c in chunks:
        reqs = pool[:b]
        plans = plan_batch(reqs, c, cfg.block_size, cfg.window_rule)
        dm = dec.prepare(reqs, plans)
        x = int(dm.host.n_tok)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            dec.device_step(dm)
            s.synchronize()
            with torch.cuda.graph(gr, stream=s):
                dec.device_step(dm)
        torch.cuda.synchronize()
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        lat = float(np.median(ts))
        samples.append((float(x), lat))
        print(f"batch {b:4d} chunk {c:3d}: x = {x:5d} computed tokens, step {lat * 1e3:8.3f} ms", flush=True)
        del gr
print(f"{len(samples)} samples in {time.time() - t0:.0f} s")
model = fit(samples)
Path(a.out + "_step_profile.csv").write_text(profile_to_csv(samples))
Path(a.out + "_cost_model.json").write_text(model.to_json())
print(model.to_json())
