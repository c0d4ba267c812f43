"""K3 (unmask partials + finalize) over window-row counts: time and HBM fraction.

    python tools/k3_sweep.py [--vocab 151936] [--lo 500 --hi 2100 --step 50] [--out profiles/...json]

Logits are bf16 [rows, vocab] (> L2 from ~400 rows at 151,936); every point is a CUDA
graph of 8 back-to-back K3s (partials + finalize), median of interleaved replays.  Algorithmic bytes:
rows x vocab x 2 B (logits read once) + 9 B per row (token, confidence, mask).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24832_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--lo", type=int, default=500)
ap.add_argument("--hi", type=int, default=2100)
ap.add_argument("--step", type=int, default=50)
ap.add_argument("--reqs", type=int, default=64)
ap.add_argument("--out", default="")
ap.add_argument("--splits", default="", help="comma list: time these vocab split counts too (default: the chooser's)")
ap.add_argument("--lib", default="", help="time another build of the C-ABI library (tools/build_variant.py)")
a = ap.parse_args()
if a.lib:
    from paper_2605_24832_b200 import _lib
    _lib.load()
    _lib._LIB = _lib.load(a.lib)
dev = torch.device("cuda")
REPS = 8
hbm, _ = bench.peaks()
V = a.vocab
x = torch.randn((a.hi, V), device=dev).to(torch.bfloat16)
points = []
for rows in range(a.lo, a.hi + 1, a.step):
    cu = torch.linspace(0, rows, a.reqs + 1, device=dev).round().to(torch.int32)
    chosen = ops.unmask_splits(rows, V)
    cands = sorted({chosen, *[int(v) for v in a.splits.split(",") if v]})
    for ns in cands:
        part = torch.empty((rows, ns, 3), dtype=torch.float32, device=dev)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for _ in range(2):
                ops.unmask_finalize(ops.unmask_partials(x[:rows], None, rows, ns, part=part), 1, rows, ns, cu, 0.9)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(REPS):  # back-to-back K3 launches: the replay gap is amortised
                    ops.unmask_finalize(ops.unmask_partials(x[:rows], None, rows, ns, part=part), 1, rows, ns, cu,
                                        0.9)
        torch.cuda.synchronize()
        points.append([(rows, ns), ns == chosen, g, part, cu])  # the graph reads these buffers: keep them alive
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = {p[0]: [] for p in points}
for _ in range(12):
    for key, _, g, _, _ in points:
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        times[key].append(e0.elapsed_time(e1) * 1e3 / REPS)
out = []
for (rows, ns), chosen, *_ in points:
    us = float(np.median(times[(rows, ns)][2:]))
    byts = rows * V * 2 + 9 * rows
    gbs = byts / (us * 1e-6) / 1e9
    out.append({"rows": rows, "n_vsplit": ns, "chosen": chosen, "us": round(us, 2), "gbs": round(gbs, 1),
                "frac": round(gbs / hbm, 4)})
    print(f"rows {rows:5d} splits {ns:3d}{'*' if chosen else ' '} {us:7.1f} us  {gbs:7.0f} GB/s  {gbs / hbm:.3f}")
fr = [o["frac"] for o in out if o["chosen"]]
summary = {"vocab": V, "peak_gbs": hbm, "reps_per_graph": REPS, "min_frac": min(fr), "median_frac": float(np.median(fr)),
           "points": out}
print(f"chooser: min frac {min(fr):.3f}  median {np.median(fr):.3f}")
if a.out:
    Path(a.out).write_text(json.dumps(summary, indent=1))
