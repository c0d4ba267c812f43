"""Where the end-to-end closed loop spends its time (diagnostics): bench.run_e2e's
ShareGPT closed loop through StreamingDecoder.step with step_backend "loop_lookahead",
with a CUDA event pair around every graph replay.  Reports per step: the wall time, the
GPU time of the iteration graph, the GPU idle gap before it (host-bound when > 0), and
the host time inside DeviceLoop.step (waiting on the in-flight iteration, then the
host apply) vs outside it (admissions, the caller).

    python tools/e2e_loop_timeline.py [--steps 40]
"""
import argparse
import dataclasses
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--workload", default="sharegpt")
a = ap.parse_args()
a.page, a.seed, a.chunk = 64, 0, 32
a.batch = 128 if a.workload == "llada" else 64
a.e2e_steps = a.steps
dev = torch.device("cuda")
W = bench.build_decoder(a, dev, world=1, rank=0)
dec, pool = W.dec, W.pool
batch, spare = list(pool[0]), list(pool[1])
dec.cfg = dataclasses.replace(dec.cfg, step_backend="loop_lookahead")

ev = []  # (start, end) per replay, in launch order


class Timed:
    def __init__(self, g):
        self.g = g

    def replay(self):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        self.g.replay()
        e.record()
        ev.append((s, e))


def one():
    global batch
    L = dec._loop
    if L is not None and L.graphs and not isinstance(L.graphs[0], Timed):
        L.graphs = [Timed(g) for g in L.graphs]
    t0 = time.perf_counter()
    summ = dec.step(batch, bench.step_chunks(a, batch))
    t1 = time.perf_counter()
    done = [r for r in batch if r.finished]
    if done:
        batch = [r for r in batch if not r.finished]
        while len(batch) < a.batch and spare:
            batch.append(spare.pop())
    t2 = time.perf_counter()
    return sum(len(s.commits) for s in summ), t1 - t0, t2 - t1


for _ in range(3):
    one()
torch.cuda.synchronize()
L = dec._loop
L.t_device = 0.0
ev.clear()
rows = []
t_all = time.perf_counter()
for _ in range(a.steps):
    c, t_in, t_out = one()
    rows.append((c, t_in, t_out))
torch.cuda.synchronize()
el = time.perf_counter() - t_all
gpu = np.array([s.elapsed_time(e) for s, e in ev]) * 1e3
gap = np.array([ev[i - 1][1].elapsed_time(ev[i][0]) for i in range(1, len(ev))]) * 1e3
commits = sum(r[0] for r in rows)
t_in = np.array([r[1] for r in rows]) * 1e6
t_out = np.array([r[2] for r in rows]) * 1e6
print(f"{a.workload} closed loop, {a.steps} steps: {commits / el:.0f} tokens/s, {el / a.steps * 1e6:.0f} us/step wall")
print(f"  iteration graph GPU time   median {np.median(gpu):7.0f} us  (min {gpu.min():.0f}, max {gpu.max():.0f})")
print(f"  GPU idle gap before graph  median {np.median(gap):7.1f} us  (sum {gap.sum() / a.steps:.1f} us/step)")
print(f"  host in DeviceLoop.step    median {np.median(t_in):7.0f} us  (of which waiting {L.t_device / a.steps * 1e6:.0f} us/step)")
print(f"  host outside (admissions)  median {np.median(t_out):7.0f} us")
print(f"  commits per step           median {np.median([r[0] for r in rows]):7.0f}")
