"""GPU time of one DeviceLoop iteration graph vs the host-planned device step on the
same batch (diagnostics): the loop graph replayed back to back (state advances; the
first iterations), events on the stream, no host work between replays."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24832_b200.device_loop import DeviceLoop  # noqa: E402
from paper_2605_24832_b200.engine import plan_batch  # noqa: E402

import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--seed-offset", type=int, default=1)
a = ap.parse_args()
a.page, a.seed, a.steps, a.chunk = 64, 0, 1, 32
a.batch = 128 if a.workload == "llada" else 64
dev = torch.device("cuda")
W = bench.build_decoder(a, dev, e2e_pools=False, reqs=bench.workload_requests(a, seed_offset=a.seed_offset))
dec = W.dec
plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), W.cfg.block_size, W.cfg.window_rule)
dm = dec.prepare(W.reqs, plans)
g = bench.capture_step(dec, dm)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(6):
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"host-planned device step (graph): {np.median(ts[1:]) * 1e3:.1f} us, split groups {dm.attn_plan.n_groups}")
dec.release_all(W.reqs)
reqs = bench.workload_requests(a, seed_offset=a.seed_offset)
loop = DeviceLoop(dec, reqs, bench.step_chunks(a, reqs))
loop.step()
torch.cuda.synchronize()
g = loop.graphs[0]
ts = []
for _ in range(6):
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"DeviceLoop iteration graph: {np.median(ts[1:]) * 1e3:.1f} us, device groups {int(loop.M['wcounts'][1])}")
