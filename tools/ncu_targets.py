"""One decode step of a workload, for ncu captures of single kernels (diagnostics).

    ncu --set full -k regex:kv_append -c 1 -o out python tools/ncu_targets.py --workload sharegpt
    python tools/ncu_targets.py --workload sharegpt --loop     # one DeviceLoop iteration (device planners)

--tp N runs rank 0's KV-head shard of tp N (as bench.py's per-rank projection).
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24832_b200.engine import plan_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--tp", type=int, default=1)
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--loop", action="store_true")
a = ap.parse_args()
a.page, a.seed, a.steps, a.chunk = 64, 0, 1, 32
a.batch = 128 if a.workload == "llada" else 64
dev = torch.device("cuda")
W = bench.build_decoder(a, dev, world=a.tp, rank=0, layers=a.layers, e2e_pools=False)
if a.loop:
    from paper_2605_24832_b200.device_loop import DeviceLoop
    loop = DeviceLoop(W.dec, W.reqs, bench.step_chunks(a, W.reqs))
    loop.step()
else:
    plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), W.cfg.block_size, W.cfg.window_rule)
    dm = W.dec.prepare(W.reqs, plans)
    W.dec.device_step(dm)
torch.cuda.synchronize()
print("done")
