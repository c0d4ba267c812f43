"""K3 on a bench workload's real step (diagnostics): the fused one-launch unmask the
step runs (window rows gathered from the logit table through row_src) against the
two-launch form and against contiguous logits rows, for several vocab split counts.
CUDA graphs of 8 back-to-back launches, interleaved rounds.

    python tools/k3_variants.py [--workload ctx4096]
"""
import argparse
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
ap.add_argument("--splits", default="1,2,3,4")
a = ap.parse_args()
a.page, a.seed, a.steps, a.chunk = 64, 0, 1, 32
a.batch = 128 if a.workload == "llada" else 64
dev = torch.device("cuda")
W = bench.build_decoder(a, dev, layers=1, e2e_pools=False)
dec, fwd, cfg = W.dec, W.fwd, W.cfg
plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), cfg.block_size, cfg.window_rule)
dm = dec.prepare(W.reqs, plans)
m = dm.host
rows = m.n_rows
table, row_src = fwd.logits(dm)
V = table.shape[-1]
contig = table[:rows]
hbm, _ = bench.peaks()
print(f"{a.workload}: {rows} window rows, {m.n_req} requests, vocab {V}, chooser splits {ops.unmask_splits(rows, V)}")
cnt = torch.zeros(max(m.n_req, 1), dtype=torch.int32, device=dev)
REPS = 8
graphs = {}
for ns in [int(x) for x in a.splits.split(",")]:
    part = torch.empty((rows, ns, 3), dtype=torch.float32, device=dev)
    for src_name, (lg, rs) in (("gather", (table, row_src)), ("contig", (contig, None))):
        for form in ("fused", "two"):
            def fn(lg=lg, rs=rs, ns=ns, part=part, form=form):
                if form == "fused":
                    if rs is None:
                        rs_ = torch.arange(rows, dtype=torch.int32, device=dev)
                    ops.unmask_fused(lg, rs if rs is not None else fn.rs, rows, ns, dm.cu_rows, dm.row_req, cnt,
                                     cfg.confidence_threshold, cfg.fallback, part=part)
                else:
                    ops.unmask_finalize(ops.unmask_partials(lg, rs, rows, ns, part=part), 1, rows, ns, dm.cu_rows,
                                        cfg.confidence_threshold)
            fn.rs = torch.arange(rows, dtype=torch.int32, device=dev)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                fn(); fn(); s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(REPS):
                        fn()
            torch.cuda.synchronize()
            graphs[(ns, src_name, form)] = (g, part)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = {k: [] for k in graphs}
for _ in range(10):
    for k, (g, _) in graphs.items():
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) * 1e3 / REPS)
byts = rows * V * table.element_size()
for k in graphs:
    us = float(np.median(times[k][2:]))
    print(f"splits {k[0]}  {k[1]:6s} {k[2]:5s} {us:7.1f} us  {byts / us / 1e3 / hbm:.3f} of HBM")
