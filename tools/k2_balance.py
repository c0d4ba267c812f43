"""How balanced one K2 launch is across its CTAs (diagnostics): per CTA the planned
load (tiles + 2.5 per item, the planner's cost model) and the traced end time (cycles
since setup), their spread and correlation, on a bench workload's batch.

    python tools/k2_balance.py [--workload sharegpt]
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
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
a.page, a.seed, a.steps, a.chunk = 64, 0, 1, 32
a.batch = 128 if a.workload == "llada" else 64
dev = torch.device("cuda")
W = bench.build_decoder(a, dev, layers=2, e2e_pools=False)
dec, fwd, cfg = W.dec, W.fwd, W.cfg
plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), cfg.block_size, cfg.window_rule)
dm = dec.prepare(W.reqs, plans)
dec.device_step(dm)
torch.cuda.synchronize()
m = dm.host
plan = dm.__dict__["attn_plan"]
out = dec._workspaces(plan, m.n_tok)


def k2(l):
    q, k, v = fwd.qkv(l, dm)
    kc, vc = dec.cache.layer(l)
    ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off, dm.vis_words,
                        dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok], ws_o=dec._ws_o, ws_ml=dec._ws_ml)


work = plan.work.cpu().numpy()
off = plan.cta_off.cpu().numpy()
tiles = np.array([sum((int(w[5]) - int(w[4]) + 63) // 64 for w in work[off[c]: off[c + 1]]) for c in range(plan.grid)])
items = np.diff(off)
load = tiles + 2.5 * items
tr = torch.zeros((plan.grid, 4096), dtype=torch.int64, device=dev)
ends = []
for rep in range(a.reps):
    k2(1)  # a launch in flight before the traced one, as in a step
    _lib.call("optimus_set_attn_trace", tr.data_ptr())
    k2(0)
    _lib.call("optimus_set_attn_trace", None)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.float64)
    start = t[:, 6 * 256 + 4 - 4]  # globaltimer at entry
    end = t[:, 6 * 256 + 4]        # globaltimer at the end
    ends.append((end - start.min()) / 1e3)
e = np.median(np.array(ends), axis=0)
print(f"{a.workload}: grid {plan.grid}, work {plan.n_work}, tiles/CTA mean {tiles.mean():.1f} max {tiles.max()}, "
      f"items/CTA mean {items.mean():.2f} max {items.max()}")
print(f"planned load (tiles + 2.5/item): mean {load.mean():.1f} max {load.max():.1f} (max/mean {load.max() / load.mean():.3f})")
print(f"CTA end us from the first entry: min {e.min():.2f} median {np.median(e):.2f} mean {e.mean():.2f} "
      f"p90 {np.percentile(e, 90):.2f} max {e.max():.2f}")
print(f"corr(end, planned load) {np.corrcoef(e, load)[0, 1]:.3f}; corr(end, items) {np.corrcoef(e, items)[0, 1]:.3f}")
fit = np.linalg.lstsq(np.stack([np.ones_like(e), tiles, items], 1), e, rcond=None)[0]
print(f"end ~ {fit[0]:.2f} + {fit[1]:.3f}/tile + {fit[2]:.3f}/item us")
order = np.argsort(-e)[:8]
print("latest CTAs (end us, tiles, items):", [(round(float(e[c]), 2), int(tiles[c]), int(items[c])) for c in order])
