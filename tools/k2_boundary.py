"""Where an item boundary's time goes inside K2 (diagnostics): from one traced launch on
a bench batch, per item boundary of every CTA, the PV issue gap across the boundary
(last PV of item e -> first PV of item e+1) against the median PV-to-PV interval inside
items, and what the first PV of e+1 waited for: O released by the epilogue of e
(role 15), its V tile (role 9), its P (role 3 of the warpgroup that owns the tile).
Cycles (clock64) since the CTA's setup stamp.

    python tools/k2_boundary.py [--workload sharegpt]
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


tr = torch.zeros((plan.grid, 4096), dtype=torch.int64, device=dev)
k2(1)
_lib.call("optimus_set_attn_trace", tr.data_ptr())
k2(0)
_lib.call("optimus_set_attn_trace", None)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.float64)
work = plan.work.cpu().numpy()
off = plan.cta_off.cpu().numpy()
R = lambda c, role, i: t[c, role * 256 + i]
gaps, inner, wait_o, wait_v, wait_p, epi_len, drain = [], [], [], [], [], [], []
v_top, v_free, v_iss, k_iss, s_iss = [], [], [], [], []
v_lat_in, v_lat_b = [], []
first_load = []
for c in range(plan.grid):
    c0 = R(c, 6, 1)
    items = work[off[c]: off[c + 1]]
    nt = [(int(w[5]) - int(w[4]) + 63) // 64 for w in items]
    if sum(nt) >= 256:
        continue
    first_load.append(R(c, 4, 0) - c0)
    tb = 0
    for e, n in enumerate(nt):
        pv = [R(c, 7, tb + j) - c0 for j in range(n)]
        inner += list(np.diff(pv))
        if e + 1 < len(nt):
            nxt = tb + n  # first tile of item e+1
            g = R(c, 7, nxt) - R(c, 7, nxt - 1)
            gaps.append(g)
            # epilogue of item e (warpgroup 0's stamps): entered, O complete, O released
            if R(c, 13, e) > 0 and R(c, 15, e) > 0:
                epi_len.append(R(c, 15, e) - R(c, 13, e))
                drain.append(R(c, 15, e) - R(c, 14, e))
                wait_o.append(R(c, 15, e) - R(c, 7, nxt - 1))
            wait_v.append(R(c, 9, nxt) - R(c, 7, nxt - 1))
            base = R(c, 7, nxt - 1)
            v_top.append(R(c, 0, nxt) - base)
            v_free.append(R(c, 10, nxt) - base)
            v_iss.append(R(c, 11, nxt) - base)
            k_iss.append(R(c, 5, nxt) - base)
            s_iss.append(R(c, 1, nxt) - base)
            v_lat_b.append(R(c, 9, nxt) - R(c, 11, nxt))
            if n >= 4:
                v_lat_in += [R(c, 9, tb + j) - R(c, 11, tb + j) for j in range(2, n)]
            wait_p.append(R(c, 7, nxt) - R(c, 9, nxt))
        tb += n
pc = lambda x: np.percentile(np.array(x), [10, 50, 90]).round(0) if len(x) else []
print(f"{a.workload}: grid {plan.grid}, work {plan.n_work}, boundaries {len(gaps)} (cycles)")
print(f"  PV-to-PV inside items          p10/50/90 {pc(inner)}")
print(f"  PV gap across item boundaries  p10/50/90 {pc(gaps)}")
print(f"  O released after last PV of e  p10/50/90 {pc(wait_o)}")
print(f"  epilogue entered -> O released p10/50/90 {pc(epi_len)}  (O complete -> released {pc(drain)})")
print(f"  next V landed after last PV    p10/50/90 {pc(wait_v)}")
print(f"  first PV of e+1 after its V    p10/50/90 {pc(wait_p)}")
print(f"  first K load issue after setup p10/50/90 {pc(first_load)}")
print("  first tile of e+1, relative to the last PV of e:")
print(f"    K producer top of tile        p10/50/90 {pc(v_top)}")
print(f"    K issued                      p10/50/90 {pc(k_iss)}")
print(f"    V slot free (v_empty)         p10/50/90 {pc(v_free)}")
print(f"    V issued                      p10/50/90 {pc(v_iss)}")
print(f"    S issued                      p10/50/90 {pc(s_iss)}")
print(f"  V latency (issued -> landed): boundary tiles {pc(v_lat_b)}, inside items {pc(v_lat_in)}")
