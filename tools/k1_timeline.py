"""Timeline of one layer boundary, K2(l) -> K1(l+1) -> K2(l+1), on the bench workload
(diagnostics, not the contract): globaltimer stamps of every K2 CTA (entry, done) and
every staged-K1 block (entry, PDL wait done, rows landed, end), relative to the first
K2(l) CTA's entry.

    python tools/k1_timeline.py [--workload sharegpt] [--reps 5]

The K1 stamps need a library exporting optimus_set_k1_trace (the staged-K1 experiment,
profiles/dead_ends/r2at_staged_k1.md); without it only the K2 columns are filled.
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
ap.add_argument("--chunk", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--between", default="k1", choices=["k1", "combine0", "combine0+k1"],
                help="what runs between K2(0) and K2(1): K1(1), a split-KV combine with a device "
                     "group count of 0 (the DeviceLoop's per-layer launch), or both")
a = ap.parse_args()
a.page, a.seed, a.steps, a.batch = 64, 0, 1, 64
dev = torch.device("cuda")
W = bench.build_decoder(a, dev, world=1, rank=0, layers=3, e2e_pools=False)
dec, fwd, cfg = W.dec, W.fwd, W.cfg
plans = plan_batch(W.reqs, bench.step_chunks(a, W.reqs), cfg.block_size, cfg.window_rule)
dm = dec.prepare(W.reqs, plans)
dec.device_step(dm)
torch.cuda.synchronize()
m = dm.host
plan = dm.__dict__["attn_plan"]
out = dec._workspaces(plan, m.n_tok)


def k1(l):
    q, k, v = fwd.qkv(l, dm)
    kc, vc = dec.cache.layer(l)
    ops.kv_append(k, v, dm.tok_req, dm.tok_pos, dm.prompt_len, dm.block_tables, kc, vc)


def k2(l):
    q, k, v = fwd.qkv(l, dm)
    kc, vc = dec.cache.layer(l)
    ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off, dm.vis_words,
                        dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok], ws_o=dec._ws_o, ws_ml=dec._ws_ml)


zero = torch.zeros(4, dtype=torch.int32, device=dev)
gdummy = torch.zeros((1, 8), dtype=torch.int32, device=dev)
ws_dummy = torch.zeros(64 * 128 * 128, dtype=torch.float32, device=dev)  # never read: 0 groups


def combine0():
    _lib.check(_lib.call(
        "optimus_paged_attn_combine_dev", gdummy.data_ptr(), zero.data_ptr(), 64, ws_dummy.data_ptr(),
        ws_dummy.data_ptr(), cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, out.data_ptr(), out.stride(0),
        torch.cuda.current_stream().cuda_stream), "combine_dev")


tra = torch.zeros((plan.grid, 4096), dtype=torch.int64, device=dev)
trb = torch.zeros_like(tra)
trk = torch.zeros((1024, 8), dtype=torch.int64, device=dev)
rows = []
HAS_K1_TRACE = hasattr(_lib.load(), "optimus_set_k1_trace")


def set_k1_trace(ptr):
    if HAS_K1_TRACE:
        _lib.call("optimus_set_k1_trace", ptr)


# one CUDA graph of K2(2), K2(0), K1(1), K2(1): launched back to back as inside a step
# (the trace pointers are read when each launch is recorded)
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s_):
    k2(2); k2(0); k1(1); k2(1)
    s_.synchronize()
    with torch.cuda.graph(g, stream=s_):
        k2(2)
        _lib.call("optimus_set_attn_trace", tra.data_ptr())
        k2(0)
        _lib.call("optimus_set_attn_trace", None)
        set_k1_trace(trk.data_ptr())
        if a.between.startswith("combine0"):
            combine0()
        if a.between.endswith("k1"):
            k1(1)
        set_k1_trace(None)
        _lib.call("optimus_set_attn_trace", trb.data_ptr())
        k2(1)
        _lib.call("optimus_set_attn_trace", None)
torch.cuda.synchronize()
for rep in range(a.reps + 1):
    for t in (tra, trb, trk):
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    if rep == 0:
        continue
    A = tra.cpu().numpy()[:, 6 * 256: 6 * 256 + 5].astype(np.float64)
    B = trb.cpu().numpy()[:, 6 * 256: 6 * 256 + 5].astype(np.float64)
    K = trk.cpu().numpy().astype(np.float64)
    K = K[K[:, 1] > 0]
    if len(K) == 0:  # the one-thread-per-vector K1 (OPTIMUS_K1_STAGED=0) is not traced
        K = np.full((1, 8), np.nan)
    t0 = A[:, 0].min()
    a_done = A[:, 4] - t0
    b_entry = B[:, 0] - t0
    b_done = B[:, 4] - t0
    Bf = trb.cpu().numpy().astype(np.float64)
    # first K tile issue of K2(l+1): clock64 since setup, at ~1.9 cycles/ns
    b_first = b_entry + (Bf[:, 4 * 256] - Bf[:, 6 * 256 + 1]) / 1.9
    rows.append(dict(
        a_done_first=a_done.min(), a_done_last=a_done.max(),
        k1_entry_min=(K[:, 1] - t0).min(), k1_entry_max=(K[:, 1] - t0).max(),
        k1_wait=(K[:, 2] - t0).max(), k1_landed_med=np.median(K[:, 3] - t0), k1_landed_max=(K[:, 3] - t0).max(),
        k1_end_max=(K[:, 4] - t0).max(), k1_blocks=len(K), k1_sms=len(set(K[:, 0].astype(int))),
        b_entry_min=b_entry.min(), b_entry_med=np.median(b_entry), b_entry_max=b_entry.max(),
        b_first_min=b_first.min(), b_first_med=np.median(b_first), b_done_last=b_done.max()))
print(f"between: {a.between}")
print(f"workload {a.workload}: K2 grid {plan.grid}, n_tok {m.n_tok}; times in us from K2(l)'s first CTA entry")
for k in rows[0]:
    v = np.array([r[k] for r in rows])
    print(f"  {k:16s} " + " ".join(f"{x / 1e3:8.2f}" if not k.startswith("k1_b") and not k.startswith("k1_s") else f"{x:8.0f}"
                                      for x in v))
