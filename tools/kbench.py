"""Kernel micro-benchmarks on the bench workload (diagnostics, not the contract)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
from paper_2605_24832_b200 import ops
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.engine import plan_batch
from paper_2605_24832_b200.synthetic import SyntheticForward

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="sharegpt")
ap.add_argument("--chunk", type=int, default=32)
ap.add_argument("--page", type=int, default=64)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--layers", type=int, default=36)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--dump", default="")
ap.add_argument("--ab", action="store_true")
ap.add_argument("--dbgs", default="0,16")  # OPTIMUS_DBG[:OPTIMUS_K2_RINGS] per variant
ap.add_argument("--plans", default="both")
ap.add_argument("--forces", default="whole,cut", help="OPTIMUS_PLAN_FORCE values to A/B (whole, cut, flat, giants, tail)")
ap.add_argument("--trace-fused", action="store_true")
a = ap.parse_args()
a.steps = 1
dev = torch.device("cuda")
reqs = bench.workload_requests(a)
P = a.page
spec_model = dict(bench.workload_spec(a.workload)["model"])
spec_model["num_layers"] = a.layers
cfg = DecodeConfig(**spec_model, page_size=P, max_batch=a.batch,
                   num_pages=bench.pages_needed(reqs, P) + 64,
                   max_pages_per_req=max((r.prompt_tokens + r.output_tokens + P - 1) // P for r in reqs) + 1)
fwd = SyntheticForward(cfg, a.batch * a.chunk, a.batch, device=dev)
dec = StreamingDecoder(cfg, fwd, device=dev)
for l in range(cfg.num_layers):
    dec.cache.k[l].normal_(); dec.cache.v[l].normal_()
plans = plan_batch(reqs, bench.step_chunks(a, reqs), cfg.block_size, cfg.window_rule)
dm = dec.prepare(reqs, plans)
dec.device_step(dm)
torch.cuda.synchronize()
m = dm.host
plan = dm.__dict__["attn_plan"]
out = dec._workspaces(plan, m.n_tok)
k2b, k1b, k3b, vis, flops = bench.algorithmic_bytes(dm, cfg)
print(f"n_tok={m.n_tok} rows={m.n_rows} vis_keys={vis} k2_bytes={k2b/1e6:.1f}MB work={plan.n_work} groups={plan.n_groups}")

def k1(l):
    q, k, v = fwd.qkv(l, dm); kc, vc = dec.cache.layer(l)
    ops.kv_append(k, v, dm.tok_req, dm.tok_pos, dm.prompt_len, dm.block_tables, kc, vc)
def k2(l):
    q, k, v = fwd.qkv(l, dm); kc, vc = dec.cache.layer(l)
    ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off, dm.vis_words,
                        dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok], ws_o=dec._ws_o, ws_ml=dec._ws_ml)
def k3():
    dec.run_unmask(dm)

def timed(fn, reps=10, label=""):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn(); s.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{label:40s} {ms*1e3:9.1f} us")
    return ms

L = cfg.num_layers
if a.ab:
    # A/B in one process, interleaved rounds (power capping drifts the clocks):
    # planner choice x epilogue overlap
    import os
    from paper_2605_24832_b200 import _lib
    variants = []
    for force in a.forces.split(","):
        os.environ["OPTIMUS_PLAN_FORCE"] = force
        pl = ops.plan_attention(m.cu_seqlens, m.key_end, cfg.num_q_heads, cfg.num_kv_heads, grid=dec.grid,
                                min_split_tiles=cfg.min_split_tiles, device=dev, page_size=cfg.page_size)
        for dbg in a.dbgs.split(","):
            variants.append((f"plan={force} dbg={dbg} groups={pl.n_groups}", pl, dbg))
        if a.plans == "whole":
            break
    os.environ.pop("OPTIMUS_PLAN_FORCE")
    graphs = []
    for name, pl, dbg in variants:
        parts = dbg.split(":")
        os.environ["OPTIMUS_DBG"] = parts[0]
        if len(parts) > 1 and parts[1]:
            os.environ["OPTIMUS_K2_RINGS"] = parts[1]
        else:
            os.environ.pop("OPTIMUS_K2_RINGS", None)
        if len(parts) > 2:  # "kernel": the separate split-KV combine kernel
            os.environ["OPTIMUS_K2_COMBINE"] = parts[2]
        else:
            os.environ.pop("OPTIMUS_K2_COMBINE", None)
        plan = pl
        out = dec._workspaces(pl, m.n_tok)
        s_ = torch.cuda.Stream(); s_.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_):
            k2(0); s_.synchronize()
            with torch.cuda.graph(g, stream=s_):
                for l in range(L):
                    k2(l)
        torch.cuda.synchronize()
        # per-variant CTA timeline (clock64 cycles)
        tr = torch.zeros((pl.grid, 4096), dtype=torch.int64, device=dev)
        _lib.call("optimus_set_attn_trace", tr.data_ptr()); k2(0); torch.cuda.synchronize()
        _lib.call("optimus_set_attn_trace", None)
        t = tr.cpu().numpy().astype(np.float64)
        done = (t[:, 6 * 256 + 3] - t[:, 6 * 256 + 1]) / 1e3
        ghz = np.median((t[:, 6 * 256 + 3] - t[:, 6 * 256 + 1]) / (t[:, 6 * 256 + 4] - t[:, 6 * 256 + 0]))
        print(f"{name}: SM clock during the traced launch ~{ghz:.2f} GHz (cycles/ns, setup excluded)")
        graphs.append((name, g, np.percentile(done, [0, 50, 90, 100]).round(1)))
    os.environ.pop("OPTIMUS_DBG")
    res = {name: [] for name, _, _ in graphs}
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    for rnd in range(12):
        for name, g, _ in graphs:
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) * 1e3 / L)
    for name, g, done in graphs:
        v = np.array(res[name][2:])
        print(f"{name:40s} K2 us/launch median {np.median(v):7.1f} min {v.min():7.1f}  CTA kcycles {done}")
    sys.exit(0)
t_k2_same = timed(lambda: [k2(0) for _ in range(L)], label="K2 x L same layer")
t_k2 = timed(lambda: [k2(l) for l in range(L)], label="K2 x L layers")
t_k1 = timed(lambda: [k1(l) for l in range(L)], label="K1 x L layers")
t_both = timed(lambda: [(k1(l), k2(l)) for l in range(L)], label="K1+K2 x L layers")
slot_abs = ops.slot_mapping(dm.tok_req, dm.tok_pos, dm.prompt_len, dm.block_tables, cfg.page_size, n_tok=m.n_tok)
def k2f(l):
    q, k, v = fwd.qkv(l, dm); kc, vc = dec.cache.layer(l)
    ops.paged_attention_append(q, k, v, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off,
                               dm.vis_words, dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok],
                               ws_o=dec._ws_o, ws_ml=dec._ws_ml, slot_abs=slot_abs)
t_k2f = timed(lambda: [k2f(l) for l in range(L)], label="K2+append fused x L layers") if plan.single_tile else 0
t_k3 = timed(k3, label="K3")
t_step = timed(lambda: dec.device_step(dm), label="full step")
print(f"K2 per launch (layers): {t_k2/L*1e3:.1f} us -> {k2b/(t_k2/L*1e-3)/1e9:.0f} GB/s; same-layer {t_k2_same/L*1e3:.1f} us")
print(f"fused K1+K2 per layer: {t_k2f/L*1e3:.1f} us vs separate {t_both/L*1e3:.1f} us")
print(f"K1 per launch: {t_k1/L*1e3:.2f} us -> {k1b/(t_k1/L*1e-3)/1e9:.0f} GB/s ; K3 {t_k3*1e3:.1f} us -> {k3b/(t_k3*1e-3)/1e9:.0f} GB/s")

# ---- timeline trace of one K2 launch
from paper_2605_24832_b200 import _lib
tr = torch.zeros((plan.grid, 4096), dtype=torch.int64, device=dev)
_lib.call("optimus_set_attn_trace", tr.data_ptr())
(k2f if a.trace_fused else k2)(0)
torch.cuda.synchronize()
_lib.call("optimus_set_attn_trace", None)
t = tr.cpu().numpy().astype(np.float64)
if a.dump:
    np.save(a.dump, t)
    np.save(a.dump.replace(".npy", "_work.npy"), plan.work.cpu().numpy())
    np.save(a.dump.replace(".npy", "_ctaoff.npy"), plan.cta_off.cpu().numpy())
np.set_printoptions(linewidth=220, precision=0, suppress=True)
R = lambda role: slice(role * 256, role * 256 + 256)
for c in (0, 70):
    c0 = t[c, 6 * 256 + 1]
    n = int((t[c, R(1)] > 0).sum())
    print(f"CTA {c}: tiles={n} (cycles since setup /100)")
    for role, name in [(0, "prod_top"), (4, "prod_free"), (5, "prod_issued"), (10, "vprod_free"), (11, "vprod_issued"),
                       (12, "mma_reachS"), (1, "mma_S"), (8, "mma_reachPV"), (9, "mma_Vlanded"), (7, "mma_PV"),
                       (2, "smx_Sready"), (3, "smx_Pdone")]:
        a0 = 20 if role in (2, 3) else 40  # softmax stamps are warpgroup 0's (every other tile)
        v = t[c, role * 256 + a0: role * 256 + a0 + 16]
        print(f"  {name:12s}", ((v - c0) / 100).round(0))
    print("  producer done / CTA done (kcycles):", (t[c, 6 * 256 + 2] - c0) / 1e3, (t[c, 6 * 256 + 3] - c0) / 1e3)
done = (t[:, 6 * 256 + 3] - t[:, 6 * 256 + 1]) / 1e3
print("CTA done kcycles pctl:", np.percentile(done, [0, 50, 90, 100]).round(1))
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(1e8))
e0.record(); k2(0); e1.record(); torch.cuda.synchronize()
print("single launch event time (us):", e0.elapsed_time(e1) * 1e3)
