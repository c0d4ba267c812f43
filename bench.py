"""Benchmark of the Optimus streaming chunked block-decode step on B200.

Metric (BASELINE.json): decoded tokens/sec and attention HBM GB/s (% roofline) at
SDAR-8B shape.  Workload (configs[1]): SDAR-8B-shaped attention (32 q heads,
8 kv heads, head_dim 128, block 32), batch 64, ShareGPT-like lengths
(213/508 in, 321/214 out), chunk 32 (``--chunk``), 36 layers, vocab 151936.

One *step* = the whole hot path once for the batch: for each of the 36 layers
K1 (KV append) + K2 (paged attention), then K3 (unmask over every window row).
``value`` = committed tokens per step x steps / device time (inputs resident,
step replayed as one CUDA graph).  ``e2e`` = the same metric through the public
per-step call ``StreamingDecoder.step`` (host planning, one H2D of the step
metadata, device step, one D2H of the commit masks, host apply) on a live
closed-loop batch.

Multi-GPU (torchrun): KV heads are sharded over ranks (8/N each) and the unmask
over vocabulary shards; the per-row (max, sum, argmax) partials are exchanged
with one NCCL all-gather so every rank takes identical commit decisions.

``--impl reference`` times the CPU oracle (oracle/numeric.py: the reference
specifies this path in prose only) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SDAR8B = dict(num_layers=36, num_q_heads=32, num_kv_heads=8, head_dim=128, vocab=151936)
# LLaDA2.0-16B-MoE-shaped attention (config 4): GQA 16/4, d=128, 20 layers, 157K vocab.
# Model dims are not in /root/reference ([external, assumed]); BASELINE.json fixes the
# 157K vocabulary, batch 128 and mixed per-request chunks.
LLADA16B = dict(num_layers=20, num_q_heads=16, num_kv_heads=4, head_dim=128, vocab=157184)
# SDAR-30B-A3B-shaped (config 5): Qwen3-30B-A3B attention geometry, 48 layers, hidden 2048
# ([external, assumed]: model dims are not in /root/reference).  4 KV heads: at TP 8 every
# KV head is replicated on 2 ranks, each rank computing 4 of its 8 query heads.
SDAR30B = dict(num_layers=48, num_q_heads=32, num_kv_heads=4, head_dim=128, vocab=151936)
SDAR30B_HIDDEN = 2048
# commit profiles (calibrated_profile, tests/golden/commits.json and SURVEY §8d)
Q_SHAREGPT_DENSE = 0.7758267092770552
Q_LONGBENCH_DENSE = 0.835508
Q_SHAREGPT_MOE = 0.6015936600147661


def workload_spec(name):
    from paper_2605_24832_b200.synthetic import LONGBENCH, SHAREGPT
    return {
        "sharegpt": dict(model=SDAR8B, batch=64, lengths=SHAREGPT, q=Q_SHAREGPT_DENSE, prompt=None, clip=None,
                         mixed=None),
        "ctx4096": dict(model=SDAR8B, batch=64, lengths=SHAREGPT, q=Q_SHAREGPT_DENSE, prompt=4096, clip=None,
                        mixed=None),
        "longbench": dict(model=SDAR8B, batch=64, lengths=LONGBENCH, q=Q_LONGBENCH_DENSE, prompt=None,
                          clip=(4096, 16384), mixed=None),
        "llada": dict(model=LLADA16B, batch=128, lengths=SHAREGPT, q=Q_SHAREGPT_MOE, prompt=None, clip=None,
                      mixed=(8, 16, 24, 32)),
        # config 5: the TP decode step with the row-parallel o-proj + all-reduce per layer
        "tp30b": dict(model=SDAR30B, batch=64, lengths=SHAREGPT, q=Q_SHAREGPT_MOE, prompt=None, clip=None,
                      mixed=None, oproj_hidden=SDAR30B_HIDDEN),
    }[name]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--chunk", type=int, default=32)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--page", type=int, default=64)
    ap.add_argument("--workload", choices=["sharegpt", "ctx4096", "longbench", "llada", "tp30b"],
                    default="sharegpt")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-target", action="store_true", help="skip the 4K-context K2 roofline line")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    if a.batch is None:
        a.batch = workload_spec(a.workload)["batch"]
    return a


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for _, _, flags in rows for n, f in zip(names, flags) if f.lower() == "active"})
        loaded = [r[0] for r in rows if r[0] > 0.5 * r[1]] or [r[0] for r in rows]
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": rows[0][1], "reasons": reasons,
                "samples": len(rows)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------- workload
def workload_requests(args, seed_offset=0, n=None):
    from paper_2605_24832_b200.synthetic import make_batch
    w = workload_spec(args.workload)
    return make_batch(args.seed + seed_offset, n or args.batch, args.chunk, lengths=w["lengths"], q=w["q"],
                      fixed_prompt=w["prompt"], prompt_clip=w["clip"], first_id=seed_offset * 100000)


def step_chunks(args, reqs):
    """One global chunk (the reference's FixedChunk/ElasticChunk iteration) or, for
    the mixed-chunk workload, one seeded chunk per request from the elastic set."""
    w = workload_spec(args.workload)
    if not w["mixed"]:
        return args.chunk
    rng = np.random.default_rng(args.seed + 7)
    return [int(c) for c in rng.choice(w["mixed"], len(reqs))]


def pages_needed(reqs, page):
    return sum((r.prompt_tokens + r.output_tokens + page - 1) // page for r in reqs)


def algorithmic_bytes(dm, cfg):
    """K2 / K1 / K3 algorithmic bytes per launch."""
    m = dm.host
    d, hq, hkv = cfg.head_dim, cfg.num_q_heads, cfg.num_kv_heads
    vis_keys = 0
    for r in range(m.n_req):
        ke = int(m.key_end[r])
        if ke == 0:
            continue
        vb = int(m.vis_base[r])
        w0, w1 = int(m.vis_off[r]), int(m.vis_off[r + 1])
        bits = np.unpackbits(m.vis_words[w0:w1].view(np.uint8), bitorder="little")[: ke - vb]
        vis_keys += vb + int(bits.sum())
    k2 = vis_keys * hkv * d * 2 * 2 + m.n_tok * hq * d * 2 * 2
    k1 = m.n_tok * hkv * d * 2 * 2 * 2 + m.n_tok * 8
    k3 = m.n_rows * cfg.vocab * 2 + m.n_rows * 9
    flops = 0
    for r in range(m.n_req):
        q_r = int(m.cu_seqlens[r + 1] - m.cu_seqlens[r])
        flops += 4 * q_r * hq * int(m.key_end[r]) * d
    return k2, k1, k3, vis_keys, flops


# ----------------------------------------------------------------------------- CPU oracle
def cpu_oracle_sample(args, reqs, plans, m, cfg, n_layers_sample=1, row_frac=None, rng_seed=0):
    """Time the CPU oracle on a bounded sample of the step; returns (seconds for
    the full step extrapolated, description)."""
    import torch
    from oracle import numeric as on
    rng = np.random.default_rng(rng_seed)
    P = args.page
    hq, hkv, d = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
    # one layer's cache for the batch, contiguous pages in batch order
    bt = np.zeros_like(m.block_tables)
    n_pages = 0
    for r, req in enumerate(reqs):
        n = (req.prompt_tokens + req.output_tokens + P - 1) // P
        bt[r, :n] = np.arange(n_pages, n_pages + n)
        n_pages += n
    kc = rng.standard_normal((n_pages, hkv, P, d), dtype=np.float32)
    vc = rng.standard_normal((n_pages, hkv, P, d), dtype=np.float32)
    q = rng.standard_normal((m.n_tok, hq, d), dtype=np.float32)
    kn = rng.standard_normal((m.n_tok, hkv, d), dtype=np.float32)
    vis_list = [on.visible_outputs(r.states, list(p.kv_positions) + list(p.window)) for r, p in zip(reqs, plans)]
    t0 = time.perf_counter()
    for _ in range(n_layers_sample):
        slots = on.slot_mapping(m.tok_req, m.tok_pos, m.prompt_len, bt, P)
        on.kv_append(kc, vc, kn, kn, slots, P)
        on.paged_attention(q, kc, vc, m.cu_seqlens, m.tok_pos, m.prompt_len, vis_list, bt,
                           cfg.block_size, P)
    t_layer = (time.perf_counter() - t0) / n_layers_sample
    n_rows = m.n_rows
    n_s = n_rows if row_frac is None else max(1, int(round(n_rows * row_frac)))
    logits = rng.standard_normal((n_s, cfg.vocab), dtype=np.float32)
    cu = np.array([0, n_s], dtype=np.int32)
    t0 = time.perf_counter()
    on.unmask(logits, cu, cfg.confidence_threshold)
    t_unmask = (time.perf_counter() - t0) * (n_rows / n_s)
    total = t_layer * cfg.num_layers + t_unmask
    threads = torch.get_num_threads()
    return total, t_layer, t_unmask, threads


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, bounded per-step sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_24832_b200.decode import DecodeConfig
    from paper_2605_24832_b200.engine import plan_batch
    from paper_2605_24832_b200.meta import build_step_meta
    M = workload_spec(args.workload)["model"]
    cfg = DecodeConfig(**M, page_size=args.page, max_batch=args.batch)
    reqs = workload_requests(args)
    plans = plan_batch(reqs, step_chunks(args, reqs), cfg.block_size, cfg.window_rule)
    bt = np.zeros((len(reqs), 1), dtype=np.int32)
    P = args.page
    maxp = max((r.prompt_tokens + r.output_tokens + P - 1) // P for r in reqs)
    bt = np.zeros((len(reqs), maxp), dtype=np.int32)
    m = build_step_meta(reqs, plans, cfg.block_size, bt)
    # commits per step as the device path would take them (same synthetic profile)
    q = workload_spec(args.workload)["q"]
    commits = sum(min(1, len(p.window)) + sum(q ** j for j in range(1, len(p.window))) for p in plans)
    times = []
    # each step: one layer (of 36) of K1+K2 for the whole batch + 1/36 of the unmask rows
    for i in range(args.warmup + args.steps):
        total, t_layer, t_unmask, threads = cpu_oracle_sample(args, reqs, plans, m, cfg, 1,
                                                              row_frac=1.0 / cfg.num_layers, rng_seed=i)
        if i >= args.warmup:
            times.append(total)
    step_s = float(np.mean(times))
    value = commits / step_s
    line = {
        "impl": "reference", "metric": "decoded_tokens_per_s", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": workload_name(args), "batch": args.batch,
                   "chunk": chunk_label(args), "layers": cfg.num_layers, "page_size": P},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": "per step: K1+K2 of 1 of 36 layers for the whole batch + unmask of 1/36 "
                                   "of the window rows (numpy oracle), scaled x36"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        if world == 1 and args.gpus > 1:
            sys.exit("--gpus N > 1 must be launched with torchrun --nproc-per-node N")
    # OPTIMUS_DIST_BACKEND=gloo (validation only): ranks may share a GPU and the
    # unmask partials travel through host memory; production is NCCL, one GPU per rank
    backend = os.environ.get("OPTIMUS_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2605_24832_b200 import ops
    from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
    from paper_2605_24832_b200.engine import plan_batch
    from paper_2605_24832_b200.parallel import TensorParallelUnmask
    from paper_2605_24832_b200.synthetic import SyntheticForward

    M = workload_spec(args.workload)["model"]
    if M["num_q_heads"] % world or (M["num_kv_heads"] % world and world % M["num_kv_heads"]):
        sys.exit(f"world size must divide the {M['num_q_heads']} query heads and divide or be a multiple "
                 f"of the {M['num_kv_heads']} KV heads")
    kv_local = max(1, M["num_kv_heads"] // world)  # > Hkv ranks: each KV head replicated
    reqs = workload_requests(args)
    P = args.page
    long_ctx = args.workload in ("longbench", "ctx4096")
    # closed-loop e2e: a second batch plus a spare pool for respawns (smaller for the
    # long-context workloads so three batches of KV fit next to each other in HBM)
    e2e_pool = [workload_requests(args, seed_offset=1),
                workload_requests(args, seed_offset=2, n=16 if long_ctx else None)]
    n_pages = pages_needed(reqs, P) + sum(pages_needed(b, P) for b in e2e_pool) + 64
    maxp = max((r.prompt_tokens + r.output_tokens + P - 1) // P for b in [reqs] + e2e_pool for r in b) + 1
    cfg = DecodeConfig(num_layers=M["num_layers"], num_q_heads=M["num_q_heads"] // world,
                       num_kv_heads=kv_local, head_dim=M["head_dim"],
                       vocab=M["vocab"], page_size=P, max_batch=args.batch,
                       num_pages=n_pages, max_pages_per_req=maxp)
    vshard = (rank * cfg.vocab // world, (rank + 1) * cfg.vocab // world)
    wl = workload_spec(args.workload)
    max_chunk = max(wl["mixed"]) if wl["mixed"] else args.chunk
    max_tok = args.batch * max(max_chunk, 2)
    if wl.get("oproj_hidden"):
        from paper_2605_24832_b200.synthetic import TPForward
        fwd = TPForward(cfg, max_tok, args.batch, wl["oproj_hidden"], M["num_q_heads"], world, rank,
                        seed=args.seed, vocab_shard=vshard, q=wl["q"], device=dev)
    else:
        fwd = SyntheticForward(cfg, max_tok, args.batch, device=dev, seed=args.seed, vocab_shard=vshard,
                               q=wl["q"])
    dec = StreamingDecoder(cfg, fwd, device=dev)
    if world > 1:
        dec.unmask_impl = TensorParallelUnmask(world, rank, vshard[0])
    # KV cache content: random bf16 (prefill is outside the path)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    for l in range(cfg.num_layers):
        dec.cache.k[l].normal_(generator=g)
        dec.cache.v[l].normal_(generator=g)

    plans = plan_batch(reqs, step_chunks(args, reqs), cfg.block_size, cfg.window_rule)
    dm = dec.prepare(reqs, plans)
    res = dec.device_step(dm)  # warm + lazy init
    torch.cuda.synchronize()
    commits_per_step = int(res.commit_mask[: dm.host.n_rows].sum().item())
    k2b, k1b, k3b, vis_keys, flops = algorithmic_bytes(dm, cfg)

    # ---- capture the device step once; replay = one step.  With N > 1 the step holds
    # the NCCL all-gather of the unmask partials: it is replayed eagerly (the launches
    # overlap the ~1.4 ms of device work) instead of capturing a collective.
    if world == 1:
        stream = torch.cuda.Stream(device=dev)
        stream.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for _ in range(2):
                dec.device_step(dm)
            stream.synchronize()
            with torch.cuda.graph(graph, stream=stream):
                dec.device_step(dm)
        torch.cuda.synchronize()
    else:
        class _Eager:
            @staticmethod
            def replay():
                dec.device_step(dm)
        graph = _Eager()
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
    n_launch = 2 * cfg.num_layers + (cfg.num_layers if dec.last_plan.n_groups else 0) + 2

    sampler = ClockSampler(local)
    sampler.start()
    # soak ~0.5 s so the timed region runs at steady clocks (sampled throughout)
    t_soak = time.time()
    while time.time() - t_soak < 0.5:
        graph.replay()
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        graph.replay()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-kernel durations: each kernel alone, back to back over the 36 layers,
    # captured in a CUDA graph and timed with CUDA events on the launching stream
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
        ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off,
                            dm.vis_words, dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok],
                            ws_o=dec._ws_o, ws_ml=dec._ws_ml)

    L = cfg.num_layers
    k1_us = graph_time(lambda: [k1(l) for l in range(L)], dev) / L * 1e3
    k2_us = graph_time(lambda: [k2(l) for l in range(L)], dev) / L * 1e3
    k3_us = graph_time(lambda: dec.run_unmask(dm), dev, use_graph=world == 1) * 1e3

    # ---- end to end through the public per-step call (closed loop, live state)
    dec.release_all(reqs)
    e2e = run_e2e(args, dec, fwd, e2e_pool, world, dev)
    dloop = run_device_loop(args, dec, world)

    hbm, peak_kind = peaks()
    achieved = k2b / (k2_us * 1e-6) / 1e9
    traffic, traffic_src = profiled_traffic(args)
    target = None
    if world == 1 and not args.no_target:
        del graph
        torch.cuda.empty_cache()
        target = target_roofline(args, dev)
    value = commits_per_step * world / world / (ms * 1e-3)  # commits are global (identical on all ranks)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        total, t_layer, t_unmask, threads = cpu_oracle_sample(args, reqs, plans, dm.host, cfg_full(args), 1,
                                                              row_frac=0.125)
        cpu = {"value": commits_per_step / total, "unit": "tokens/s", "cores": threads, "kind": "port",
               "sample": f"numpy oracle: K1+K2 of 1 layer for the whole batch ({t_layer*1e3:.0f} ms) x36 "
                         f"+ unmask of 1/8 of the {dm.host.n_rows} window rows scaled to all "
                         f"({t_unmask*1e3:.0f} ms)"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": "decoded_tokens_per_s", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": workload_name(args), "batch": args.batch,
                   "chunk": chunk_label(args), "layers": cfg.num_layers, "q_heads": M["num_q_heads"],
                   "kv_heads": M["num_kv_heads"], "head_dim": cfg.head_dim, "block": cfg.block_size,
                   "page_size": P, "vocab": cfg.vocab, "tp": world,
                   "tokens_per_step": int(dm.host.n_tok), "window_rows": int(dm.host.n_rows),
                   "commits_per_step": commits_per_step, "visible_keys": vis_keys,
                   "l2": "inputs > L2: 36 per-layer KV caches read once per step "
                         f"({vis_keys * cfg.num_kv_heads * cfg.head_dim * 4 * cfg.num_layers / 1e9:.2f} GB)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "kernel": "paged_attn_kernel (K2)",
                     "peak_kind": peak_kind, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": k2b, "launch_us": k2_us},
        "kernels_us": {"k1_kv_append": k1_us, "k2_paged_attn": k2_us, "k3_unmask": k3_us,
                       "k2_share_of_step": k2_us * cfg.num_layers / (ms * 1e3),
                       "k1_gbs": k1b / (k1_us * 1e-6) / 1e9, "k3_gbs": k3b / (k3_us * 1e-6) / 1e9,
                       "k2_tflops": flops / (k2_us * 1e-6) / 1e12},
        "attention_hbm_gbs": achieved,
        "roofline_target_4k": target,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_device_loop": dloop,
        "gpu_launches": n_launch * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def target_roofline(args, dev, n_layers=8):
    """K2 roofline at BASELINE north_star's target shape (SDAR-8B heads, block 32,
    4K context, batch 64, chunk 32): 8 per-layer caches (9 GB, > L2) read back to back."""
    import torch
    from paper_2605_24832_b200 import ops
    from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
    from paper_2605_24832_b200.engine import plan_batch
    from paper_2605_24832_b200.synthetic import SyntheticForward

    class A:
        pass
    a = A()
    a.workload, a.chunk, a.page, a.batch, a.seed, a.steps = "ctx4096", 32, args.page, 64, args.seed, 1
    reqs = workload_requests(a)
    P = a.page
    M = SDAR8B
    cfg = DecodeConfig(num_layers=n_layers, num_q_heads=M["num_q_heads"], num_kv_heads=M["num_kv_heads"],
                       head_dim=M["head_dim"], vocab=M["vocab"], page_size=P, max_batch=a.batch,
                       num_pages=pages_needed(reqs, P) + 64,
                       max_pages_per_req=max((r.prompt_tokens + r.output_tokens + P - 1) // P for r in reqs) + 1)
    fwd = SyntheticForward(cfg, a.batch * a.chunk, a.batch, device=dev, seed=args.seed)
    dec = StreamingDecoder(cfg, fwd, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    for l in range(n_layers):
        dec.cache.k[l].normal_(generator=g)
        dec.cache.v[l].normal_(generator=g)
    dm = dec.prepare(reqs, plan_batch(reqs, a.chunk, cfg.block_size, cfg.window_rule))
    dec.device_step(dm)
    torch.cuda.synchronize()
    m = dm.host
    plan = dm.__dict__["attn_plan"]
    out = dec._workspaces(plan, m.n_tok)
    k2b = algorithmic_bytes(dm, cfg)[0]

    def k2(l):
        q, k, v = fwd.qkv(l, dm)
        kc, vc = dec.cache.layer(l)
        ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off,
                            dm.vis_words, dm.block_tables, plan, cfg.block_size, out=out[: m.n_tok],
                            ws_o=dec._ws_o, ws_ml=dec._ws_ml)
    us = graph_time(lambda: [k2(l) for l in range(n_layers)], dev) / n_layers * 1e3
    hbm, kind = peaks()
    ach = k2b / (us * 1e-6) / 1e9
    res = {"workload": "sdar8b-attn-ctx4096 (north_star target: 4K context, batch 64, chunk 32)",
           "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "peak_kind": kind,
           "algorithmic_bytes_per_launch": k2b, "launch_us": us, "split_kv_groups": plan.n_groups}
    del dec, fwd
    torch.cuda.empty_cache()
    return res


def profiled_traffic(args):
    """DRAM bytes per K2 launch from the committed ncu --set full capture of this
    workload (profiles/*_ncu.json, tools/ncu_summary.py), else None."""
    if args.workload != "sharegpt" or args.chunk != 32 or args.page != 64:
        return None, None
    best = None
    for f in sorted((ROOT / "profiles").glob("*_ncu.json")):
        try:
            d = json.loads(f.read_text()).get("k2_sharegpt")
        except (OSError, ValueError):
            continue
        if d and "dram_bytes_per_launch" in d:
            best = (d["dram_bytes_per_launch"], f.name)
    return best if best else (None, None)


def graph_time(fn, dev, reps=10, use_graph=True):
    """Milliseconds per replay of fn captured as one CUDA graph (events on the stream);
    use_graph=False times eager calls (fn holds a collective)."""
    import torch
    if not use_graph:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cfg_full(args):
    from paper_2605_24832_b200.decode import DecodeConfig
    return DecodeConfig(**workload_spec(args.workload)["model"], page_size=args.page, max_batch=args.batch)


def workload_name(args):
    if args.workload == "tp30b":
        return "sdar30b-tp-attn-oproj-allreduce-unmask"
    base = "llada16b" if args.workload == "llada" else "sdar8b"
    return f"{base}-attn-unmask-{args.workload}"


def chunk_label(args):
    w = workload_spec(args.workload)
    return f"mixed{list(w['mixed'])}" if w["mixed"] else args.chunk


def run_e2e(args, dec, fwd, pool, world, dev):
    """Closed loop through StreamingDecoder.step: finished requests are replaced
    from a pool so the batch stays full; the timed region includes host planning,
    the H2D of the step metadata, the device step, the D2H of the commits and the
    host apply."""
    import torch
    import torch.distributed as dist
    batch = list(pool[0])
    spare = list(pool[1])
    n_steps = args.e2e_steps if args.e2e_steps is not None else max(args.steps, 20)

    def one():
        nonlocal batch
        summ = dec.step(batch, step_chunks(args, batch))
        fwd.next_version()
        done = [r for r in batch if r.finished]
        if done:
            batch = [r for r in batch if not r.finished]
            while len(batch) < args.batch and spare:
                batch.append(spare.pop())
        return sum(len(s.commits) for s in summ)

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    commits = 0
    h2d = d2h = 0
    for _ in range(n_steps):
        commits += one()
        h2d += dec.h2d_bytes
        d2h += dec.d2h_bytes
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    dec.release_all(batch)
    if world > 1:
        t = torch.tensor([el], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    return {"value": commits / el, "unit": "tokens/s", "h2d_bytes_per_step": h2d // n_steps,
            "d2h_bytes_per_step": d2h // n_steps, "steps": n_steps, "ms_per_step": el / n_steps * 1e3,
            "path": "StreamingDecoder.step (plan_batch -> H2D meta -> L x (K1,K2) -> K3 -> D2H -> apply_batch)"}


def run_device_loop(args, dec, world):
    """Fixed batch through DeviceLoop: plan, attention work list, L x
    (K1, K2, combine), K3 and apply as ONE CUDA graph on device-resident request
    state; per step the host copies back the plan and commit mask and replays the
    transitions on its Request objects.  No H2D per step (the state stays resident);
    D2H = the plan arrays + mask.  Timed on the host clock around whole steps."""
    import torch
    from paper_2605_24832_b200.device_loop import DeviceLoop
    from paper_2605_24832_b200.errors import ConfigError
    if world != 1 or args.workload == "tp30b":
        return None
    long_ctx = args.workload in ("longbench", "ctx4096")
    # the same batch and spare pool as run_e2e (fresh objects): the two e2e numbers
    # decode the same requests
    reqs = workload_requests(args, seed_offset=1)
    spare = workload_requests(args, seed_offset=2, n=16 if long_ctx else None)
    try:
        loop = DeviceLoop(dec, reqs, step_chunks(args, reqs), lookahead=True)
    except (ConfigError, RuntimeError) as e:
        dec.release_all(reqs)
        return {"unavailable": str(e)[:200]}
    n_steps = args.e2e_steps if args.e2e_steps is not None else max(args.steps, 20)
    h2d = 0

    def one():
        nonlocal h2d
        c = loop.step(summaries=False)
        for i in sorted(loop.free):  # continuous batching: refill finished positions
            if not spare:
                break
            loop.replace(i, spare.pop())
            h2d += sum(loop.D[k][0].numel() * loop.D[k].element_size() for k in loop.state_keys) + \
                loop.Dt.shape[1] * 4
        return c

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    h2d = 0
    t0 = time.perf_counter()
    commits = 0
    for _ in range(n_steps):
        commits += one()
    el = time.perf_counter() - t0
    loop.drain()
    d2h = sum(t.numel() * t.element_size() for t in loop.H.values())
    dec.release_all([r for r in loop.requests if not r.finished])
    return {"value": commits / el, "unit": "tokens/s", "steps": n_steps, "ms_per_step": el / n_steps * 1e3,
            "h2d_bytes_per_step": h2d // n_steps, "d2h_bytes_per_step": d2h,
            "batch": "closed loop: finished positions refilled from a spare pool (DeviceLoop.replace)",
            "path": "DeviceLoop.step, lookahead (one graph: device plan -> work plan -> L x (K1,K2,combine) -> "
                    "K3 -> device apply; D2H plan + mask; the next graph runs during the host apply)"}


if __name__ == "__main__":
    main()
