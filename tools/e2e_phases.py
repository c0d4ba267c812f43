"""Per-phase host timing of the native decode step (diagnostics)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.synthetic import SyntheticForward

class A: pass
a = A(); a.workload = "sharegpt"; a.chunk = 32; a.page = 64; a.batch = 64; a.seed = 0; a.steps = 1
dev = torch.device("cuda")
pool = [bench.workload_requests(a, seed_offset=k + 1) for k in range(2)]
P = a.page
cfg = DecodeConfig(page_size=P, max_batch=64, num_pages=sum(bench.pages_needed(b, P) for b in pool) + 64,
                   max_pages_per_req=max((r.prompt_tokens + r.output_tokens + P - 1) // P for b in pool for r in b) + 1)
fwd = SyntheticForward(cfg, 64 * 32, 64, device=dev)
dec = StreamingDecoder(cfg, fwd, device=dev)
nat = dec.native()
batch = list(pool[0]); spare = list(pool[1])
T = {k: [] for k in ("plan", "rowsrc", "upload", "layers", "unmask", "sync_apply", "summ", "release")}
for it in range(40):
    t0 = time.perf_counter()
    dm = nat.plan(batch, 32); t1 = time.perf_counter()
    fwd.fill_row_src(dm); t2 = time.perf_counter()
    nat.upload(dm); t3 = time.perf_counter()
    dec.run_layers(dm); t4 = time.perf_counter()
    res = dec.run_unmask(dm); t5 = time.perf_counter()
    counts = nat.fetch_and_apply(dm, res); t6 = time.perf_counter()
    mask = nat.mask_host.numpy()[:dm.host.n_rows].astype(bool)
    t7 = time.perf_counter()
    for r in batch:
        if r.finished:
            nat.release(r)
    batch = [r for r in batch if not r.finished]
    while len(batch) < 64 and spare:
        batch.append(spare.pop())
    t8 = time.perf_counter()
    fwd.next_version()
    if it >= 5:
        for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6, t8 - t7)):
            T[k].append(v * 1e3)
print({k: round(float(np.mean(v)), 3) for k, v in T.items()}, "total", round(sum(float(np.mean(v)) for v in T.values()), 3))
import ctypes as C
from paper_2605_24832_b200 import _lib
A = nat.arena; L = nat.lib
n = len(batch)
bs = nat.bs
import types
t = time.perf_counter()
for _ in range(20):
    nat.plan(batch, 32)
print("nat.plan (python + host_plan + attn_plan) ms", (time.perf_counter() - t) / 20 * 1e3)
cu = A.h("cu_seqlens", n + 1).copy(); ke = A.h("key_end", n).copy()
t = time.perf_counter()
for _ in range(50):
    ng, npart = C.c_int(0), C.c_int(0)
    L.optimus_attn_plan(n, cu.ctypes.data, ke.ctypes.data, 32, 8, nat.grid, 4, 64, A.hptr("work"), nat.max_work,
                        A.hptr("cta_off"), A.hptr("groups"), nat.max_groups, C.byref(ng), C.byref(npart))
print("attn_plan C++ ms", (time.perf_counter() - t) / 50 * 1e3)
