import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.synthetic import SyntheticForward
import paper_2605_24832_b200.native_step as ns
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
T = {}
def tic(k, t0):
    T.setdefault(k, []).append(time.perf_counter() - t0)
    return time.perf_counter()
for it in range(120):
    t = time.perf_counter()
    dm = nat.plan(batch, 32); t = tic("plan", t)
    fwd.fill_row_src(dm); t = tic("rowsrc", t)
    nat.upload(dm); t = tic("upload", t)
    res = dec.device_step(dm); t = tic("enqueue", t)
    torch.cuda.current_stream().synchronize(); t = tic("gpu_wait", t)
    counts = nat.fetch_and_apply(dm, res); t = tic("d2h_apply", t)
    for r in batch:
        if r.finished: nat.release(r)
    batch = [r for r in batch if not r.finished]
    while len(batch) < 64 and spare: batch.append(spare.pop())
    t = tic("release", t)
    fwd.next_version()
print({k: round(1e3 * float(np.mean(v[20:])), 3) for k, v in T.items()})
# inside plan
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for it in range(100):
    dm = nat.plan(batch, 32)
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(12)
t = time.perf_counter()
for it in range(100): dm = nat.plan(batch, 32)
print("plan only ms", (time.perf_counter() - t) * 10)
