"""e2e tokens/s of the graph-captured device loop vs the host native step on the
same fixed batch (ShareGPT workload, SDAR-8B attention, 36 layers), diagnostics."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.device_loop import DeviceLoop
from paper_2605_24832_b200.synthetic import SyntheticForward


def setup():
    class A:
        pass
    a = A()
    a.workload, a.chunk, a.page, a.batch, a.seed, a.steps = "sharegpt", 32, 64, 64, 0, 1
    reqs = bench.workload_requests(a, seed_offset=1)
    P = 64
    cfg = DecodeConfig(page_size=P, max_batch=64, num_pages=bench.pages_needed(reqs, P) + 256,
                       max_pages_per_req=max((r.prompt_tokens + r.output_tokens + P - 1) // P for r in reqs) + 2)
    dev = torch.device("cuda")
    fwd = SyntheticForward(cfg, 64 * 32, 64, device=dev)
    dec = StreamingDecoder(cfg, fwd, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for l in range(cfg.num_layers):  # KV content: random bf16 (uninitialised memory can hold inf/NaN)
        dec.cache.k[l].normal_(generator=g)
        dec.cache.v[l].normal_(generator=g)
    return reqs, dec


def profile_loop(steps=2):
    """The device loop's kernels for `steps` graph replays, bracketed by the CUDA
    profiler API (ncu --profile-from-start off)."""
    reqs, dec = setup()
    loop = DeviceLoop(dec, reqs, 32)
    for _ in range(3):
        loop.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(steps):
        loop.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


def main():
    N = 60
    reqs, dec = setup()
    for _ in range(3):
        dec.step([r for r in reqs if not r.finished], 32)
    torch.cuda.synchronize()
    t = time.perf_counter()
    c = 0
    for _ in range(N):
        c += sum(len(s.commits) for s in dec.step([r for r in reqs if not r.finished], 32))
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print(f"host native step : {c / el:9.0f} tok/s  {el / N * 1e3:.3f} ms/step")
    reqs, dec = setup()
    loop = DeviceLoop(dec, reqs, 32)
    for _ in range(3):
        loop.step()
    torch.cuda.synchronize()
    t = time.perf_counter()
    c = 0
    for _ in range(N):
        c += sum(len(s.commits) for s in loop.step())
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print(f"device loop graph: {c / el:9.0f} tok/s  {el / N * 1e3:.3f} ms/step, replay+sync {loop.t_device / (N + 3) * 1e3:.3f} ms")
    loop.t_device = 0.0
    t0 = time.perf_counter()
    for _ in range(20):
        loop.step()
    el = time.perf_counter() - t0
    print(f"full step {el / 20 * 1e3:.3f} ms, of which replay+sync {loop.t_device / 20 * 1e3:.3f} ms")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "profile":
        profile_loop()
    else:
        main()
