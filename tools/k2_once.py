"""Run the bench workload's K2 a few times (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2605_24832_b200 import ops
from paper_2605_24832_b200.decode import DecodeConfig, StreamingDecoder
from paper_2605_24832_b200.engine import plan_batch
from paper_2605_24832_b200.synthetic import SyntheticForward

class A: pass
a = A(); a.workload = sys.argv[1] if len(sys.argv) > 1 else "sharegpt"; a.chunk = 32; a.page = 64; a.batch = 64; a.seed = 0; a.steps = 1
dev = torch.device("cuda")
reqs = bench.workload_requests(a)
cfg = DecodeConfig(num_layers=2, page_size=a.page, max_batch=a.batch, num_pages=bench.pages_needed(reqs, a.page) + 64,
                   max_pages_per_req=max((r.prompt_tokens + r.output_tokens + a.page - 1) // a.page for r in reqs) + 1)
fwd = SyntheticForward(cfg, a.batch * a.chunk, a.batch, device=dev)
dec = StreamingDecoder(cfg, fwd, device=dev)
for l in range(cfg.num_layers):
    dec.cache.k[l].normal_(); dec.cache.v[l].normal_()
dm = dec.prepare(reqs, plan_batch(reqs, a.chunk, cfg.block_size, cfg.window_rule))
for _ in range(3):
    dec.device_step(dm)
torch.cuda.synchronize()
print("ok")
