"""f3: fused LM head + unmask partials vs cuBLAS GEMM (bf16 logits) + K3, at the
ShareGPT step's window rows (SDAR-8B: hidden 4096, vocab 151,936).  Prints one JSON
line; times are CUDA-event medians over CUDA-graph replays.  The fused kernel
should beat the unfused pair once its GEMM is within the logits traffic of cuBLAS."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2605_24832_b200 import _lib, ops


def graph_us(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1121
    k, vocab = 4096, 151936
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    H = torch.randn(rows, k, device=dev, generator=g).to(torch.bfloat16)
    W = (torch.randn(vocab, k, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    # 64 requests' window rows (the ShareGPT step's layout)
    cu = torch.from_numpy(np.linspace(0, rows, 65).astype(np.int32)).to(dev)
    n_vt = int(_lib.call("optimus_lmhead_splits", vocab))
    part = torch.empty((rows, n_vt, 3), dtype=torch.float32, device=dev)
    logits = torch.empty((rows, vocab), dtype=torch.bfloat16, device=dev)
    n_vs = ops.unmask_splits(rows, vocab)
    part2 = torch.empty((rows, n_vs, 3), dtype=torch.float32, device=dev)

    merged = torch.empty((rows, 1, 3), dtype=torch.float32, device=dev)

    def fused():
        ops.lmhead_unmask_partials(H, W, part=part, merge=True, merged=merged)
        ops.unmask_finalize(merged, 1, rows, 1, cu, 0.9)

    def fused_gemm_only():
        ops.lmhead_unmask_partials(H, W, part=part)

    def unfused():
        torch.matmul(H, W.T, out=logits)
        ops.unmask_partials(logits, None, rows, n_vs, part=part2)
        ops.unmask_finalize(part2, 1, rows, n_vs, cu, 0.9)

    def gemm_only():
        torch.matmul(H, W.T, out=logits)

    t = {name: graph_us(fn) for name, fn in (("fused", fused), ("fused_kernel", fused_gemm_only),
                                              ("cublas_plus_k3", unfused), ("cublas_gemm", gemm_only))}
    flops = 2.0 * rows * k * vocab
    a = ops.unmask_finalize(ops.lmhead_unmask_partials(H, W, merge=True), 1, rows, 1, cu, 0.9)
    torch.matmul(H, W.T, out=logits)
    b = ops.unmask_commit(logits, cu, 0.9)
    torch.cuda.synchronize()
    agree = float((a.tokens[:rows] == b.tokens[:rows]).float().mean())
    peak = 1590.0
    line = {"rows": rows, "k": k, "vocab": vocab, "us": t,
            "tflops": {n: flops / (v * 1e-6) / 1e12 for n, v in t.items() if n in ("fused_kernel", "cublas_gemm")},
            "fused_kernel_frac_of_bf16_fallback_peak": flops / (t["fused_kernel"] * 1e-6) / 1e12 / peak,
            "logits_bytes_avoided": rows * vocab * 2 * 2, "argmax_agreement_vs_bf16_logits": agree}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
