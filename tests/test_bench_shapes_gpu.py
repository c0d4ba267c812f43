"""Parity at exactly the shapes bench.py measures (every benchmarked
number must rest on kernels checked at that shape).

Each case builds the benchmark's own decoder (bench.build_decoder: the workload's
batch, lengths, chunk sizes, page size, heads, vocabulary, page tables and split
plan), runs its device step and checks it with bench.parity_check — the same
check the bench line reports under "parity":

* K1: slot mapping and the written K/V rows bit-exact (rule S / rule K);
* K2: the attention of the sampled requests (the longest ones + a seeded draw)
  against the fp32 CPU oracle, relative error <= 2e-3 (north_star tolerance);
* K3: the commit mask and argmax tokens of every window row exact (rows with
  |conf - tau| <= 1e-4 excluded; the recipe keeps them at 0.07 from tau).

Long-context cases keep the exact batch and lengths with fewer layers (every
layer runs the same kernels on its own cache).  The f3 case runs the fused LM
head at the ShareGPT step's 1,121 rows x 4,096 x 151,936 vocabulary against a
PyTorch fp32 reference of the same op.
"""

import argparse

import numpy as np
import pytest
import torch

import bench
from paper_2605_24832_b200.engine import plan_batch

pytestmark = pytest.mark.gpu


def _args(workload, batch, chunk=32, page=64, seed=0):
    return argparse.Namespace(workload=workload, batch=batch, chunk=chunk, page=page, seed=seed, steps=1,
                              warmup=1)


def _run(a, layers=None, plans=None, layer=0, n_sample=12, reqs=None):
    dev = torch.device("cuda")
    W = bench.build_decoder(a, dev, layers=layers, e2e_pools=False, reqs=reqs)
    reqs = W.reqs
    if plans is None:
        plans = plan_batch(reqs, bench.step_chunks(a, reqs), W.cfg.block_size, W.cfg.window_rule)
    dm = W.dec.prepare(reqs, plans)
    res = W.dec.device_step(dm)
    torch.cuda.synchronize()
    p = bench.parity_check(W, dm, res, layer=layer, n_sample=n_sample)
    print(a.workload, a.chunk, {k: v for k, v in p.items()})
    plan = dm.__dict__["attn_plan"]
    return p, dm.host, plan


def _assert_ok(p):
    assert p["k1_slots_exact"] and p["k1_rows_bit_exact"]
    assert p["k2_rel_err"] <= 2e-3, p["k2_rel_err"]
    assert p["k3_commit_mask_exact"] and p["k3_tokens_exact"]
    assert p["ok"]


def test_sharegpt_headline_step_36_layers():
    """configs[1]: b64, c32, page 64, ShareGPT lengths, 36-layer cache, last layer."""
    p, m, plan = _run(_args("sharegpt", 64), layer=35, n_sample=16)
    _assert_ok(p)
    assert m.n_req == 64 and m.n_rows == 1121 and p["k3_rows"] == 1121


@pytest.mark.parametrize("chunk", [1, 4, 8, 16])
def test_sharegpt_chunk_sweep(chunk):
    a = _args("sharegpt", 64, chunk=chunk)
    plans = None
    if chunk == 1:
        plans = bench.chunk1_plans(bench.workload_requests(a), 32)
    p, m, _ = _run(a, layers=2, plans=plans)
    _assert_ok(p)


def test_ctx4096_north_star_shape_split_kv():
    """north_star: 4K context, b64, c32 — the split-KV plan (combine groups)."""
    p, m, plan = _run(_args("ctx4096", 64), layers=2, n_sample=8)
    _assert_ok(p)
    assert plan.n_groups > 0  # split-KV groups merged by the combine kernel
    assert int(m.key_end.max()) >= 4096


def test_longbench_batch():
    """configs[2]: the benchmark's LongBench batch (prompts clipped to [4096, 16384]);
    the sample holds its longest requests."""
    p, m, plan = _run(_args("longbench", 64), layers=2, n_sample=8)
    _assert_ok(p)
    assert int(m.key_end.min()) >= 4096 and int(m.key_end.max()) > 8000


def test_longbench_at_the_16k_clip():
    """The clip's upper end: requests with 16,384-token prompts (up to 16,384 +
    output keys), split-KV pieces merged."""
    from paper_2605_24832_b200.synthetic import LONGBENCH, make_batch
    a = _args("longbench", 16)
    reqs = make_batch(5, 16, 32, lengths=LONGBENCH, q=bench.Q_LONGBENCH_DENSE, fixed_prompt=16384)
    p, m, plan = _run(a, layers=2, n_sample=6, reqs=reqs)
    _assert_ok(p)
    assert int(m.key_end.max()) > 16384
    assert plan.n_groups > 0


def test_llada_mixed_chunks_157k_vocab():
    """configs[3]: 16q/4kv, batch 128, mixed per-request chunks 8..32, K3 at V = 157,184."""
    a = _args("llada", 128)
    p, m, _ = _run(a, layers=2)
    _assert_ok(p)
    chunks = set(bench.step_chunks(a, list(range(128))))
    assert chunks == {8, 16, 24, 32}


def test_tp30b_group_of_8_two_query_tiles():
    """configs[5] at N = 1: 32q/4kv (G = 8), chunk 32 -> 256 query rows per
    (request, KV head), i.e. two M = 128 tiles."""
    p, m, plan = _run(_args("tp30b", 64), layers=2)
    _assert_ok(p)
    counts = np.diff(m.cu_seqlens)
    assert (counts * 8 > 128).any()


def test_lmhead_fused_at_sharegpt_step_shape():
    """f3 at 1,121 rows x 4,096 hidden x 151,936 vocab (the ShareGPT step's window
    rows through the SDAR-8B LM head) against cuBLAS fp32 logits + the same rule."""
    from paper_2605_24832_b200 import ops
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    rows, k, vocab = 1121, 4096, 151936
    H = torch.randn(rows, k, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(vocab, k, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
    H[::2] *= 3.0  # a mix of confident and unconfident rows
    cu = torch.arange(0, rows + 1, 17, dtype=torch.int32, device="cuda")
    cu = torch.cat([cu, torch.tensor([rows], dtype=torch.int32, device="cuda")]) if cu[-1] != rows else cu
    a = ops.lmhead_unmask_commit(H, W, cu, 0.9)
    torch.backends.cuda.matmul.allow_tf32 = False
    logits = H.float() @ W.float().T
    m = logits.max(dim=1).values
    s = torch.exp(logits - m[:, None]).sum(dim=1)
    conf_ref = (1.0 / s).cpu().numpy()
    top2 = torch.topk(logits, 2, dim=1).values
    clear = ((top2[:, 0] - top2[:, 1]) > 1e-2).cpu().numpy()
    ref_tok = logits.argmax(dim=1).cpu().numpy()
    torch.cuda.synchronize()
    conf = a.conf.cpu().numpy()[:rows]
    np.testing.assert_allclose(conf, conf_ref, rtol=2e-3, atol=1e-6)
    tok = a.tokens.cpu().numpy()[:rows]
    assert clear.mean() > 0.9
    assert np.array_equal(tok[clear], ref_tok[clear])
    far = np.abs(conf_ref - 0.9) > 2e-3
    b = ops.unmask_commit(logits.contiguous(), cu, 0.9)
    torch.cuda.synchronize()
    assert np.array_equal(a.commit_mask.cpu().numpy()[:rows][far], b.commit_mask.cpu().numpy()[:rows][far])
