"""f3: the fused LM-head + unmask-partials kernel against a plain
PyTorch fp32 reference of the same op (logits = H W^T in fp32, then the
confidence-threshold rule of K3 on them).  The kernel accumulates in fp32 on the
tensor cores, so only the summation order differs from the reference."""

import numpy as np
import pytest
import torch

from paper_2605_24832_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,k,vocab,scale", [(300, 512, 5000, 0.06), (128, 256, 256, 0.2), (77, 4096, 2056, 0.02),
                                                (150, 200, 1000, 0.1), (513, 1024, 40000, 0.05),
                                                (1, 64, 700, 0.5)])
def test_lmhead_unmask_matches_fp32_reference(rows, k, vocab, scale):
    g = torch.Generator(device="cuda")
    g.manual_seed(rows + k + vocab)
    H = torch.randn(rows, k, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(vocab, k, device="cuda", generator=g) * scale).to(torch.bfloat16)
    part = ops.lmhead_unmask_partials(H, W, vocab_offset=0)
    n_vt = part.shape[1]
    cu_rows = torch.tensor([0, rows], dtype=torch.int32, device="cuda")
    res = ops.unmask_finalize(part, 1, rows, n_vt, cu_rows, 0.9)
    torch.cuda.synchronize()
    logits = H.double() @ W.double().T
    m = logits.max(dim=1).values
    s = torch.exp(logits - m[:, None]).sum(dim=1)
    conf_ref = (1.0 / s).cpu().numpy()
    conf = res.conf.cpu().numpy()[:rows]
    np.testing.assert_allclose(conf, conf_ref, rtol=2e-3, atol=1e-6)
    # argmax: exact unless the top two logits are within the fp32 accumulation noise
    top2 = torch.topk(logits, 2, dim=1).values
    clear = ((top2[:, 0] - top2[:, 1]) > 1e-3).cpu().numpy()
    tok = res.tokens.cpu().numpy()[:rows]
    ref_tok = logits.argmax(dim=1).cpu().numpy()
    assert np.array_equal(tok[clear], ref_tok[clear])
    # merged per row first (optimus_unmask_merge_splits): the same decisions
    mg = ops.lmhead_unmask_partials(H, W, merge=True)
    res2 = ops.unmask_finalize(mg, 1, rows, 1, cu_rows, 0.9)
    torch.cuda.synchronize()
    assert torch.equal(res2.tokens[:rows], res.tokens[:rows])
    np.testing.assert_allclose(res2.conf.cpu().numpy()[:rows], conf, rtol=1e-5)
    # the raw partials: per-tile max equals the reference tile max
    pm = part[:, :, 0].cpu().numpy()
    lg = logits.float().cpu().numpy()
    for t in range(n_vt):
        ref = lg[:, t * 256:(t + 1) * 256].max(axis=1)
        np.testing.assert_allclose(pm[:, t], ref, rtol=1e-4, atol=1e-4)


def test_lmhead_vocab_offset_and_sharded_merge():
    """Two vocabulary shards with offsets merge (n_outer = 2) to the unsharded result."""
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    rows, k, vocab = 190, 512, 3000
    H = torch.randn(rows, k, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(vocab, k, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    cu_rows = torch.tensor([0, 100, rows], dtype=torch.int32, device="cuda")
    full = ops.unmask_finalize(ops.lmhead_unmask_partials(H, W), 1, rows, ops._lib.call("optimus_lmhead_splits", vocab),
                               cu_rows, 0.9)
    half = vocab // 2
    pa = ops.lmhead_unmask_partials(H, W[:half].contiguous(), vocab_offset=0)
    pb = ops.lmhead_unmask_partials(H, W[half:].contiguous(), vocab_offset=half)
    assert pa.shape[1] == pb.shape[1]
    both = torch.stack([pa, pb])  # [n_outer][rows][splits][3]
    sh = ops.unmask_finalize(both, 2, rows, pa.shape[1], cu_rows, 0.9)
    torch.cuda.synchronize()
    assert torch.equal(full.tokens[:rows], sh.tokens[:rows])
    torch.testing.assert_close(full.conf[:rows], sh.conf[:rows], rtol=1e-5, atol=1e-7)
    assert torch.equal(full.commit_mask[:rows], sh.commit_mask[:rows])


def test_lmhead_unmask_commit_equals_unmask_commit_on_fp32_logits():
    """One-call f3 API == K3 (`unmask_commit`) on the fp32 logits of the same LM
    head, per request (progress rule included), away from the tau boundary."""
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    rows, k, vocab = 260, 1024, 4096
    H = torch.randn(rows, k, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(vocab, k, device="cuda", generator=g) * 0.08).to(torch.bfloat16)
    H[::3] *= 4  # sharper rows: a mix of committed and uncommitted positions
    cu = torch.tensor([0, 7, 40, 41, 120, 260], dtype=torch.int32, device="cuda")
    a = ops.lmhead_unmask_commit(H, W, cu, 0.9)
    logits = (H.float() @ W.float().T).contiguous()
    b = ops.unmask_commit(logits, cu, 0.9)
    torch.cuda.synchronize()
    conf = b.conf.cpu().numpy()[:rows]
    far = np.abs(conf - 0.9) > 1e-3
    assert far.sum() > rows // 2
    assert np.array_equal(a.commit_mask.cpu().numpy()[:rows][far], b.commit_mask.cpu().numpy()[:rows][far])
    assert 0 < int(a.commit_mask[:rows].sum()) < rows
    np.testing.assert_allclose(a.conf.cpu().numpy()[:rows], conf, rtol=2e-3, atol=1e-6)
