"""BASELINE config 1 end to end: the tiny random-init SDAR-style dLLM decoding 4
requests through the B200 path (K1/K2 inside a real forward, LM head on window
rows, K3 unmask), checked step by step against the numpy oracle of the same model
(oracle/tiny_model.py), teacher-forced on the GPU's committed tokens.

Tolerances: logits within 2e-3 relative (max-norm per step); argmax tokens equal
where the top-2 logit gap exceeds 1e-2; commit masks equal where |conf - 0.9| > 0.02.
"""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import numeric as on
from oracle.tiny_model import TinyOracle
from paper_2605_24832_b200 import engine as pe
from paper_2605_24832_b200.core import Request
from paper_2605_24832_b200.decode import StreamingDecoder
from paper_2605_24832_b200.tiny_model import TinyConfig, TinyDLLM, tiny_weights

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kv_heads", [4, 2])
def test_tiny_dllm_decode_matches_oracle(kv_heads):
    cfg = TinyConfig(kv_heads=kv_heads, seed=kv_heads)
    block, chunk = 32, 8
    dcfg = cfg.decode_config(max_batch=4, num_pages=256, max_pages_per_req=16, max_output_tokens=256)
    model = TinyDLLM(cfg, max_slots=4, max_out=256)
    dec = StreamingDecoder(dcfg, model)
    rng = np.random.default_rng(kv_heads)
    reqs, prompts = [], []
    for i in range(4):
        p, o = int(rng.integers(5, 41)), int(rng.integers(64, 97))
        reqs.append(Request(id=i, arrival_time=0.0, prompt_tokens=p, output_tokens=o))
        prompts.append(rng.integers(0, cfg.vocab - 1, p))
    oracle = TinyOracle(cfg, tiny_weights(cfg))
    model.prefill(dec, reqs, prompts)
    for r, ids in zip(reqs, prompts):
        oracle.prefill(r.id, ids, r.output_tokens)
    committed_tok = {r.id: {} for r in reqs}
    cap = {}
    orig_logits, orig_commit = model.logits, model.on_commit

    def logits_hook(dm):
        out = orig_logits(dm)
        cap["logits"] = out[0].detach().float().cpu().numpy().copy()
        return out

    def commit_hook(dm, mask, tokens):
        cap["mask"], cap["tok"] = mask.copy(), tokens.copy()
        orig_commit(dm, mask, tokens)

    model.logits, model.on_commit = logits_hook, commit_hook
    steps = errs = checked = extra_commits = 0
    while not all(r.finished for r in reqs):
        active = [r for r in reqs if not r.finished]
        plans = pe.plan_batch(active, chunk, block)
        snaps = [SimpleNamespace(id=r.id, prompt_tokens=r.prompt_tokens, output_tokens=r.output_tokens,
                                 states=np.array(r.states, copy=True)) for r in active]
        dec.step(active, chunk)
        L_ref = oracle.step(snaps, plans, lambda rq, p: committed_tok[rq.id][p], block)
        L = cap["logits"][: L_ref.shape[0]]
        rel = np.abs(L - L_ref).max() / np.abs(L_ref).max()
        assert rel < 2e-3, (steps, rel)
        cu = np.concatenate([[0], np.cumsum([len(p.window) for p in plans])])
        c_ref, t_ref, conf_ref = on.unmask(L_ref, cu, 0.9)
        srt = np.sort(L_ref, axis=1)
        clear_tok = (srt[:, -1] - srt[:, -2]) > 1e-2
        assert np.array_equal(cap["tok"][: len(t_ref)][clear_tok], t_ref[clear_tok])
        clear = np.abs(conf_ref - 0.9) > 0.02
        assert np.array_equal(cap["mask"][: len(c_ref)][clear], c_ref[clear])
        checked += int(clear.sum())
        # teacher forcing: record the GPU's committed tokens for the next steps' kv rows
        k = 0
        for r, plan in zip(active, plans):
            for j, p in enumerate(plan.window):
                if cap["mask"][k]:
                    committed_tok[r.id][p] = int(cap["tok"][k])
                    extra_commits += int(j > 0)
                k += 1
        steps += 1
        assert steps < 200
    assert checked > 100
    assert extra_commits > 0  # some rows beyond the progress rule clear tau


@pytest.mark.parametrize("lm_head", ["torch", "f3"])
def test_tiny_dllm_device_loop_matches_oracle(lm_head):
    """BASELINE config 1 through the graph-captured DeviceLoop: the tiny model's
    forward runs from the device plan over the loop's capacity buffers (TinyDLLM loop
    hooks), committed token ids stay on the device (K3 writes them), and with
    lm_head="f3" the LM head is the fused LM-head + unmask kernel.  Checked step by
    step against the numpy oracle model, teacher-forced on the loop's own commits.
    Tolerances as test_tiny_dllm_decode_matches_oracle for the fp32 head; the f3 head
    rounds its operands to bf16 (|logit| ~ 16 -> ~0.06 logit error), so its token and
    commit checks use a 0.5 top-2 gap and a 0.05 confidence margin."""
    from paper_2605_24832_b200.device_loop import DeviceLoop

    cfg = TinyConfig(kv_heads=2, seed=7)
    block, chunk = 32, 8
    dcfg = cfg.decode_config(max_batch=4, num_pages=256, max_pages_per_req=16, max_output_tokens=256)
    model = TinyDLLM(cfg, max_slots=4, max_out=256, lm_head=lm_head)
    dec = StreamingDecoder(dcfg, model)
    rng = np.random.default_rng(17)
    reqs, prompts = [], []
    for i in range(4):
        p, o = int(rng.integers(5, 41)), int(rng.integers(64, 97))
        reqs.append(Request(id=i, arrival_time=0.0, prompt_tokens=p, output_tokens=o))
        prompts.append(rng.integers(0, cfg.vocab - 1, p))
    oracle = TinyOracle(cfg, tiny_weights(cfg))
    model.prefill(dec, reqs, prompts)
    for r, ids in zip(reqs, prompts):
        oracle.prefill(r.id, ids, r.output_tokens)
    loop = DeviceLoop(dec, reqs, chunk)
    gap, margin = (1e-2, 0.02) if lm_head == "torch" else (0.5, 0.05)
    committed_tok = {r.id: {} for r in reqs}
    steps = checked = 0
    while not all(r.finished for r in reqs):
        active = [r for r in reqs if not r.finished]
        plans = pe.plan_batch(active, chunk, block)
        snaps = [SimpleNamespace(id=r.id, prompt_tokens=r.prompt_tokens, output_tokens=r.output_tokens,
                                 states=np.array(r.states, copy=True)) for r in active]
        summ = loop.step()
        n_rows = sum(len(p.window) for p in plans)
        mask = loop.res.commit_mask[:n_rows].cpu().numpy().astype(bool)
        tok = loop.res.tokens[:n_rows].cpu().numpy()
        L_ref = oracle.step(snaps, plans, lambda rq, p: committed_tok[rq.id][p], block)
        cu = np.concatenate([[0], np.cumsum([len(p.window) for p in plans])])
        c_ref, t_ref, conf_ref = on.unmask(L_ref, cu, 0.9)
        srt = np.sort(L_ref, axis=1)
        clear_tok = (srt[:, -1] - srt[:, -2]) > gap
        assert np.array_equal(tok[clear_tok], t_ref[clear_tok]), steps
        clear = np.abs(conf_ref - 0.9) > margin
        assert np.array_equal(mask[clear], c_ref[clear]), steps
        checked += int(clear.sum())
        k = 0
        by_id = {r.id: s for r, s in zip(loop.requests, summ)}
        for r, plan in zip(active, plans):
            got = set()
            for p in plan.window:
                if mask[k]:
                    committed_tok[r.id][p] = int(tok[k])
                    got.add(p)
                k += 1
            assert got == set(by_id[r.id].commits), (steps, r.id)
        steps += 1
        assert steps < 200
    assert checked > 100
    # the device token buffer holds every committed token the host saw
    lt = model.loop_tok.cpu().numpy()
    for i, r in enumerate(loop.requests):
        for p, t in committed_tok[r.id].items():
            assert lt[i, p] == t
