"""Multi-GPU decomposition checked on CPU with torch.distributed (gloo, world 2):
KV-head sharding of attention and the vocab-sharded unmask whose 12-byte partials
are all-gathered and merged in a fixed order on every rank (parallel.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numeric as on
from paper_2605_24832_b200.parallel import shard_for


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shards_partition_heads_and_vocab():
    for world in (1, 2, 4, 8):
        shards = [shard_for(r, world, 32, 8, 151936) for r in range(world)]
        assert [h for sh in shards for h in range(*sh.kv_heads)] == list(range(8))
        assert [h for sh in shards for h in range(*sh.q_heads)] == list(range(32))
        assert shards[0].vocab[0] == 0 and shards[-1].vocab[1] == 151936
        for a, b in zip(shards, shards[1:]):
            assert a.vocab[1] == b.vocab[0]
    with pytest.raises(ValueError):
        shard_for(0, 3, 32, 8, 100)


def _unmask_worker(rank, world, port, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(seed)
    n, vocab = 40, 4000
    toks = rng.integers(0, vocab, n)
    confs = rng.choice([0.97, 0.8, 0.5], n)
    logits = on.peaked_logits(rng, n, vocab, toks, confs)  # identical on every rank
    sh = shard_for(rank, world, 8, 8, vocab)
    m, s, i = on.unmask_partial_ref(logits[:, sh.vocab[0]:sh.vocab[1]], sh.vocab[0])
    rec = torch.from_numpy(np.stack([m, s, i.astype(np.float64)], axis=1))
    gathered = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(gathered, rec)
    parts = [(g[:, 0].numpy(), g[:, 1].numpy(), g[:, 2].numpy().astype(np.int64)) for g in gathered]
    M, S, I = on.unmask_merge_ref(parts)
    out[rank] = (I.copy(), (1.0 / S).copy())
    dist.destroy_process_group()


def test_vocab_sharded_unmask_merge_matches_full_vocab():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_unmask_worker, args=(world, port, 7, out), nprocs=world, join=True)
    rng = np.random.default_rng(7)
    n, vocab = 40, 4000
    toks = rng.integers(0, vocab, n)
    confs = rng.choice([0.97, 0.8, 0.5], n)
    logits = on.peaked_logits(rng, n, vocab, toks, confs)
    _, t_ref, c_ref = on.unmask(logits, np.array([0, n]), 0.9)
    i0, c0 = out[0]
    i1, c1 = out[1]
    assert np.array_equal(i0, i1) and np.array_equal(c0, c1)  # bitwise identical on all ranks
    assert np.array_equal(i0, t_ref)
    np.testing.assert_allclose(c0, c_ref, rtol=1e-12)


def _attn_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    hq, hkv, d, page, block = 8, 4, 16, 8, 8
    n_pages = 12
    k = rng.standard_normal((n_pages, hkv, page, d)).astype(np.float32)
    v = rng.standard_normal((n_pages, hkv, page, d)).astype(np.float32)
    q = rng.standard_normal((5, hq, d)).astype(np.float32)
    bt = np.arange(n_pages, dtype=np.int32)[None, :]
    states = np.array([2, 2, 0, 1, 0, 0, 0, 0], dtype=np.int8)
    vis = [on.visible_outputs(states, [3, 2, 4, 5, 6])]
    sh = shard_for(rank, world, hq, hkv, 100)
    lo, hi = sh.kv_heads
    qlo, qhi = sh.q_heads
    o = on.paged_attention(q[:, qlo:qhi], k[:, lo:hi], v[:, lo:hi], np.array([0, 5]),
                           np.array([3, 2, 4, 5, 6]), np.array([20]), vis, bt, block, page)
    t = torch.from_numpy(o)
    g = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(g, t)
    out[rank] = torch.cat(g, dim=1).numpy()
    dist.destroy_process_group()


def test_kv_head_sharded_attention_concatenates_to_full():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_attn_worker, args=(world, port, out), nprocs=world, join=True)
    rng = np.random.default_rng(3)
    hq, hkv, d, page, block = 8, 4, 16, 8, 8
    n_pages = 12
    k = rng.standard_normal((n_pages, hkv, page, d)).astype(np.float32)
    v = rng.standard_normal((n_pages, hkv, page, d)).astype(np.float32)
    q = rng.standard_normal((5, hq, d)).astype(np.float32)
    bt = np.arange(n_pages, dtype=np.int32)[None, :]
    states = np.array([2, 2, 0, 1, 0, 0, 0, 0], dtype=np.int8)
    vis = [on.visible_outputs(states, [3, 2, 4, 5, 6])]
    full = on.paged_attention(q, k, v, np.array([0, 5]), np.array([3, 2, 4, 5, 6]), np.array([20]),
                              vis, bt, block, page)
    np.testing.assert_allclose(out[0], full, rtol=1e-6, atol=1e-6)
    np.testing.assert_array_equal(out[0], out[1])
