"""Tiny random-init SDAR-style diffusion LM around the B200 path (BASELINE config 1).

2 layers, 4 query heads (4 or 2 KV heads), head_dim 64, hidden 256, vocab 1024,
block 32, chunk 8, page 16.  One decode step per ``StreamingDecoder.step``:

    ids      kv rows -> their committed token, window rows -> MASK
    x        = embed(ids)
    per layer: h = rmsnorm(x); q,k,v = h Wqkv; RoPE(q, k) at absolute positions
               K1 kv_append(k, v) ; K2 paged attention ; x += attn Wo
               h = rmsnorm(x) ; x += (silu(h Wg) * h Wu) Wd
    logits   = rmsnorm(x[window rows]) Wlm * logit_scale        (LM head on window rows only)
    K3       unmask at tau -> commits + argmax tokens (recorded as the committed tokens)

Activations and GEMMs are fp32 (cuBLAS, TF32 off); only what the kernels consume
is bf16 (q, k, v; attention output), exactly as the oracle model in
``oracle/tiny_model.py`` rounds it.  Prompts are prefilled (out of the path) with
causal attention and their KV appended through K1 at negative output positions
(absolute = prompt + position).  Weights are random N(0, 0.02) from a seed; the
LM head is scaled so that some window rows clear the 0.9 threshold.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import ops
from .decode import DecodeConfig, Forward


@dataclass(frozen=True)
class TinyConfig:
    vocab: int = 1024
    hidden: int = 256
    layers: int = 2
    heads: int = 4
    kv_heads: int = 4
    head_dim: int = 64
    ffn: int = 512
    rope_theta: float = 10000.0
    logit_scale: float = 50.0
    seed: int = 0

    @property
    def mask_id(self) -> int:
        return self.vocab - 1

    def decode_config(self, **kw) -> DecodeConfig:
        base = dict(num_layers=self.layers, num_q_heads=self.heads, num_kv_heads=self.kv_heads,
                    head_dim=self.head_dim, vocab=self.vocab, block_size=32, page_size=16,
                    logits_dtype=torch.float32)
        base.update(kw)
        return DecodeConfig(**base)


def tiny_weights(cfg: TinyConfig) -> dict:
    """Seeded fp32 numpy weights (shared by the B200 model and the oracle)."""
    rng = np.random.default_rng(cfg.seed)
    H, d = cfg.hidden, cfg.head_dim
    n_qkv = (cfg.heads + 2 * cfg.kv_heads) * d
    w = {"emb": rng.normal(0, 1.0, (cfg.vocab, H)).astype(np.float32),
         "ln_f": np.ones(H, np.float32),
         "lm": rng.normal(0, 0.02, (H, cfg.vocab)).astype(np.float32)}
    for l in range(cfg.layers):
        w[f"ln1.{l}"] = np.ones(H, np.float32)
        w[f"ln2.{l}"] = np.ones(H, np.float32)
        w[f"qkv.{l}"] = rng.normal(0, 0.02 * 4, (H, n_qkv)).astype(np.float32)
        w[f"o.{l}"] = rng.normal(0, 0.02, (cfg.heads * d, H)).astype(np.float32)
        w[f"g.{l}"] = rng.normal(0, 0.02, (H, cfg.ffn)).astype(np.float32)
        w[f"u.{l}"] = rng.normal(0, 0.02, (H, cfg.ffn)).astype(np.float32)
        w[f"d.{l}"] = rng.normal(0, 0.02, (cfg.ffn, H)).astype(np.float32)
    return w


def rope_tables(positions: torch.Tensor, d: int, theta: float):
    inv = 1.0 / (theta ** (torch.arange(0, d, 2, device=positions.device, dtype=torch.float32) / d))
    ang = positions.to(torch.float32)[:, None] * inv[None, :]
    return torch.cos(ang), torch.sin(ang)


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [n, heads, d] (fp32), rotate-half convention."""
    x1, x2 = x[..., ::2], x[..., 1::2]
    c, s = cos[:, None, :], sin[:, None, :]
    out = torch.empty_like(x)
    out[..., ::2] = x1 * c - x2 * s
    out[..., 1::2] = x1 * s + x2 * c
    return out


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


class TinyDLLM(Forward):
    """The tiny dLLM as the decoder's Forward; keeps each slot's committed token ids.

    It also runs inside ``DeviceLoop`` (``loop_model``): the loop hooks below compute
    the same forward over the loop's capacity-sized token and row buffers from the
    device plan (graph-capturable, no host round trip), with the committed token ids
    kept on the device (written by K3's finalize).  ``lm_head="f3"`` makes the loop's
    LM head the fused LM-head + unmask kernel (optimus_lmhead_unmask_partials, bf16
    operands, logits never written) instead of an fp32 GEMM followed by K3."""

    needs_tokens = True
    loop_model = True

    def __init__(self, cfg: TinyConfig, max_slots: int, max_out: int, device="cuda", lm_head: str = "torch"):
        torch.backends.cuda.matmul.allow_tf32 = False
        if lm_head not in ("torch", "f3"):
            raise ValueError(f"lm_head must be 'torch' or 'f3', got {lm_head!r}")
        self.cfg = cfg
        self.device = torch.device(device)
        self.w = {k: torch.from_numpy(v).to(self.device) for k, v in tiny_weights(cfg).items()}
        self.tokens = np.full((max_slots, max_out), cfg.mask_id, dtype=np.int64)  # committed ids
        self.max_out = max_out
        self.lm_head = lm_head
        self.prompt_ids = {}
        self.x = None

    # -------------------------------------------------------------- prefill
    def prefill(self, decoder, requests, prompt_ids) -> None:
        """Causal prefill of every prompt (outside the decode path): writes each
        prompt's K/V into the pages through K1 at output positions -P..-1."""
        cfg = self.cfg
        d, hq, hkv = cfg.head_dim, cfg.heads, cfg.kv_heads
        for req, ids in zip(requests, prompt_ids):
            slot = decoder.tables.slot(req.id)
            if slot is None:
                slot = decoder.admit(req)
            self.prompt_ids[req.id] = np.asarray(ids)
            n = len(ids)
            x = self.w["emb"][torch.as_tensor(ids, device=self.device)]
            pos = torch.arange(n, device=self.device)
            cos, sin = rope_tables(pos, d, cfg.rope_theta)
            bt = torch.from_numpy(decoder.tables.table[slot:slot + 1]).to(self.device)
            tok_req = torch.zeros(n, dtype=torch.int32, device=self.device)
            tok_pos = (pos - n).to(torch.int32)
            prompt_len = torch.tensor([n], dtype=torch.int32, device=self.device)
            for l in range(cfg.layers):
                h = rmsnorm(x, self.w[f"ln1.{l}"])
                qkv = (h @ self.w[f"qkv.{l}"]).view(n, hq + 2 * hkv, d)
                q = apply_rope(qkv[:, :hq], cos, sin).to(torch.bfloat16)
                k = apply_rope(qkv[:, hq:hq + hkv], cos, sin).to(torch.bfloat16)
                v = qkv[:, hq + hkv:].to(torch.bfloat16)
                kc, vc = decoder.cache.layer(l)
                ops.kv_append(k.contiguous(), v.contiguous(), tok_req, tok_pos, prompt_len, bt, kc, vc)
                att = F.scaled_dot_product_attention(
                    q.float().transpose(0, 1), k.float().repeat_interleave(hq // hkv, 1).transpose(0, 1),
                    v.float().repeat_interleave(hq // hkv, 1).transpose(0, 1), is_causal=True)
                att = att.transpose(0, 1).to(torch.bfloat16).float().reshape(n, hq * d)
                x = x + att @ self.w[f"o.{l}"]
                h = rmsnorm(x, self.w[f"ln2.{l}"])
                x = x + (F.silu(h @ self.w[f"g.{l}"]) * (h @ self.w[f"u.{l}"])) @ self.w[f"d.{l}"]

    # -------------------------------------------------------------- decode step
    def begin_step(self, dm) -> None:
        cfg = self.cfg
        m = dm.host
        reqs = dm.__dict__["requests"]
        slots = dm.__dict__["slots"]
        ids = np.full(m.n_tok, cfg.mask_id, dtype=np.int64)
        nwin = m.cu_rows[1:] - m.cu_rows[:-1]
        for r in range(m.n_req):
            t0, t1 = int(m.cu_seqlens[r]), int(m.cu_seqlens[r + 1])
            nkv = (t1 - t0) - int(nwin[r])
            if nkv:
                ids[t0:t0 + nkv] = self.tokens[slots[r], m.tok_pos[t0:t0 + nkv]]
        pos_abs = np.asarray(m.prompt_len)[np.repeat(np.arange(m.n_req), m.cu_seqlens[1:] - m.cu_seqlens[:-1])] \
            + np.asarray(m.tok_pos[: m.n_tok])
        self.x = self.w["emb"][torch.as_tensor(ids, device=self.device)]
        self.cos, self.sin = rope_tables(torch.as_tensor(pos_abs, device=self.device), cfg.head_dim,
                                         cfg.rope_theta)

    def qkv(self, layer: int, dm):
        cfg = self.cfg
        n = dm.host.n_tok
        d, hq, hkv = cfg.head_dim, cfg.heads, cfg.kv_heads
        h = rmsnorm(self.x, self.w[f"ln1.{layer}"])
        qkv = (h @ self.w[f"qkv.{layer}"]).view(n, hq + 2 * hkv, d)
        q = apply_rope(qkv[:, :hq], self.cos, self.sin).to(torch.bfloat16).contiguous()
        k = apply_rope(qkv[:, hq:hq + hkv], self.cos, self.sin).to(torch.bfloat16).contiguous()
        v = qkv[:, hq + hkv:].to(torch.bfloat16).contiguous()
        return q, k, v

    def post_attn(self, layer: int, attn_out: torch.Tensor, dm) -> None:
        cfg = self.cfg
        n = dm.host.n_tok
        att = attn_out[:n].float().reshape(n, cfg.heads * cfg.head_dim)
        self.x = self.x + att @ self.w[f"o.{layer}"]
        h = rmsnorm(self.x, self.w[f"ln2.{layer}"])
        self.x = self.x + (F.silu(h @ self.w[f"g.{layer}"]) * (h @ self.w[f"u.{layer}"])) @ self.w[f"d.{layer}"]

    def logits(self, dm):
        m = dm.host
        rows = torch.as_tensor(np.asarray(m.row_tok[: m.n_rows]), device=self.device, dtype=torch.int64)
        xw = rmsnorm(self.x[rows], self.w["ln_f"])
        return (xw @ self.w["lm"]) * self.cfg.logit_scale, None

    def on_commit(self, dm, mask: np.ndarray, tokens: np.ndarray) -> None:
        """Record the argmax tokens of the committed window rows (host)."""
        m = dm.host
        slots = dm.__dict__["slots"]
        rows = np.flatnonzero(mask[: m.n_rows])
        self.tokens[slots[m.row_req[rows]], m.row_pos[rows]] = tokens[rows]

    # -------------------------------------------------------------- DeviceLoop hooks
    def loop_setup(self, loop) -> None:
        """Capacity buffers of the graph-captured loop: committed token ids per loop
        position on the device (K3's finalize writes them), and the f3 weight."""
        cfg = self.cfg
        self.loop_tok = torch.full((loop.n, self.max_out), cfg.mask_id, dtype=torch.int32, device=self.device)
        for i, req in enumerate(loop.requests):  # tokens committed before the loop started
            s = loop.slots_h[i]
            self.loop_tok[i] = torch.from_numpy(self.tokens[s, : self.max_out].astype(np.int32))
        if self.lm_head == "f3":
            # logits = rmsnorm(x) (W_lm * scale): the scale folds into the bf16 weight [vocab, hidden]
            self.loop_w_lm = (self.w["lm"].t() * cfg.logit_scale).to(torch.bfloat16).contiguous()
            self.loop_merged = torch.empty((max(loop.caps[1], 1), 1, 3), dtype=torch.float32, device=self.device)
        self.loop_counters = torch.zeros(loop.n, dtype=torch.int32, device=self.device)

    def loop_begin(self, loop, M) -> None:
        """Token ids (kv rows: their committed token; window rows: MASK) and RoPE
        tables for the loop's capacity tokens, from the device plan."""
        cfg = self.cfg
        ct = loop.caps[0]
        r = M["tok_req"][:ct].long()
        pos = M["tok_pos"][:ct].long().clamp(0, self.max_out - 1)
        cu, cur = M["cu_seqlens"].long(), M["cu_rows"].long()
        win_start = cu[r + 1] - (cur[r + 1] - cur[r])  # ChunkPlan order: kv rows, then the window
        is_win = torch.arange(ct, device=self.device) >= win_start
        ids = torch.where(is_win, torch.full_like(pos, cfg.mask_id), self.loop_tok[r, pos].long())
        self.x = self.w["emb"][ids]
        self.cos, self.sin = rope_tables(M["prompt_len"][r].long() + M["tok_pos"][:ct].long(), cfg.head_dim,
                                         cfg.rope_theta)

    def loop_qkv(self, loop, layer: int, M):
        cfg = self.cfg
        ct = loop.caps[0]
        d, hq, hkv = cfg.head_dim, cfg.heads, cfg.kv_heads
        h = rmsnorm(self.x, self.w[f"ln1.{layer}"])
        qkv = (h @ self.w[f"qkv.{layer}"]).view(ct, hq + 2 * hkv, d)
        q = apply_rope(qkv[:, :hq], self.cos, self.sin).to(torch.bfloat16).contiguous()
        k = apply_rope(qkv[:, hq:hq + hkv], self.cos, self.sin).to(torch.bfloat16).contiguous()
        v = qkv[:, hq + hkv:].to(torch.bfloat16).contiguous()
        return q, k, v

    def loop_post_attn(self, loop, layer: int, attn_out: torch.Tensor, M) -> None:
        cfg = self.cfg
        ct = loop.caps[0]
        att = attn_out[:ct].float().reshape(ct, cfg.heads * cfg.head_dim)
        self.x = self.x + att @ self.w[f"o.{layer}"]
        h = rmsnorm(self.x, self.w[f"ln2.{layer}"])
        self.x = self.x + (F.silu(h @ self.w[f"g.{layer}"]) * (h @ self.w[f"u.{layer}"])) @ self.w[f"d.{layer}"]

    def loop_unmask(self, loop, M) -> None:
        """LM head on the window rows, then K3 into loop.res; committed tokens land in
        loop_tok (the next iterations' kv-row inputs)."""
        dcfg = loop.cfg
        cr = loop.caps[1]
        xw = rmsnorm(self.x[M["row_tok"][:cr].long()], self.w["ln_f"])
        if self.lm_head == "f3":
            merged = ops.lmhead_unmask_partials(xw.to(torch.bfloat16), self.loop_w_lm, merge=True,
                                                merged=self.loop_merged)
            ops.unmask_finalize(merged, 1, cr, 1, M["cu_rows"], dcfg.confidence_threshold, dcfg.fallback,
                                row_pos=M["row_pos"], token_buf=self.loop_tok, result=loop.res)
        else:
            logits = (xw @ self.w["lm"]) * self.cfg.logit_scale
            ops.unmask_fused(logits, None, cr, loop.n_vsplit, M["cu_rows"], M["row_req"], self.loop_counters,
                             dcfg.confidence_threshold, dcfg.fallback, row_pos=M["row_pos"], token_buf=self.loop_tok,
                             result=loop.res, part=loop.part, n_rows_dev=M["counts"][1:])
