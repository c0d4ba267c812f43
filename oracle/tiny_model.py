"""CPU oracle of the tiny SDAR-style dLLM (BASELINE config 1) — TEST INFRASTRUCTURE.

The same model as paper_2605_24832_b200/tiny_model.py in numpy, with the same
precision points (fp32 activations and GEMMs; q, k, v and the attention output
rounded to bf16 because that is what the B200 kernels consume/produce).  KV is
kept per layer and per request as dense arrays over absolute positions; each
decode step appends every planned token's K/V first (rule K) and then attends
with the rule-V visibility mask (oracle/numeric.py).
"""

from __future__ import annotations

import numpy as np

from oracle import numeric as on


def _rms(x, w, eps=1e-6):
    return x * (1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)) * w


def _rope(x, pos, d, theta):
    inv = 1.0 / (theta ** (np.arange(0, d, 2, dtype=np.float32) / d))
    ang = pos.astype(np.float32)[:, None] * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    out = np.empty_like(x)
    out[..., ::2] = x[..., ::2] * c - x[..., 1::2] * s
    out[..., 1::2] = x[..., ::2] * s + x[..., 1::2] * c
    return out


def _silu(x):
    return x / (1.0 + np.exp(-x))


class TinyOracle:
    def __init__(self, cfg, weights: dict):
        self.cfg = cfg
        self.w = weights
        self.K = {}  # (layer, req_id) -> [n_abs, Hkv, d]
        self.V = {}

    def _layer_qkv(self, x, l, pos):
        c = self.cfg
        n = x.shape[0]
        h = _rms(x, self.w[f"ln1.{l}"])
        qkv = (h @ self.w[f"qkv.{l}"]).reshape(n, c.heads + 2 * c.kv_heads, c.head_dim)
        q = on.bf16_round(_rope(qkv[:, :c.heads], pos, c.head_dim, c.rope_theta))
        k = on.bf16_round(_rope(qkv[:, c.heads:c.heads + c.kv_heads], pos, c.head_dim, c.rope_theta))
        v = on.bf16_round(qkv[:, c.heads + c.kv_heads:])
        return q, k, v

    def _mlp(self, x, att, l):
        x = x + att @ self.w[f"o.{l}"]
        h = _rms(x, self.w[f"ln2.{l}"])
        return x + (_silu(h @ self.w[f"g.{l}"]) * (h @ self.w[f"u.{l}"])) @ self.w[f"d.{l}"]

    def prefill(self, rid, ids, out_len):
        c = self.cfg
        n = len(ids)
        x = self.w["emb"][np.asarray(ids)]
        pos = np.arange(n)
        G = c.heads // c.kv_heads
        for l in range(c.layers):
            q, k, v = self._layer_qkv(x, l, pos)
            K = np.zeros((n + out_len, c.kv_heads, c.head_dim), np.float32)
            V = np.zeros_like(K)
            K[:n], V[:n] = k, v
            self.K[(l, rid)], self.V[(l, rid)] = K, V
            att = np.zeros((n, c.heads, c.head_dim), np.float32)
            mask = np.tril(np.ones((n, n), bool))
            for h in range(c.kv_heads):
                for g in range(G):
                    S = (q[:, h * G + g] @ k[:, h].T) / np.sqrt(c.head_dim)
                    S = np.where(mask, S, -np.inf)
                    P = np.exp(S - S.max(1, keepdims=True))
                    att[:, h * G + g] = (P / P.sum(1, keepdims=True)) @ v[:, h]
            x = self._mlp(x, on.bf16_round(att).reshape(n, -1), l)

    def step(self, reqs, plans, tokens_of, block):
        """Logits [window rows, V] for one decode step; ``tokens_of(req, p)`` gives
        the committed token id of output position p (kv rows)."""
        c = self.cfg
        ids, pos_abs, owner, tpos = [], [], [], []
        for r, (req, plan) in enumerate(zip(reqs, plans)):
            for p in plan.kv_positions:
                ids.append(tokens_of(req, p))
            ids += [c.mask_id] * len(plan.window)
            for p in list(plan.kv_positions) + list(plan.window):
                pos_abs.append(req.prompt_tokens + p)
                owner.append(r)
                tpos.append(p)
        ids, pos_abs, owner, tpos = map(np.asarray, (ids, pos_abs, owner, tpos))
        x = self.w["emb"][ids]
        G = c.heads // c.kv_heads
        for l in range(c.layers):
            q, k, v = self._layer_qkv(x, l, pos_abs)
            att = np.zeros((len(ids), c.heads, c.head_dim), np.float32)
            for r, (req, plan) in enumerate(zip(reqs, plans)):
                sel = np.flatnonzero(owner == r)
                if sel.size == 0:
                    continue
                K, V = self.K[(l, req.id)], self.V[(l, req.id)]
                K[pos_abs[sel]] = k[sel]   # rule K: append every planned token first
                V[pos_abs[sel]] = v[sel]
                vis = on.visible_outputs(req.states, list(plan.kv_positions) + list(plan.window))
                n_keys = req.prompt_tokens + req.output_tokens
                mask = on.key_mask(req.prompt_tokens, vis, tpos[sel], block, n_keys)
                for h in range(c.kv_heads):
                    for g in range(G):
                        S = (q[sel, h * G + g] @ K[:n_keys, h].T) / np.sqrt(c.head_dim)
                        S = np.where(mask, S, -np.inf)
                        P = np.exp(S - S.max(1, keepdims=True))
                        att[sel, h * G + g] = (P / P.sum(1, keepdims=True)) @ V[:n_keys, h]
            x = self._mlp(x, on.bf16_round(att).reshape(len(ids), -1), l)
        rows = np.concatenate([np.flatnonzero(owner == r)[len(plan.kv_positions):]
                               for r, plan in enumerate(plans)]) if len(ids) else np.zeros(0, int)
        xw = _rms(x[rows], self.w["ln_f"])
        return (xw @ self.w["lm"]) * c.logit_scale
