"""Native batched host step: plan, pack, launch, apply with no per-request Python.

``NativeStepper.step(requests, chunk)`` is the same decode iteration as
``StreamingDecoder.step_python`` (plan_batch -> build_step_meta -> device step ->
apply_batch), but the control half runs in C++ over the packed ``BatchState``
(csrc/host_step.cu: ``optimus_host_plan`` / ``optimus_host_apply``), the step
metadata and the attention work list are written straight into one fixed-capacity
pinned arena, and that arena goes to the device in ONE H2D copy.  The commit mask
comes back in ONE D2H copy.
"""

from __future__ import annotations

import ctypes as C
import os
from types import SimpleNamespace
from typing import Optional

import numpy as np
import torch

from . import _lib, ops
from .batch_state import BatchState
from .core import rule_value
from .engine import StepSummary
from .errors import ConfigError


class Arena:
    """Fixed offsets for every per-step array in one pinned int32 buffer + device mirror."""

    def __init__(self, device, caps: dict):
        self.caps = dict(caps)
        self.offs = {}
        total = 0
        for name, n in caps.items():
            self.offs[name] = total
            total += ((int(n) + 3) // 4) * 4  # 16-byte aligned fields
        self.total = total
        self.host_t = torch.empty(total, dtype=torch.int32, pin_memory=True)
        self.host = self.host_t.numpy()
        self.dev = torch.empty(total, dtype=torch.int32, device=device)
        base = self.host.ctypes.data  # (numpy builds a ctypes object per .ctypes access)
        self.ptr = {name: base + 4 * o for name, o in self.offs.items()}

    def h(self, name, n=None):
        o = self.offs[name]
        return self.host[o:o + (self.caps[name] if n is None else n)]

    def d(self, name, n=None):
        o = self.offs[name]
        return self.dev[o:o + (self.caps[name] if n is None else n)]

    def hptr(self, name):
        return self.ptr[name]


class NativeStepper:
    def __init__(self, decoder, max_out: int = 4096, qcap: int = 512, max_chunk: int = 64):
        cfg = decoder.cfg
        self.dec = decoder
        self.cfg = cfg
        self.max_chunk = max_chunk
        B = cfg.max_batch
        self.bs = BatchState(B, max_out, qcap)
        # fixed host arrays: their addresses once (numpy builds a ctypes object per access)
        self._bsp = {k: getattr(self.bs, k).ctypes.data for k in (
            "states", "queue", "q_head", "q_len", "block_index", "cached_prefix", "prompt", "out_len",
            "committed", "steps_taken")}
        self._bsp["table"] = decoder.tables.table.ctypes.data
        T = B * max_chunk
        R = B * min(max_chunk, cfg.block_size)
        W = B * (max_out // 32 + 4)
        MP = cfg.max_pages_per_req
        G = cfg.num_q_heads // cfg.num_kv_heads
        mtiles = max(1, -(-max_chunk // max(1, 128 // G)))
        self.max_work = B * cfg.num_kv_heads * mtiles * 8
        self.max_groups = B * cfg.num_kv_heads * mtiles
        self.grid = decoder.grid
        # device-read fields first; the sparse tails (vis_words, work, groups) are
        # uploaded up to their used length only
        caps = dict(cu_seqlens=B + 1, tok_req=T, tok_pos=T, prompt_len=B, key_end=B, vis_base=B,
                    vis_off=B + 1, cu_rows=B + 1, row_tok=R, row_pos=R, row_req=R, row_src=R,
                    block_tables=B * MP, cta_off=self.grid + 1, vis_words=W,
                    work=self.max_work * 8, groups=self.max_groups * 8, slots=B, counts=4, commits=B, chunks=B)
        self.arena = Arena(decoder.device, caps)
        self.mask_host = torch.empty(max(R, 1), dtype=torch.uint8, pin_memory=True)
        self.tok_host = torch.empty(max(R, 1), dtype=torch.int32, pin_memory=True)
        self.lib = _lib.load()
        self._view_cache = {}
        self._graphs = {}  # (batch size, vocab splits, arena) -> captured device step
        self._g = None     # capacity-sized workspaces of the captured step
        self._cnt_h = torch.zeros(4, dtype=torch.int32, pin_memory=True)
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _grow(self, max_work: int, max_groups: int) -> None:
        """Re-lay the arena with room for a larger attention work list (long contexts
        split into many key ranges).  Per-step fields are rebuilt every step, so
        nothing needs copying; the host-side plan fields are re-planned below."""
        old = self.arena
        caps = dict(old.caps)
        caps["work"] = max_work * 8
        caps["groups"] = max_groups * 8
        self.max_work, self.max_groups = max_work, max_groups
        new = Arena(self.dec.device, caps)
        # keep this step's already-planned prefix (everything before vis_words + counts)
        new.host[: old.offs["vis_words"]] = old.host[: old.offs["vis_words"]]
        nw = int(old.h("counts", 3)[2])
        new.h("vis_words", nw)[:] = old.h("vis_words", nw)
        new.h("slots")[:] = old.h("slots")
        new.h("counts")[:] = old.h("counts")
        new.h("chunks")[:] = old.h("chunks")
        self.arena = new
        self._view_cache = {}
        self._graphs = {}

    def _views(self, n: int) -> dict:
        """Device views of the arena (capacity-sized; batch-sized where a kernel
        reads the length from the shape), cached per batch size."""
        v = self._view_cache.get(n)
        if v is None:
            A, MP = self.arena, self.cfg.max_pages_per_req
            v = {k: A.d(k) for k in ("tok_req", "tok_pos", "prompt_len", "vis_base", "vis_off", "vis_words",
                                     "row_pos", "row_req", "row_src", "cta_off")}
            v["work"] = A.d("work").view(-1, 8)
            v["groups"] = A.d("groups").view(-1, 8)
            v["block_tables"] = A.d("block_tables", n * MP).view(n, MP)
            v["cu_rows"] = A.d("cu_rows", n + 1)
            self._view_cache[n] = v
        return v

    # ------------------------------------------------------------------ admission
    def _slot(self, req, slot=None) -> int:
        tables = self.dec.tables
        s = tables.slot(req.id)
        if s is None:
            s = self.dec.admit(req, slot)
        if self.bs._req.get(s) is not req:  # admitted elsewhere (e.g. prefill): bind now
            self.bs.bind(req, s)
        return s

    def release(self, req) -> None:
        s = self.dec.tables.slot(req.id)
        if s is None:
            return
        self.bs.unbind(s)
        self.dec.tables.release(req.id)

    # ------------------------------------------------------------------ the step
    def plan(self, requests, chunk):
        """``chunk``: one chunk size for the batch, or one per request (mixed chunks)."""
        cfg = self.cfg
        n = len(requests)
        A = self.arena
        if np.ndim(chunk):
            per = A.h("chunks", n)
            per[:] = np.asarray(chunk, dtype=np.int32)
            chunk_ptr, chunk0 = A.hptr("chunks"), 0
            cmax = int(per.max()) if n else 0
        else:
            chunk_ptr, chunk0, cmax = None, int(chunk), int(chunk)
        if cmax > self.max_chunk:
            raise ConfigError(f"chunk {cmax} > native stepper max_chunk {self.max_chunk}")
        slots = A.h("slots", n)
        for i, req in enumerate(requests):
            slots[i] = self._slot(req)
        bs = self.bs
        # pages for the current block up front (the common case needs no re-gather);
        # positions the plan reaches beyond them (OUT_BLOCK windows can lie in any
        # later block) are allocated from the exact plan below
        sl = slots.astype(np.int64)
        reach = np.minimum(bs.out_len[sl], (bs.block_index[sl] + 1) * cfg.block_size)
        need = (bs.prompt[sl] + reach + cfg.page_size - 1) // cfg.page_size
        tables = self.dec.tables
        for i in np.flatnonzero(need > tables.n_pages[sl]):
            tables.ensure(int(sl[i]), int(bs.prompt[sl[i]] + reach[i]))
        MP = cfg.max_pages_per_req
        L = self.lib
        st = L.optimus_host_plan(
            n, A.hptr("slots"), chunk0, chunk_ptr, cfg.block_size,
            0 if rule_value(cfg.window_rule) == "in_block" else 1,
            self._bsp['states'], bs.states.shape[1], self._bsp['queue'], bs.qcap,
            self._bsp['q_head'], self._bsp['q_len'], self._bsp['block_index'],
            self._bsp['cached_prefix'], self._bsp['prompt'], self._bsp['out_len'],
            self._bsp['table'], MP, A.hptr("cu_seqlens"), A.hptr("tok_req"), A.hptr("tok_pos"),
            A.caps["tok_pos"], A.hptr("prompt_len"), A.hptr("key_end"), A.hptr("vis_base"),
            A.hptr("vis_off"), A.hptr("vis_words"), A.caps["vis_words"], A.hptr("cu_rows"),
            A.hptr("row_tok"), A.hptr("row_pos"), A.hptr("row_req"), A.caps["row_pos"],
            A.hptr("block_tables"), A.hptr("counts"))
        _lib.check(st, "optimus_host_plan")
        n_tok, n_rows, n_words = (int(x) for x in A.h("counts", 3))
        self._cover_planned(n, sl, A, n_tok)
        # attention work list straight into the arena
        ng, npart = C.c_int(0), C.c_int(0)
        mw, mg = C.c_int(0), C.c_int(0)
        _lib.check(L.optimus_attn_plan_bounds(n, A.hptr("cu_seqlens"), A.hptr("key_end"), cfg.num_q_heads,
                                              cfg.num_kv_heads, cfg.min_split_tiles, cfg.page_size,
                                              C.byref(mw), C.byref(mg)), "optimus_attn_plan_bounds")
        if mw.value > self.max_work or mg.value > self.max_groups:
            self._grow(max(mw.value, self.max_work), max(mg.value, self.max_groups))
            A = self.arena
        nw = L.optimus_attn_plan(n, A.hptr("cu_seqlens"), A.hptr("key_end"), cfg.num_q_heads,
                                 cfg.num_kv_heads, self.grid, cfg.min_split_tiles, cfg.page_size,
                                 A.hptr("work"), self.max_work, A.hptr("cta_off"), A.hptr("groups"),
                                 self.max_groups, C.byref(ng), C.byref(npart))
        if nw < 0:
            _lib.check(nw, "optimus_attn_plan")
        host = SimpleNamespace(
            n_req=n, n_tok=n_tok, n_rows=n_rows, cu_seqlens=A.h("cu_seqlens", n + 1),
            cu_rows=A.h("cu_rows", n + 1), row_req=A.h("row_req", n_rows), row_pos=A.h("row_pos", n_rows),
            row_tok=A.h("row_tok", n_rows), tok_pos=A.h("tok_pos", n_tok), key_end=A.h("key_end", n),
            vis_base=A.h("vis_base", n), vis_off=A.h("vis_off", n + 1), vis_words=A.h("vis_words", n_words).view(np.uint32),
            prompt_len=A.h("prompt_len", n), block_tables=A.h("block_tables", n * MP).reshape(n, MP))
        V = self._views(n)
        plan = ops.AttnPlan(self.grid, nw, ng.value, npart.value, V["work"], V["cta_off"], V["groups"],
                            A.h("work", nw * 8).reshape(-1, 8), A.h("cta_off"), A.h("groups", ng.value * 8).reshape(-1, 8),
                            ops.single_query_tile(host.cu_seqlens, cfg.num_q_heads, cfg.num_kv_heads))
        dm = SimpleNamespace(host=host, tok_req=V["tok_req"], tok_pos=V["tok_pos"],
                             prompt_len=V["prompt_len"], vis_base=V["vis_base"], vis_off=V["vis_off"],
                             vis_words=V["vis_words"], block_tables=V["block_tables"],
                             cu_rows=V["cu_rows"], row_pos=V["row_pos"], row_req=V["row_req"], row_src=V["row_src"])
        dm.__dict__.update(attn_plan=plan, slots=slots.astype(np.int64), requests=requests, plans=None,
                           row_src_host=A.h("row_src"))
        return dm

    def _cover_planned(self, n, sl, A, n_tok) -> None:
        """Every planned position must have a page before K1 writes it: allocate the
        pages the plan reaches beyond the current block and re-gather those requests'
        block-table rows into the arena."""
        if not n_tok:
            return
        cfg, tables, bs = self.cfg, self.dec.tables, self.bs
        cu = A.h("cu_seqlens", n + 1)
        pos = A.h("tok_pos", n_tok)
        nz = np.flatnonzero(cu[1:] > cu[:-1])
        hi = np.full(n, -1, dtype=np.int64)
        hi[nz] = np.maximum.reduceat(pos, cu[:-1][nz])
        need = (bs.prompt[sl] + hi + cfg.page_size) // cfg.page_size
        short = np.flatnonzero((hi >= 0) & (need > tables.n_pages[sl]))
        if short.size:
            MP = cfg.max_pages_per_req
            bt = A.h("block_tables", n * MP).reshape(n, MP)
            for i in short:
                tables.ensure(int(sl[i]), int(bs.prompt[sl[i]] + hi[i] + 1))
                bt[i] = tables.table[sl[i]]

    def upload(self, dm) -> None:
        A = self.arena
        plan = dm.__dict__["attn_plan"]
        n_words = int(A.h("counts", 3)[2])
        spans = [(0, A.offs["vis_words"]), (A.offs["vis_words"], max(n_words, 1)),
                 (A.offs["work"], max(plan.n_work, 1) * 8), (A.offs["groups"], max(plan.n_groups, 1) * 8)]
        nbytes = 0
        for o, n in spans:
            A.dev[o:o + n].copy_(A.host_t[o:o + n], non_blocking=True)
            nbytes += 4 * n
        self.h2d_bytes = nbytes

    def fetch_and_apply(self, dm, res) -> np.ndarray:
        n, n_rows = dm.host.n_req, dm.host.n_rows
        A = self.arena
        fwd = self.dec.forward
        want_tok = getattr(fwd, "needs_tokens", False)
        if n_rows:
            self.mask_host[:n_rows].copy_(res.commit_mask[:n_rows], non_blocking=True)
            if want_tok:
                self.tok_host[:n_rows].copy_(res.tokens[:n_rows], non_blocking=True)
        gate = self.dec.v_gate
        if gate is not None:
            gate.issue()
        # always: the next plan() rewrites the pinned arena this step's non-blocking
        # upload reads from, so that upload must have completed (even with no rows)
        torch.cuda.current_stream().synchronize()
        if gate is not None:
            gate.check()
        self.d2h_bytes = n_rows * (5 if want_tok else 1)
        if want_tok and n_rows:
            fwd.on_commit(dm, self.mask_host.numpy()[:n_rows].astype(bool), self.tok_host.numpy()[:n_rows])
        bs = self.bs
        st = self.lib.optimus_host_apply(
            n, A.hptr("slots"), self.cfg.block_size, A.hptr("cu_seqlens"), A.hptr("tok_pos"),
            A.hptr("cu_rows"), A.hptr("row_pos"), self.mask_host.data_ptr(), self._bsp['states'],
            bs.states.shape[1], self._bsp['queue'], bs.qcap, self._bsp['q_head'], self._bsp['q_len'],
            self._bsp['block_index'], self._bsp['committed'], self._bsp['steps_taken'],
            self._bsp['cached_prefix'], self._bsp['out_len'], A.hptr("commits"))
        _lib.check(st, "optimus_host_apply")
        return A.h("commits", n)

    # ------------------------------------------------------------------ graph step
    def _graph_ok(self, dm) -> bool:
        """The device step can replay as one captured graph: activations and the
        logits table are resident (fixed addresses), K1 runs as its own kernel, and
        every per-step count is read on the device (K1 / K3 / split-KV combine).

        Off by default (OPTIMUS_STEP_GRAPH=1 enables it): measured 2.27 ms/step against
        1.96-2.20 ms eager on the ShareGPT closed loop.  The capacity-sized grids (K3
        over every row slot, K1 over every token slot) and a capture per new (batch,
        split) key cost more than the 72 launches they replace; DeviceLoop is the
        graph path that pays."""
        dec, fwd = self.dec, self.dec.forward
        return (os.environ.get("OPTIMUS_STEP_GRAPH", "0") != "0" and dm.host.n_tok > 0
                and getattr(fwd, "resident_layers", False) and hasattr(fwd, "fill_row_src")
                and dec.unmask_impl is None and dec.append_mode == "k1")

    def _graph_workspaces(self):
        cfg, fwd = self.cfg, self.dec.forward
        cap_tok = min(self.arena.caps["tok_req"], fwd.qkv_capacity)
        R = self.arena.caps["row_src"]
        g = self._g
        if g is None or g["max_work"] != self.max_work:
            dev = self.dec.device
            g = dict(max_work=self.max_work, cap_tok=cap_tok, R=R,
                     out=torch.empty((cap_tok, cfg.num_q_heads, cfg.head_dim), dtype=torch.bfloat16, device=dev),
                     ws_o=torch.empty(self.max_work * 128 * cfg.head_dim, dtype=torch.float32, device=dev),
                     ws_ml=torch.empty(self.max_work * 256, dtype=torch.float32, device=dev),
                     cnt=torch.zeros(4, dtype=torch.int32, device=dev),
                     res=ops.UnmaskResult(torch.empty(R, dtype=torch.uint8, device=dev),
                                          torch.empty(R, dtype=torch.int32, device=dev),
                                          torch.empty(R, dtype=torch.float32, device=dev)))
            self._g = g
            self._graphs = {}
        return g

    def _enqueue_step(self, dm, n, n_vsplit, stream) -> None:
        """L x (K1, K2, split-KV combine) + K3 over the arena at capacity, counts from
        the device (what the captured graph holds)."""
        cfg, fwd, g, A = self.cfg, self.dec.forward, self._g, self.arena
        V = self._views(n)
        p = lambda t: t.data_ptr()
        hq, hkv, d = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
        v_dtype = ops._v_dtype(self.dec.cache.v)
        MP = cfg.max_pages_per_req
        cnt = g["cnt"]
        for layer in range(cfg.num_layers):
            buf = fwd.qkv_buf[layer % len(fwd.qkv_buf)]
            kc, vc = self.dec.cache.layer(layer)
            _lib.check(_lib.call(
                "optimus_kv_append_dev", p(buf[:, hq]), p(buf[:, hq + hkv]), buf.stride(0), p(V["tok_req"]),
                p(V["tok_pos"]), p(V["prompt_len"]), p(A.d("block_tables")), MP, g["cap_tok"], p(cnt), hkv, d,
                cfg.page_size, p(kc), p(vc), v_dtype, stream), "kv_append_dev")
            _lib.check(_lib.call(
                "optimus_paged_attn", p(buf), buf.stride(0), g["cap_tok"], p(kc), p(vc), kc.shape[0],
                p(V["tok_pos"]), p(V["prompt_len"]), p(V["vis_base"]), p(V["vis_off"]), p(V["vis_words"]),
                p(A.d("block_tables")), MP, p(V["work"]), p(V["cta_off"]), self.grid, p(V["groups"]), 0,
                cfg.block_size, hq, hkv, d, cfg.page_size, 1.0 / float(d) ** 0.5, p(g["out"]), g["out"].stride(0),
                p(g["ws_o"]), p(g["ws_ml"]), v_dtype, stream), "paged_attn")
            _lib.check(_lib.call(
                "optimus_paged_attn_combine_dev", p(V["groups"]), p(cnt[2:]), self.max_groups, p(g["ws_o"]),
                p(g["ws_ml"]), hq, hkv, d, p(g["out"]), g["out"].stride(0), stream), "paged_attn_combine_dev")
        logits = fwd.logit_table
        dt = 0 if logits.dtype == torch.bfloat16 else 1
        R = g["R"]
        part = g["part"][: R * n_vsplit * 3]
        if fwd.vocab_offset == 0:
            if g.get("k3_counters") is None or g["k3_counters"].numel() < max(n, 1):
                g["k3_counters"] = torch.zeros(max(n, cfg.max_batch, 1), dtype=torch.int32, device=logits.device)
            ops.unmask_fused(logits, V["row_src"], R, n_vsplit, V["cu_rows"], V["row_req"], g["k3_counters"],
                             cfg.confidence_threshold, cfg.fallback, result=g["res"], part=part.view(R, n_vsplit, 3),
                             n_rows_dev=cnt[1:], stream=torch.cuda.ExternalStream(stream))
            return
        _lib.check(_lib.call(
            "optimus_unmask_partials_dev", p(logits), dt, logits.stride(0), p(V["row_src"]), R, p(cnt[1:]),
            logits.shape[-1], fwd.vocab_offset, n_vsplit, p(part), stream), "unmask_partials_dev")
        ops.unmask_finalize(part.view(R, n_vsplit, 3), 1, R, n_vsplit, V["cu_rows"], cfg.confidence_threshold,
                            cfg.fallback, result=g["res"], stream=torch.cuda.ExternalStream(stream))

    def device_step_graph(self, dm):
        """The device step as one CUDA graph replay (captured per batch size and
        vocab-split count), after the per-step counts' H2D."""
        m = dm.host
        fwd = self.dec.forward
        n_vsplit = ops.unmask_splits(m.n_rows, fwd.logit_table.shape[-1])
        g = self._graph_workspaces()
        need = g["R"] * n_vsplit * 3
        if g.get("part") is None or g["part"].numel() < need:
            g["part"] = torch.empty(max(need, g["R"] * 32 * 3), dtype=torch.float32, device=self.dec.device)
            self._graphs = {}
        key = (m.n_req, n_vsplit)
        self._cnt_h.numpy()[:] = (m.n_tok, m.n_rows, dm.attn_plan.n_groups, 0)
        g["cnt"].copy_(self._cnt_h, non_blocking=True)
        graph = self._graphs.get(key)
        if graph is None:
            s = torch.cuda.Stream(device=self.dec.device)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._enqueue_step(dm, m.n_req, n_vsplit, s.cuda_stream)  # warm: lazy kernel attributes
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=s):
                    self._enqueue_step(dm, m.n_req, n_vsplit, s.cuda_stream)
            torch.cuda.current_stream().wait_stream(s)
            self._graphs[key] = graph
        graph.replay()
        return g["res"]

    def step(self, requests, chunk: int, summaries: bool = True):
        dm = self.plan(requests, chunk)
        if hasattr(self.dec.forward, "fill_row_src"):
            self.dec.forward.fill_row_src(dm)
        self.upload(dm)
        res = self.device_step_graph(dm) if self._graph_ok(dm) else self.dec.device_step(dm)
        mask_rows = dm.host.n_rows
        counts = self.fetch_and_apply(dm, res)
        out = None
        if summaries:
            cu_t, cu_r = dm.host.cu_seqlens, dm.host.cu_rows
            mask = self.mask_host.numpy()[:mask_rows].astype(bool)
            pos = dm.host.row_pos
            out = []
            for r in range(dm.host.n_req):
                a, b = int(cu_r[r]), int(cu_r[r + 1])
                out.append(StepSummary(computed=int(cu_t[r + 1] - cu_t[r]),
                                       commits=frozenset(pos[a:b][mask[a:b]].tolist())))
        for req in requests:
            if req.finished:
                self.release(req)
        return out if summaries else int(counts.sum())
