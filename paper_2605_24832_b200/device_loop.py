"""Graph-captured streaming decode step with its control half on the device.

``DeviceLoop`` runs the whole iteration of the streaming branch of ``_Loop.run_decode``
(sim.py:269-305) as ONE CUDA graph on device-resident request state:

    optimus_device_plan       plan_chunk for every request + the step metadata
    optimus_device_attn_plan  the attention work list (LPT placement, balanced split-KV cuts)
    optimus_slot_mapping_dev  the step's slot map (append mode "slots", the default)
    L x (optimus_kv_append_slots_dev | optimus_kv_append_dev, optimus_paged_attn,
         optimus_paged_attn_combine_dev)
    optimus_device_row_src, optimus_unmask_commit (K3 in one launch)
    optimus_device_apply      apply_chunk + advance_blocks
    D2H of the plan arrays and the commit mask into pinned buffers

so no host round trip sits between steps.  The host keeps the reference-facing
``Request`` objects exact by replaying the same transitions with
``optimus_host_apply`` from the copied plan (bit-identical to the device's; see
tests/test_device_loop_gpu.py, which also checks the whole loop against the host
native step).  The batch is fixed for the loop's lifetime (finished requests plan
zero tokens, ``replace`` refills a finished position); every request's pages are
allocated up front.

The chunk is elastic: the device plan always reads a per-position chunk array, so
``step(chunk=c)`` / ``set_chunk`` change it between iterations without a re-capture
(one chunk for the batch, as ElasticChunk picks it every iteration, sim.py:219-232,
270-272, or one per position).  Capacities are sized for ``max_chunk``.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib, ops
from .core import rule_value
from .engine import StepSummary
from .errors import ConfigError


class DeviceLoop:
    MAX_REQ, MAX_CHUNK, MAX_OUT, MAX_UNITS = 256, 128, 4096, 4096

    @classmethod
    def _check_request(cls, r, nat) -> None:
        if r.output_tokens > min(cls.MAX_OUT, nat.bs.states.shape[1]):
            raise ConfigError(f"DeviceLoop: request {r.id} has {r.output_tokens} output tokens > "
                              f"{min(cls.MAX_OUT, nat.bs.states.shape[1])}")

    def __init__(self, decoder, requests, chunk, lookahead: bool = False, max_chunk: int = None):
        cfg = decoder.cfg
        fwd = decoder.forward
        # two kinds of forward: a model with loop hooks (loop_setup / loop_begin / loop_qkv /
        # loop_post_attn / loop_unmask, capacity-shaped and graph-capturable: TinyDLLM), or
        # resident per-layer activations with a slot-indexed logits table (SyntheticForward)
        self.model = bool(getattr(fwd, "loop_model", False))
        if not self.model and (not getattr(fwd, "resident_layers", False) or not hasattr(fwd, "row_src_host")):
            raise ConfigError("DeviceLoop needs a forward with loop hooks (loop_model) or resident per-layer "
                              "activations and a slot-indexed logits table (SyntheticForward)")
        self.dec, self.cfg = decoder, cfg
        # one chunk for the batch, or one per loop position (mixed chunks, the elastic
        # scheduler's per-request sizes); capacities follow the largest
        mixed = np.ndim(chunk) > 0
        self.chunk_h = np.asarray(chunk if mixed else [chunk] * len(requests), dtype=np.int32)
        if len(self.chunk_h) != len(requests) or self.chunk_h.min() < 2:
            raise ConfigError("DeviceLoop: one chunk >= 2 per request")
        # capacity chunk: the largest chunk any later iteration may ask for
        self.chunk = max(int(self.chunk_h.max()), int(max_chunk or 0))
        nat = decoder.native()
        # the device planners' hard limits (csrc/device_step.cu): checked here so a
        # captured graph never runs a step they would reject
        if len(requests) > self.MAX_REQ:
            raise ConfigError(f"DeviceLoop: {len(requests)} requests > {self.MAX_REQ}")
        if self.chunk > self.MAX_CHUNK:
            raise ConfigError(f"DeviceLoop: chunk {self.chunk} > {self.MAX_CHUNK}")
        for r in requests:
            self._check_request(r, nat)
        G = cfg.num_q_heads // cfg.num_kv_heads
        units = len(requests) * cfg.num_kv_heads * -(-self.chunk // max(1, 128 // G))
        if units > self.MAX_UNITS:
            raise ConfigError(f"DeviceLoop: {units} attention units > {self.MAX_UNITS}")
        self.nat = nat
        self.requests = list(requests)
        self.n = n = len(self.requests)
        dev = decoder.device
        self.dev = dev
        slots = []
        for r in self.requests:
            s = nat._slot(r)
            decoder.tables.ensure(s, r.prompt_tokens + r.output_tokens)
            slots.append(s)
        self.slots_h = np.asarray(slots, dtype=np.int32)
        max_pages = cfg.max_pages_per_req
        bs = nat.bs
        self.bs = bs
        self.state_keys = ("states", "queue", "q_head", "q_len", "block_index", "committed", "steps_taken",
                           "cached_prefix", "prompt", "out_len")
        self.D = {k: torch.from_numpy(np.ascontiguousarray(getattr(bs, k))).to(dev) for k in self.state_keys}
        self.Dt = torch.from_numpy(np.ascontiguousarray(decoder.tables.table)).to(dev)
        self.slots = torch.from_numpy(self.slots_h).to(dev)
        # per-position chunks, read by the device plan every replay (elastic chunk)
        self.chunks_d = torch.from_numpy(self.chunk_h).to(dev)
        self._chunks_pin = torch.from_numpy(self.chunk_h.copy()).pin_memory()
        self._chunks_ev = None  # the last staging copy (the pinned buffer is reused)
        ct = n * self.chunk
        cr = n * min(self.chunk, cfg.block_size)
        cw = n * (bs.states.shape[1] // 32 + 4)
        self.caps = (ct, cr, cw)
        z = lambda m, dt=torch.int32: torch.zeros(max(m, 1), dtype=dt, device=dev)
        M = dict(cu_seqlens=z(n + 1), tok_req=z(ct), tok_pos=z(ct), prompt_len=z(n), key_end=z(n), vis_base=z(n),
                 vis_off=z(n + 1), vis_words=z(cw), cu_rows=z(n + 1), row_tok=z(cr), row_pos=z(cr), row_req=z(cr),
                 counts=z(4), row_src=z(cr), commits=z(n), slot_abs=z(2 * ct))
        M["block_tables"] = torch.zeros((n, max_pages), dtype=torch.int32, device=dev)
        G = cfg.num_q_heads // cfg.num_kv_heads
        T = 128 // G
        self.grid = decoder.grid
        # units + the cut pieces (a balanced cut adds < 2 pieces per CTA) + page-cap cuts
        units = n * cfg.num_kv_heads * ((self.chunk + T - 1) // T)
        cap_cuts = units * (-(-max_pages // 255) - 1)  # any admitted request fits max_pages
        self.max_work = min(4096, units + 2 * self.grid + 64 + cap_cuts)
        M["work"] = torch.zeros((self.max_work, 8), dtype=torch.int32, device=dev)
        M["cta_off"] = z(self.grid + 1)
        M["groups"] = torch.zeros((min(units, 1024), 8), dtype=torch.int32, device=dev)
        # split-KV partials (m, l, O) of the cut pieces: at most one per work item
        self.ws_o = torch.empty(self.max_work * 128 * cfg.head_dim, dtype=torch.float32, device=dev)
        self.ws_ml = torch.empty(self.max_work * 128 * 2, dtype=torch.float32, device=dev)
        # what the host replay reads back every iteration lives in ONE device buffer
        # (16-byte aligned views), so each iteration ends with one D2H copy, not seven
        rb = [("counts", 4), ("wcounts", 4), ("cu_seqlens", n + 1), ("tok_pos", max(ct, 1)),
              ("cu_rows", n + 1), ("row_pos", max(cr, 1)), ("mask", (max(cr, 1) + 3) // 4)]
        offs, o = {}, 0
        for k, m in rb:
            offs[k] = (o, m)
            o += -(-m // 4) * 4
        self._rb = torch.zeros(o, dtype=torch.int32, device=dev)
        for k, (o0, m) in offs.items():
            if k != "mask":
                M[k] = self._rb[o0: o0 + m]
        o0, m = offs["mask"]
        mask_d = self._rb[o0: o0 + m].view(torch.uint8)[: max(cr, 1)]
        self._rb_offs = offs
        self.M = M
        vocab = cfg.vocab if self.model else fwd.logit_table.shape[-1]
        self.logits = None if self.model else fwd.logit_table
        # vocab slices for about half the row capacity (window rows vary step to step)
        self.n_vsplit = ops.unmask_splits(max(cr // 2, 1), vocab)
        self.part = torch.empty((cr, self.n_vsplit, 3), dtype=torch.float32, device=dev)
        self.k3_counters = torch.zeros(n, dtype=torch.int32, device=dev)  # unmask_fused arrivals (zero between steps)
        self.res = ops.UnmaskResult(mask_d, z(cr), z(cr, torch.float32))
        self.out = torch.empty((ct, cfg.num_q_heads, cfg.head_dim), dtype=torch.bfloat16, device=dev)
        # pinned host mirrors of what the host replay needs
        # with lookahead two graphs alternate, each reading back into its own buffers, so
        # the next iteration is launched before this one's results are read
        def host_mirror():
            buf = torch.zeros(self._rb.numel(), dtype=torch.int32, pin_memory=True)
            H = {"_all": buf}
            for k, (o0, m) in offs.items():
                H[k] = buf[o0: o0 + m] if k != "mask" else buf[o0: o0 + m].view(torch.uint8)[: max(cr, 1)]
            H["vsat"] = torch.zeros(2, dtype=torch.int32, pin_memory=True)  # fp16 V clamp flags
            return H
        self.Hs = [host_mirror() for _ in range(2 if lookahead else 1)]
        self.H = self.Hs[0]
        self.graphs = []
        self._events = [torch.cuda.Event() for _ in self.Hs]
        self._cur = 0
        self.t_device = 0.0  # host seconds spent in replay + sync (diagnostics)
        self.free = set()  # loop indices whose request finished and was released
        self.lookahead = bool(lookahead)
        self._inflight = False  # a lookahead iteration was launched and not yet consumed
        self._stale = set()  # positions refilled while an iteration was in flight
        self._last = (np.zeros(n + 1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.uint8))
        self._h2d = 0
        self.h2d_bytes = self.d2h_bytes = 0
        # admissions (replace) are packed into one record per request and copied into the
        # device state by ONE H2D + ONE optimus_device_admit launch before the next replay
        self._rec_ints = _lib.call("optimus_admit_record_ints", bs.states.shape[1], bs.qcap, self.Dt.shape[1])
        _lib.check(min(self._rec_ints, 0), "optimus_admit_record_ints")
        self._pending = []
        self._adm_pin = torch.zeros((n, self._rec_ints), dtype=torch.int32, pin_memory=True)
        self._adm_dev = torch.zeros((n, self._rec_ints), dtype=torch.int32, device=dev)
        self._adm_ev = None  # the last staging copy (the pinned buffer is reused)
        if self.model:
            fwd.loop_setup(self)

    # ------------------------------------------------------------------ device
    def _enqueue(self, stream, H=None) -> None:
        cfg, D, M, n = self.cfg, self.D, self.M, self.n
        H = self.H if H is None else H
        ct, cr, cw = self.caps
        p = lambda t: t.data_ptr()
        L = _lib
        rule = 0 if rule_value(cfg.window_rule) == "in_block" else 1
        _lib.check(L.call(
            "optimus_device_plan", n, p(self.slots), self.chunk, p(self.chunks_d), cfg.block_size, rule,
            p(D["states"]),
            D["states"].shape[1], p(D["queue"]), self.bs.qcap, p(D["q_head"]), p(D["q_len"]), p(D["block_index"]),
            p(D["cached_prefix"]), p(D["prompt"]), p(D["out_len"]), p(self.Dt), self.Dt.shape[1],
            p(M["cu_seqlens"]), p(M["tok_req"]), p(M["tok_pos"]), ct, p(M["prompt_len"]), p(M["key_end"]),
            p(M["vis_base"]), p(M["vis_off"]), p(M["vis_words"]), cw, p(M["cu_rows"]), p(M["row_tok"]),
            p(M["row_pos"]), p(M["row_req"]), cr, p(M["block_tables"]), p(M["counts"]), stream), "device_plan")
        _lib.check(L.call(
            "optimus_device_attn_plan", n, p(M["cu_seqlens"]), p(M["key_end"]), cfg.num_q_heads, cfg.num_kv_heads,
            self.grid, cfg.page_size, 1, p(M["work"]), self.max_work, p(M["cta_off"]), p(M["groups"]),
            M["groups"].shape[0], p(M["wcounts"]), stream), "device_attn_plan")
        fwd = self.dec.forward
        scale = 1.0 / float(cfg.head_dim) ** 0.5
        v_dtype = ops._v_dtype(self.dec.cache.v)
        # K1 over the step's slot map (the decoder's append mode "slots", default): the
        # map once per iteration, then one round trip per row in every layer
        slots = self.dec.append_mode != "k1"
        if slots:
            _lib.check(L.call(
                "optimus_slot_mapping_dev", p(M["tok_req"]), p(M["tok_pos"]), p(M["prompt_len"]),
                p(M["block_tables"]), M["block_tables"].shape[1], ct, p(M["counts"]), cfg.page_size,
                p(M["slot_abs"]), stream), "slot_mapping_dev")
        if self.model:
            fwd.loop_begin(self, M)
        for layer in range(cfg.num_layers):
            hq, hkv = cfg.num_q_heads, cfg.num_kv_heads
            if self.model:
                q, k, v = fwd.loop_qkv(self, layer, M)  # capacity rows, bf16, unit inner strides
                if k.stride(0) != v.stride(0):
                    raise ConfigError("DeviceLoop: the model's K and V rows must share a row stride")
            else:
                buf = fwd.qkv_buf[layer]
                q, k, v = buf, buf[:, hq], buf[:, hq + hkv]
            kc, vc = self.dec.cache.layer(layer)
            if slots:
                _lib.check(L.call(
                    "optimus_kv_append_slots_dev", p(k), p(v), k.stride(0), p(M["slot_abs"]), ct, p(M["counts"]),
                    hkv, cfg.head_dim, cfg.page_size, p(kc), p(vc), v_dtype, stream), "kv_append_slots_dev")
            else:
                _lib.check(L.call(
                    "optimus_kv_append_dev", p(k), p(v), k.stride(0), p(M["tok_req"]),
                    p(M["tok_pos"]), p(M["prompt_len"]), p(M["block_tables"]), M["block_tables"].shape[1], ct,
                    p(M["counts"]), hkv, cfg.head_dim, cfg.page_size, p(kc), p(vc), v_dtype, stream),
                    "kv_append_dev")
            _lib.check(L.call(
                "optimus_paged_attn", p(q), q.stride(0), q.shape[0], p(kc), p(vc), kc.shape[0],
                p(M["tok_pos"]), p(M["prompt_len"]), p(M["vis_base"]), p(M["vis_off"]), p(M["vis_words"]),
                p(M["block_tables"]), M["block_tables"].shape[1], p(M["work"]), p(M["cta_off"]), self.grid,
                p(M["groups"]), 0, cfg.block_size, hq, hkv, cfg.head_dim, cfg.page_size, scale, p(self.out),
                self.out.stride(0), p(self.ws_o), p(self.ws_ml), v_dtype, stream), "paged_attn")
            _lib.check(L.call(
                "optimus_paged_attn_combine_dev", p(M["groups"]), p(M["wcounts"][1:]), M["groups"].shape[0],
                p(self.ws_o), p(self.ws_ml), hq, hkv, cfg.head_dim, p(self.out), self.out.stride(0), stream),
                "paged_attn_combine_dev")
            if self.model:
                fwd.loop_post_attn(self, layer, self.out, M)
        if self.model:
            fwd.loop_unmask(self, M)  # LM head on the window rows -> K3 into self.res
        else:
            self._unmask_synthetic(M, stream)
        _lib.check(L.call(
            "optimus_device_apply", n, p(self.slots), cfg.block_size, p(M["cu_seqlens"]), p(M["tok_pos"]),
            p(M["cu_rows"]), p(M["row_pos"]), p(self.res.commit_mask), p(D["states"]), D["states"].shape[1],
            p(D["queue"]), self.bs.qcap, p(D["q_head"]), p(D["q_len"]), p(D["block_index"]), p(D["committed"]),
            p(D["steps_taken"]), p(D["cached_prefix"]), p(D["out_len"]), p(M["commits"]), p(M["counts"][3:]),
            stream), "device_apply")  # apply's status = the plan's counts[3]: a rejected plan skips apply
        H["_all"].copy_(self._rb, non_blocking=True)  # counts, plan arrays and commit mask at once
        if self.dec.v_gate is not None:  # fp16 V clamp flags, read after the iteration completed
            _lib.check(L.call("optimus_v_saturated", H["vsat"].data_ptr(), 1, stream), "optimus_v_saturated")

    def _unmask_synthetic(self, M, stream) -> None:
        cfg, fwd, cr = self.cfg, self.dec.forward, self.caps[1]
        p = lambda t: t.data_ptr()
        L = _lib
        _lib.check(L.call(
            "optimus_device_row_src", p(M["counts"]), p(self.slots), p(M["cu_rows"]), p(M["row_req"]), cr,
            fwd.rows_per_slot, fwd.version * fwd.max_slots * fwd.rows_per_slot, p(M["row_src"]), stream),
            "device_row_src")
        dt = 0 if self.logits.dtype == torch.bfloat16 else 1
        if fwd.vocab_offset == 0:
            # K3 in one launch, row count from the device plan
            ops.unmask_fused(self.logits, M["row_src"], cr, self.n_vsplit, M["cu_rows"], M["row_req"],
                             self.k3_counters, cfg.confidence_threshold, cfg.fallback, result=self.res,
                             part=self.part, n_rows_dev=M["counts"][1:], stream=torch.cuda.ExternalStream(stream))
        else:
            _lib.check(L.call(
                "optimus_unmask_partials_dev", p(self.logits), dt, self.logits.stride(0), p(M["row_src"]), cr,
                p(M["counts"][1:]), self.logits.shape[-1], fwd.vocab_offset, self.n_vsplit, p(self.part), stream),
                "unmask_partials_dev")
            ops.unmask_finalize(self.part, 1, cr, self.n_vsplit, M["cu_rows"], cfg.confidence_threshold,
                                cfg.fallback, result=self.res, stream=torch.cuda.ExternalStream(stream))

    def capture(self) -> None:
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        # the captured step mutates the device state: capture on a scratch copy,
        # then restore it
        saved = {k: v.clone() for k, v in self.D.items()}
        with torch.cuda.stream(s):
            self._enqueue(s.cuda_stream)  # warm (lazy kernel attributes)
            s.synchronize()
            self.graphs = []
            for H in self.Hs:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self._enqueue(s.cuda_stream, H)
                self.graphs.append(g)
        torch.cuda.synchronize()
        for k, v in saved.items():
            self.D[k].copy_(v)
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ host
    def set_chunk(self, chunk) -> None:
        """Chunk size(s) for the next launched iteration: one int for the batch (the
        elastic scheduler's per-iteration choice) or one per loop position.  Stream-
        ordered before the next replay; no re-capture."""
        c = np.asarray(chunk if np.ndim(chunk) else [chunk] * self.n, dtype=np.int32)
        if c.shape != (self.n,) or c.min() < 2 or c.max() > self.chunk:
            raise ConfigError(f"DeviceLoop.set_chunk: chunks must be in [2, {self.chunk}] (the capacity chunk), "
                              f"one per position")
        if np.array_equal(c, self.chunk_h):
            return
        if self._chunks_ev is not None:
            self._chunks_ev.synchronize()  # the previous staging copy has read the pinned buffer
        self._chunks_pin.numpy()[:] = c
        self.chunks_d.copy_(self._chunks_pin, non_blocking=True)
        self._h2d += c.nbytes
        self._chunks_ev = torch.cuda.Event()
        self._chunks_ev.record()
        self.chunk_h = c

    def step(self, summaries: bool = True, chunk=None):
        """One iteration: replay the graph, then replay the same transitions on the
        host mirror (Request objects) from the copied plan and commit mask.

        ``chunk`` (optional) sets the chunk size(s) first (``set_chunk``).

        With ``lookahead`` the next iteration's graph is launched before the host
        apply of this one (the device state is already advanced), so the host work
        overlaps the GPU; a request admitted by ``replace`` — and a chunk given here —
        then takes effect one iteration later (the in-flight iteration was planned
        with the previous state)."""
        if not self.graphs:
            self.capture()
        if chunk is not None:
            self.set_chunk(chunk)
        self.flush_admissions()
        # per-step copies: what this step's host calls staged (admissions, chunks) and the
        # plan arrays + commit mask every replay reads back
        self.h2d_bytes, self._h2d = self._h2d, 0
        self.d2h_bytes = (self.H["_all"].numel() + self.H["vsat"].numel()) * 4
        t0 = time.perf_counter()
        if not self.lookahead:
            self.graphs[0].replay()
            torch.cuda.current_stream().synchronize()
            H = self.Hs[0]
        else:
            if not self._inflight:  # first call: this iteration was not launched yet
                self.graphs[self._cur].replay()
                self._events[self._cur].record()
            # the next iteration goes in before this one is waited for: the GPU never idles
            # on the host (its plan reads the state this one leaves; its read-back buffers
            # are the other graph's)
            nxt = len(self.graphs) - 1 - self._cur
            self.graphs[nxt].replay()
            self._events[nxt].record()
            self._events[self._cur].synchronize()
            H = self.Hs[self._cur]
            self._cur = nxt
            self._inflight = True
        self.t_device += time.perf_counter() - t0
        if self.dec.v_gate is not None:
            vs = H["vsat"]
            if int(vs[0]) or int(vs[1]):
                vs.zero_()
                raise ConfigError("fp16 V cache: V values beyond +-65504 were clamped (cvt.satfinite); this "
                                  "model's V range needs a bf16 V cache (DecodeConfig(v_dtype=torch.bfloat16))")
        n = self.n
        n_tok, n_rows = int(H["counts"][0]), int(H["counts"][1])
        if int(H["counts"][3]) != 0:
            raise ConfigError("device step rejected (plan capacity / chunk bounds, or an illegal commit); "
                              "the device state was left unchanged")
        if int(H["wcounts"][3]) != 0:
            raise ConfigError("device attention planner rejected the step (work / group capacity)")
        cu = H["cu_seqlens"].numpy()[: n + 1].copy()
        cur = H["cu_rows"].numpy()[: n + 1].copy()
        tok_pos = H["tok_pos"].numpy()[: max(n_tok, 1)].copy()
        row_pos = H["row_pos"].numpy()[: max(n_rows, 1)].copy()
        mask = H["mask"].numpy()[: max(n_rows, 1)].copy()
        stale, self._stale = sorted(self._stale), set()
        # positions refilled after this iteration was launched: it planned nothing for
        # them (their previous request had finished); drop them from the host replay
        for i in stale:
            if cu[i] != cu[i + 1] or cur[i] != cur[i + 1]:
                raise ConfigError("DeviceLoop: a refilled position was planned by the in-flight iteration")
        keep = np.setdiff1d(np.arange(n), stale) if stale else None
        slots_c = np.ascontiguousarray(self.slots_h[keep] if stale else self.slots_h)
        cu_c = np.ascontiguousarray(np.delete(cu, stale) if stale else cu)
        cur_c = np.ascontiguousarray(np.delete(cur, stale) if stale else cur)
        m = len(slots_c)
        commits = np.zeros(m, dtype=np.int32)
        bs = self.bs
        bp = self.nat._bsp
        st = self.nat.lib.optimus_host_apply(
            m, slots_c.ctypes.data, self.cfg.block_size, cu_c.ctypes.data, tok_pos.ctypes.data,
            cur_c.ctypes.data, row_pos.ctypes.data, mask.ctypes.data, bp["states"], bs.states.shape[1],
            bp["queue"], bs.qcap, bp["q_head"], bp["q_len"], bp["block_index"], bp["committed"],
            bp["steps_taken"], bp["cached_prefix"], bp["out_len"], commits.ctypes.data)
        _lib.check(st, "optimus_host_apply")
        self._last = (cur, row_pos, mask)
        for i, r in enumerate(self.requests):  # finished: release pages and slot (it plans nothing)
            if i not in self.free and r.finished:
                self.nat.release(r)
                self.free.add(i)
        if not summaries:
            return int(commits.sum())
        out = []
        for r in range(n):
            a, b = int(cur[r]), int(cur[r + 1])
            out.append(StepSummary(computed=int(cu[r + 1] - cu[r]),
                                   commits=frozenset(row_pos[a:b][mask[a:b].astype(bool)].tolist())))
        return out

    def window_observations(self) -> list:
        """(window size, committed window ranks) of every position that had a window in
        the last iteration, in position order: what ElasticChunk's estimator folds in
        per request-step (sim.py:289-293, ``CommitEstimator.observe``)."""
        cur, row_pos, mask = self._last
        out = []
        for r in range(self.n):
            a, b = int(cur[r]), int(cur[r + 1])
            if b > a:
                out.append((b - a, set(np.flatnonzero(mask[a:b]).tolist())))
        return out

    def drain(self) -> None:
        """Wait for an in-flight lookahead iteration and discard it (its effects on
        the device state are kept: call only when every request has finished)."""
        self.flush_admissions()
        if self._inflight:
            torch.cuda.current_stream().synchronize()
            self._inflight = False
            self._cur = 0

    def replace(self, i: int, request) -> None:
        """Continuous batching: admit `request` into loop position i, whose request
        finished (released by step()).  The new request's batch-state row and
        block-table row are copied into the device state the graph reads; the graph
        itself is unchanged (it reads the slot map and the state by pointer)."""
        if i not in self.free:
            raise ConfigError(f"DeviceLoop.replace: position {i} still holds a live request")
        self._check_request(request, self.nat)
        # the position keeps its batch slot: another free position's slot map still
        # points at its own (finished, idle) slot
        s = self.nat._slot(request, int(self.slots_h[i]))
        self.dec.tables.ensure(s, request.prompt_tokens + request.output_tokens)
        bs = self.bs
        # the slot's packed rows as one record (flush_admissions copies them in)
        rec = np.empty(self._rec_ints, dtype=np.int32)
        rec[0] = s
        for j, k in enumerate(("q_head", "q_len", "block_index", "committed", "steps_taken", "cached_prefix",
                               "prompt", "out_len")):
            rec[1 + j] = getattr(bs, k)[s]
        sw = bs.states.shape[1] // 4
        rec[9: 9 + sw] = np.ascontiguousarray(bs.states[s]).view(np.int32)
        rec[9 + sw: 9 + sw + bs.qcap] = bs.queue[s]
        rec[9 + sw + bs.qcap:] = self.dec.tables.table[s]
        self._pending = [r for r in self._pending if r[0] != s] + [rec]
        self.requests[i] = request
        self.free.discard(i)
        if self._inflight:
            self._stale.add(i)

    def flush_admissions(self) -> None:
        """Copy the pending admissions into the device state: one H2D of the packed
        records + one optimus_device_admit launch, stream-ordered after any in-flight
        iteration (step() calls it before each replay)."""
        if not self._pending:
            return
        recs = np.stack(self._pending)
        m = len(recs)
        if self._adm_ev is not None:
            self._adm_ev.synchronize()  # the previous flush's copy has read the pinned buffer
        self._adm_pin.numpy()[:m] = recs
        self._adm_dev[:m].copy_(self._adm_pin[:m], non_blocking=True)
        D, p = self.D, lambda t: t.data_ptr()
        _lib.check(_lib.call(
            "optimus_device_admit", m, p(self._adm_dev), p(D["states"]), D["states"].shape[1], p(D["queue"]),
            self.bs.qcap, p(D["q_head"]), p(D["q_len"]), p(D["block_index"]), p(D["committed"]),
            p(D["steps_taken"]), p(D["cached_prefix"]), p(D["prompt"]), p(D["out_len"]), p(self.Dt),
            self.Dt.shape[1], torch.cuda.current_stream().cuda_stream), "optimus_device_admit")
        self._adm_ev = torch.cuda.Event()
        self._adm_ev.record()
        self._h2d += recs.nbytes
        self._pending = []

    def finished(self) -> bool:
        return all(r.finished for r in self.requests)
