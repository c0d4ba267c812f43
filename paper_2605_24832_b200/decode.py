"""The per-step decode call on B200: plan-all -> one device step -> apply-all.

Reference call chain (``pkg/src/dllmsim/sim.py:269-305``, streaming branch of
``_Loop.run_decode``): for each request of the batch ``plan_chunk`` ->
``oracle.commits(req, plan.window)`` -> ``consume`` -> ``apply_chunk``, then one
latency charge for the whole batch.  Every per-request input is request-local
(SURVEY §3.2), so reordering into plan-all / device step / apply-all changes no
output; ``StreamingDecoder.step`` does exactly that with the real forward in the
middle:

    host:   plans = plan_batch(batch, chunk, B, rule)            (engine.py mirror)
            meta  = build_step_meta(...) -> ONE pinned H2D copy
    device: for each layer: forward.qkv -> K1 kv_append -> K2 paged_attn
                            -> forward.post_attn
            forward.logits (window rows) -> K3 unmask partials + finalize
    host:   ONE D2H of commit masks/tokens -> apply_batch       (engine.py mirror)

``B200Oracle`` is the same device step behind the reference's oracle protocol
(``commits(request, window)`` / ``consume``, engine.py:105-110, sim.py:278-280)
so it plugs into ``Scenario.oracle_factory`` (sim.py:64) unchanged.
"""

from __future__ import annotations

import os

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import ops
from .core import rule_value
from .engine import ChunkPlan, StepSummary, apply_batch, apply_block, plan_batch, plan_block
from .errors import ConfigError
from .kvcache import BlockTables, PagedKVCache, PagePool
from .meta import DeviceMeta, build_step_meta


@dataclass(frozen=True)
class DecodeConfig:
    """Knobs of the decode path.

    ``block_size`` / ``window_rule`` / chunk size are the reference's knobs
    (scheduler.py:140-200); ``confidence_threshold``, ``page_size``,
    ``fallback`` and the model shape are new (SURVEY §5 config keys).
    """

    num_layers: int = 36
    num_q_heads: int = 32
    num_kv_heads: int = 8
    head_dim: int = 128
    vocab: int = 151936
    block_size: int = 32
    page_size: int = 64
    window_rule: str = "in_block"
    confidence_threshold: float = 0.9
    fallback: str = "earliest"
    max_batch: int = 64
    max_pages_per_req: int = 512
    num_pages: int = 16384
    min_split_tiles: int = 4
    logits_dtype: torch.dtype = torch.bfloat16
    # V cache dtype: fp16 (default: one fp16 P.V MMA in K2; bf16 V values beyond +-65504
    # are clamped and flagged, see ops.VRangeGate) or bf16 (exact, two MMAs)
    v_dtype: torch.dtype = torch.float16
    max_output_tokens: int = 4096   # per-request capacity of the packed native state
    # StreamingDecoder.step backend: "host" (C++ host plan -> H2D -> device step -> D2H ->
    # host apply), "loop" (the graph-captured DeviceLoop: planning on the device, one graph
    # per iteration; same results) or "loop_lookahead" (the next iteration is launched
    # before step() returns: admissions and chunk changes take effect one call later)
    step_backend: str = "host"
    max_chunk: int = 64

    def __post_init__(self):
        if self.num_q_heads % self.num_kv_heads:
            raise ConfigError("num_q_heads must be a multiple of num_kv_heads")
        if not 0.0 < self.confidence_threshold <= 1.0:
            raise ConfigError("confidence_threshold must lie in (0, 1]")
        rule_value(self.window_rule)
        if self.fallback not in ops.FALLBACK_MODES:
            raise ConfigError(f"fallback must be one of {sorted(ops.FALLBACK_MODES)}")
        if self.step_backend not in ("host", "loop", "loop_lookahead"):
            raise ConfigError("step_backend must be 'host', 'loop' or 'loop_lookahead'")


class Forward:
    """What the decode step needs from the model (the reference has none:
    ``SPEC.md:14`` puts weights out of scope).  Implementations: synthetic
    SDAR-shaped activations (bench / parity) and a tiny random-init dLLM."""

    def begin_step(self, dmeta: DeviceMeta) -> None:  # pragma: no cover - interface
        pass

    def qkv(self, layer: int, dmeta: DeviceMeta):  # -> (q [n,Hq,d], k [n,Hkv,d], v [n,Hkv,d])
        raise NotImplementedError

    def post_attn(self, layer: int, attn_out: torch.Tensor, dmeta: DeviceMeta) -> None:
        pass

    def logits(self, dmeta: DeviceMeta):  # -> (logits [rows, V], row_src or None)
        raise NotImplementedError


class StreamingDecoder:
    """Batched streaming chunked block decoding over a paged KV cache."""

    def __init__(self, cfg: DecodeConfig, forward: Forward, device="cuda",
                 cache: Optional[PagedKVCache] = None):
        self.cfg = cfg
        self.forward = forward
        self.device = torch.device(device)
        self.cache = cache or PagedKVCache(cfg.num_layers, cfg.num_pages, cfg.num_kv_heads,
                                           cfg.page_size, cfg.head_dim, device=self.device, v_dtype=cfg.v_dtype)
        # fp16 V: every step's D2H point also reads the clamp flags (ops.VRangeGate)
        self.v_gate = ops.VRangeGate() if self.cache.v.dtype == torch.float16 else None
        if self.v_gate is not None and torch.cuda.is_available():
            # the flags are per process: start from a clean state (earlier clamps were
            # reported, or belong to caches this decoder never reads)
            self.v_gate.issue()
            torch.cuda.current_stream().synchronize()
            self.v_gate.buf.zero_()
        self.pool = PagePool(self.cache.num_pages)
        self.tables = BlockTables(self.pool, cfg.max_batch, cfg.max_pages_per_req, cfg.page_size)
        self.grid = ops.sm_count()
        self._pinned = None
        self._dev_buf = None
        self._ws_o = None
        self._ws_ml = None
        self._attn_out = None
        self.last_meta: Optional[DeviceMeta] = None
        self.last_plan: Optional[ops.AttnPlan] = None
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        # multi-GPU: a TensorParallelUnmask merges vocab-shard partials across ranks
        self.unmask_impl = None
        self._loop = None  # DeviceLoop behind step() when cfg.step_backend != "host"
        self._unmask_counters = None  # K3 arrival counters (unmask_fused), zero between launches
        # native (C++) batched host step over packed request state; the Python path
        # (step_python) stays for foreign callers and as the readable specification
        self.use_native = True
        # fold K1 into K2 (optimus_paged_attn_append) whenever every request's query
        # tokens fit one MMA tile (chunk x Hq/Hkv <= 128)
        # per-layer KV append: "k1" = K1 then K2 (default), "slots" = K1 over the step's
        # slot map, "fused" = K1 folded into K2 (needs one query tile per request).
        # Interleaved A/B (tools/ab_step.py): fused -0.8% at ShareGPT, +4.6% at 4K;
        # slots = k1 within noise.
        # K1 form: "slots" = the step's slot map once, then one round trip per row in every
        # layer (default: ShareGPT / LLaDA whole step -1.2% against "k1", gpurun r2d7);
        # "k1" = each layer's K1 derives the slots itself; "fused" = K1 folded into K2
        self.append_mode = os.environ.get("OPTIMUS_APPEND", "slots")
        self._native = None

    # ------------------------------------------------------------------ admission
    def admit(self, request, slot=None) -> int:
        """Give a request a batch slot (`slot` if given) and pages for its prompt +
        first block."""
        first = min(request.output_tokens, self.cfg.block_size)
        return self.tables.admit(request.id, request.prompt_tokens + first, slot)

    def release(self, request) -> None:
        if self._native is not None and getattr(request, "_bs", None) is self._native.bs:
            self._native.release(request)
        else:
            self.tables.release(request.id)

    def release_all(self, requests) -> None:
        if self._loop is not None:
            self._loop.drain()
            self._loop = None
        for r in requests:
            if self.tables.slot(r.id) is not None:
                self.release(r)

    def native(self):
        if self._native is None:
            from .native_step import NativeStepper

            self._native = NativeStepper(self, max_out=self.cfg.max_output_tokens,
                                         max_chunk=self.cfg.max_chunk)
        return self._native

    def _ensure_pages(self, requests, plans) -> np.ndarray:
        rows = np.empty(len(requests), dtype=np.int64)
        for i, (req, plan) in enumerate(zip(requests, plans)):
            slot = self.tables.slot(req.id)
            if slot is None:
                slot = self.admit(req)
            rows[i] = slot
            hi = max(plan.window[-1] if plan.window else -1,
                     max(plan.kv_positions) if plan.kv_positions else -1)
            if hi >= 0:
                self.tables.ensure(slot, req.prompt_tokens + hi + 1)
        return rows

    # ------------------------------------------------------------------ device step
    def prepare(self, requests: Sequence, plans: Sequence[ChunkPlan]) -> DeviceMeta:
        rows = self._ensure_pages(requests, plans)
        bt = self.tables.table[rows]
        meta = build_step_meta(requests, plans, self.cfg.block_size, bt)
        dm = DeviceMeta.upload(meta, self.device, self._pinned, self._dev_buf)
        self._pinned = dm.__dict__["pinned"]
        self._dev_buf = dm.buf
        self.h2d_bytes = dm.h2d_bytes
        plan = ops.plan_attention(meta.cu_seqlens, meta.key_end, self.cfg.num_q_heads,
                                  self.cfg.num_kv_heads, grid=self.grid,
                                  min_split_tiles=self.cfg.min_split_tiles, device=self.device,
                                  page_size=self.cfg.page_size)
        self.h2d_bytes += plan.work_host.nbytes + plan.cta_off_host.nbytes + plan.groups_host.nbytes
        dm.__dict__["attn_plan"] = plan
        dm.__dict__["slots"] = rows
        dm.__dict__["requests"] = requests
        dm.__dict__["plans"] = plans
        self.last_meta = dm
        self.last_plan = plan
        return dm

    def _workspaces(self, plan: ops.AttnPlan, n_tok: int):
        cfg = self.cfg
        if plan.n_partials:
            need = plan.n_partials * 128 * cfg.head_dim
            if self._ws_o is None or self._ws_o.numel() < need:
                self._ws_o = torch.empty(need, dtype=torch.float32, device=self.device)
                self._ws_ml = torch.empty(plan.n_partials * 256, dtype=torch.float32, device=self.device)
            elif self._ws_ml.numel() < plan.n_partials * 256:
                self._ws_ml = torch.empty(plan.n_partials * 256, dtype=torch.float32, device=self.device)
        shape = (max(n_tok, 1), cfg.num_q_heads, cfg.head_dim)
        if self._attn_out is None or self._attn_out.shape[0] < shape[0]:
            self._attn_out = torch.empty(shape, dtype=torch.bfloat16, device=self.device)
        return self._attn_out[: max(n_tok, 1)]

    def run_layers(self, dm: DeviceMeta) -> None:
        """K1 + K2 for every layer (the part repeated L times per step)."""
        cfg = self.cfg
        m = dm.host
        plan = dm.__dict__["attn_plan"]
        out = self._workspaces(plan, m.n_tok)
        if getattr(self.forward, "resident_layers", False) and m.n_tok:
            # activations already resident for every layer: one native call enqueues
            # all K1/K2 launches (csrc/capi.cu optimus_attn_layers)
            self._run_layers_native(dm, plan, out)
            return
        self.forward.begin_step(dm)
        fused = bool(m.n_tok and plan.single_tile and self.append_mode == "fused")
        slot_abs = (ops.slot_mapping(dm.tok_req, dm.tok_pos, dm.prompt_len, dm.block_tables, cfg.page_size,
                                     n_tok=m.n_tok) if m.n_tok and self.append_mode != "k1" else None)
        for layer in range(cfg.num_layers):
            q, k, v = self.forward.qkv(layer, dm)
            kc, vc = self.cache.layer(layer)
            if fused:
                ops.paged_attention_append(q, k, v, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base,
                                           dm.vis_off, dm.vis_words, dm.block_tables, plan,
                                           cfg.block_size, out=out[: m.n_tok], ws_o=self._ws_o,
                                           ws_ml=self._ws_ml, slot_abs=slot_abs)
            elif m.n_tok:
                ops.kv_append(k, v, dm.tok_req, dm.tok_pos, dm.prompt_len, dm.block_tables, kc, vc,
                              slot_abs=slot_abs)
                ops.paged_attention(q, kc, vc, dm.tok_pos, dm.prompt_len, dm.vis_base, dm.vis_off,
                                    dm.vis_words, dm.block_tables, plan, cfg.block_size,
                                    out=out[: m.n_tok], ws_o=self._ws_o, ws_ml=self._ws_ml)
            self.forward.post_attn(layer, out[: m.n_tok], dm)

    def _slot_ws_ptr(self, n_tok: int) -> int:
        """int32 [2, n_tok] workspace of the fused append's per-step slot map."""
        ws = self.__dict__.get("_slot_ws")
        if ws is None or ws.numel() < 2 * max(n_tok, 1):
            ws = torch.empty(2 * max(n_tok, 1024), dtype=torch.int32, device=self.device)
            self._slot_ws = ws
        return ws.data_ptr()

    def _run_layers_native(self, dm, plan, out) -> None:
        import ctypes as C

        from . import _lib

        cfg = self.cfg
        m = dm.host
        L = cfg.num_layers
        ptrs = self.__dict__.get("_layer_ptrs")
        if ptrs is None:
            q_l, k_l, v_l, kc_l, vc_l = [], [], [], [], []
            for layer in range(L):
                q, k, v = self.forward.qkv(layer, dm)
                kc, vc = self.cache.layer(layer)
                q_l.append(q.data_ptr()); k_l.append(k.data_ptr()); v_l.append(v.data_ptr())
                kc_l.append(kc.data_ptr()); vc_l.append(vc.data_ptr())
                strides = (q.stride(0), k.stride(0), self.forward.qkv_capacity)
            arr = lambda xs: (C.c_void_p * L)(*xs)
            ptrs = (arr(q_l), arr(k_l), arr(v_l), arr(kc_l), arr(vc_l), strides)
            self._layer_ptrs = ptrs
        q_a, k_a, v_a, kc_a, vc_a, (q_stride, kv_stride, cap) = ptrs
        out_a = (C.c_void_p * L)(*([out.data_ptr()] * L))
        mode = {"k1": 0, "slots": 1, "fused": 2 if plan.single_tile else 1}[self.append_mode]
        kc0 = self.cache.k[0]
        st = _lib.call(
            "optimus_attn_layers", L, q_a, k_a, v_a, q_stride, kv_stride, cap, m.n_tok, kc_a, vc_a,
            kc0.shape[0], dm.tok_req.data_ptr(), dm.tok_pos.data_ptr(), dm.prompt_len.data_ptr(),
            dm.vis_base.data_ptr(), dm.vis_off.data_ptr(), dm.vis_words.data_ptr(),
            dm.block_tables.data_ptr(), dm.block_tables.shape[1], plan.work.data_ptr(),
            plan.cta_off.data_ptr(), plan.grid if plan.n_work else 0, plan.groups.data_ptr(),
            plan.n_groups, cfg.block_size, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim,
            cfg.page_size, 1.0 / float(cfg.head_dim) ** 0.5, out_a, out.stride(0),
            self._ws_o.data_ptr() if plan.n_partials else None,
            self._ws_ml.data_ptr() if plan.n_partials else None,
            ops._v_dtype(self.cache.v), mode, self._slot_ws_ptr(m.n_tok) if mode else None,
            torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "optimus_attn_layers")

    def run_unmask(self, dm: DeviceMeta) -> ops.UnmaskResult:
        m = dm.host
        logits, row_src = self.forward.logits(dm)
        if self.unmask_impl is not None:
            return self.unmask_impl(self, dm, logits, row_src)
        n_vsplit = ops.unmask_splits(m.n_rows, logits.shape[-1])
        # per-decoder workspaces, grown on demand (no allocation per step)
        rows = max(m.n_rows, 1)
        ws = self.__dict__.get("_unmask_ws")
        if ws is None or ws[0].numel() < rows * n_vsplit * 3 or ws[1].commit_mask.numel() < rows:
            cap = max(rows, 2 * (ws[1].commit_mask.numel() if ws else 0), 256)
            part = torch.empty(cap * max(n_vsplit, 32) * 3, dtype=torch.float32, device=self.device)
            res = ops.UnmaskResult(torch.empty(cap, dtype=torch.uint8, device=self.device),
                                   torch.empty(cap, dtype=torch.int32, device=self.device),
                                   torch.empty(cap, dtype=torch.float32, device=self.device))
            ws = self._unmask_ws = (part, res)
        if self._unmask_counters is None or self._unmask_counters.numel() < max(m.n_req, 1):
            self._unmask_counters = torch.zeros(max(m.n_req, self.cfg.max_batch, 1), dtype=torch.int32,
                                                device=self.device)
        # one launch: the CTA completing a request's vocab slices finalizes it
        return ops.unmask_fused(logits, row_src, m.n_rows, n_vsplit, dm.cu_rows, dm.row_req, self._unmask_counters,
                                self.cfg.confidence_threshold, self.cfg.fallback, result=ws[1],
                                part=ws[0][: rows * n_vsplit * 3].view(rows, n_vsplit, 3))

    def device_step(self, dm: DeviceMeta) -> ops.UnmaskResult:
        self.run_layers(dm)
        return self.run_unmask(dm)

    def fetch_commits(self, dm: DeviceMeta, res: ops.UnmaskResult) -> list:
        """One D2H copy of the commit mask -> per-request commit sets."""
        m = dm.host
        if self.v_gate is not None:
            self.v_gate.issue()
        if m.n_rows == 0:
            torch.cuda.current_stream().synchronize()
            if self.v_gate is not None:
                self.v_gate.check()
            return [set() for _ in range(m.n_req)]
        mask = res.commit_mask[: m.n_rows].cpu().numpy().astype(bool)
        if self.v_gate is not None:
            self.v_gate.check()
        self.d2h_bytes = m.n_rows
        rows = np.flatnonzero(mask)
        req_of = m.row_req[rows]
        pos = m.row_pos[rows]
        out = [set() for _ in range(m.n_req)]
        for r, p in zip(req_of.tolist(), pos.tolist()):
            out[r].add(p)
        return out

    # ------------------------------------------------------------------ the call
    def step(self, requests: Sequence, chunk_size) -> list:
        """One streaming decode iteration for the whole batch (sim.py:269-305)."""
        if self.cfg.step_backend != "host":
            return self._loop_step(requests, chunk_size)
        if self.use_native:
            nat = self.native()
            out = nat.step(requests, chunk_size)
            self.h2d_bytes, self.d2h_bytes = nat.h2d_bytes, nat.d2h_bytes
            return out
        return self.step_python(requests, chunk_size)

    def step_baseline(self, requests: Sequence, mode: str) -> list:
        """One iteration of a baseline policy on the same kernels: the
        batched twin of _Loop.run_decode's AR / block branches (sim.py:253-267) —
        ``mode`` "bd" (block_diffusion_step), "prefix" (prefix_cached_step) or "ar"
        (ar_step, engine.py:98-157).  One device step (K1, K2, K3) for the batch, then
        the reference's state rules per request."""
        cfg = self.cfg
        block = cfg.block_size
        plans = [plan_block(r, block, mode) for r in requests]
        dm = self.prepare(requests, plans)
        res = self.device_step(dm)
        commits = self.fetch_commits(dm, res)
        if mode == "ar":  # the next position commits whatever its confidence
            commits = [{p.window[0]} for p in plans]
        summaries = [apply_block(r, p, c, block, mode) for r, p, c in zip(requests, plans, commits)]
        for req in requests:
            if req.finished:
                self.release(req)
        return summaries

    def _loop_step(self, requests: Sequence, chunk_size) -> list:
        """``step`` on the graph-captured DeviceLoop.  The loop keeps one position per
        request of the first call; later calls may drop FINISHED requests and bring new
        ones into the freed positions (``DeviceLoop.replace``); the chunk may change
        every call (elastic, up to ``max_chunk``)."""
        from .device_loop import DeviceLoop

        reqs = list(requests)
        look = self.cfg.step_backend == "loop_lookahead"
        L = self._loop
        if L is None:
            self._loop = L = DeviceLoop(self, reqs, chunk_size, lookahead=look,
                                        max_chunk=max(int(np.max(chunk_size)), 32))
        else:
            ids = {r.id for r in reqs}
            pos = {r.id: i for i, r in enumerate(L.requests) if i not in L.free}
            if any(rid not in ids for rid in pos):
                raise ConfigError("step_backend loop: a live request left the batch before finishing "
                                  "(only finished requests may be dropped)")
            new = [r for r in reqs if r.id not in pos]
            free = sorted(L.free)
            if len(new) > len(free):
                raise ConfigError(f"step_backend loop: {len(new)} new requests but {len(free)} free positions "
                                  f"(the loop holds {L.n}; start it with the full batch)")
            for i, r in zip(free, new):
                L.replace(i, r)
        where = {r.id: i for i, r in enumerate(L.requests)}
        if np.ndim(chunk_size):
            per = np.full(L.n, int(np.min(chunk_size)), dtype=np.int32)
            for r, c in zip(reqs, chunk_size):
                per[where[r.id]] = c
            chunk = per
        else:
            chunk = int(chunk_size)
        summ = L.step(chunk=chunk)
        self.h2d_bytes, self.d2h_bytes = L.h2d_bytes, L.d2h_bytes
        return [summ[where[r.id]] for r in reqs]

    def step_python(self, requests: Sequence, chunk_size: int) -> list:
        """The same iteration with the host half in Python (plan_batch / apply_batch)."""
        cfg = self.cfg
        plans = plan_batch(requests, chunk_size, cfg.block_size, cfg.window_rule)
        dm = self.prepare(requests, plans)
        res = self.device_step(dm)
        commits = self.fetch_commits(dm, res)
        summaries = apply_batch(requests, plans, commits, cfg.block_size)
        for req in requests:
            if req.finished:
                self.release(req)
        return summaries


class B200Oracle:
    """The reference's commit-oracle protocol served by the B200 decode step.

    Plugs into ``Scenario.oracle_factory`` (sim.py:64,128-132) unchanged:
    ``commits(request, window)`` (commit.py:279-280 signature) runs one device step
    (K1 -> K2 per layer -> K3) for that request; ``commits_batch(requests, plans)``
    runs ONE device step for a whole batch (the batched twin of the loop, see
    ``sim_bridge.BatchedLoop``).  ``consume`` (commit.py:310-312) is forwarded to the
    forward when it wants it (reference-oracle-driven logits).

    KV bookkeeping.  The reference calls the oracle only when the plan's window is
    non-empty (sim.py:278), yet ``apply_chunk`` still marks that plan's kv positions
    DECODED_CACHED (engine.py:84-88): a step whose backlog filled the whole chunk
    (engine.py:58-59) never reaches the device.  So the oracle keeps, per request,
    the positions it committed in commit order (the device's view of the FIFO) and
    how many of them the device has recomputed; every device step recomputes the
    missed ones first, then the plan's own kv positions (rule K: each committed
    position's final KV is computed exactly once, with its committed token).  A
    request's pages are released when the commits returned finish it.
    """

    def __init__(self, decoder: StreamingDecoder, mode: str = "stream"):
        self.decoder = decoder
        self.mode = mode  # "stream" (chunked), or the block baselines "bd" / "prefix"
        self._cache: dict = {}
        self._fifo: dict = {}   # request id -> positions committed through this oracle, in order
        self._sent: dict = {}   # request id -> how many of them the device has recomputed
        self.recomputed: dict = {}  # request id -> positions recomputed as kv rows, in order (diagnostics)
        self.device_steps = 0

    # ------------------------------------------------------------------ bookkeeping
    def _track(self, req):
        if req.id not in self._fifo:  # first sight: the current backlog is what is pending
            self._fifo[req.id] = [int(p) for p in req.uncached_queue]
            self._sent[req.id] = 0
            self.recomputed[req.id] = []
        return self._fifo[req.id]

    def _device_plan(self, req, plan: ChunkPlan) -> tuple:
        """(kv rows the device recomputes this step, index past them in the fifo)."""
        fifo = self._track(req)
        sent = self._sent[req.id]
        queue = [int(p) for p in req.uncached_queue]
        pending = fifo[sent:]
        if queue and queue != pending[len(pending) - len(queue):]:
            raise ConfigError(f"B200Oracle: request {req.id}'s uncached queue is not the tail of the positions "
                              f"this oracle committed (was it committed by another oracle?)")
        kv = tuple(int(p) for p in plan.kv_positions)
        if tuple(queue[: len(kv)]) != kv:
            raise ConfigError(f"B200Oracle: request {req.id}'s kv positions are not its FIFO head (engine.py:58)")
        end = sent + (len(pending) - len(queue)) + len(kv)  # missed kv-only steps, then this plan's kv
        return tuple(fifo[sent:end]), end

    def _finish(self, req, committed) -> None:
        self._fifo[req.id].extend(sorted(int(p) for p in committed))
        if req.committed + len(committed) >= req.output_tokens:  # apply_chunk will finish it
            if self.decoder.tables.slot(req.id) is not None:
                self.decoder.release(req)
            for d in (self._fifo, self._sent, self.recomputed):
                d.pop(req.id, None)

    # ------------------------------------------------------------------ protocol
    def commits_batch(self, requests: Sequence, plans: Sequence[ChunkPlan]) -> list:
        result = [set() for _ in requests]
        if self.mode in ("bd", "prefix"):
            idx = [i for i, p in enumerate(plans) if p.kv_positions or p.window]
            dev_plans = [plans[i] for i in idx]
            ends = None
        else:
            idx, dev_plans, ends = [], [], []
            for i, (req, plan) in enumerate(zip(requests, plans)):
                kv, end = self._device_plan(req, plan)
                if kv or plan.window:
                    idx.append(i)
                    dev_plans.append(ChunkPlan(kv_positions=kv, window=tuple(plan.window)))
                    ends.append(end)
        sub_r = [requests[i] for i in idx]
        if sub_r:
            dm = self.decoder.prepare(sub_r, dev_plans)
            res = self.decoder.device_step(dm)
            self.device_steps += 1
            for i, c in zip(idx, self.decoder.fetch_commits(dm, res)):
                result[i] = c
        if ends is not None:
            for i, dp, end in zip(idx, dev_plans, ends):
                req = requests[i]
                self.recomputed[req.id].extend(dp.kv_positions)
                self._sent[req.id] = end
        for req, c in zip(requests, result):
            if self.mode in ("bd", "prefix"):
                if req.committed + len(c) >= req.output_tokens and self.decoder.tables.slot(req.id) is not None:
                    self.decoder.release(req)
            else:
                self._finish(req, c)
        for req, plan, c in zip(requests, plans, result):
            if plan.window:  # the reference never asks about an empty window (sim.py:278)
                self._cache[(req.id, tuple(plan.window))] = c
        return result

    def commits(self, request, window) -> set:
        key = (request.id, tuple(window))
        if key in self._cache:
            return self._cache.pop(key)
        # Standalone use inside dllmsim's loop.  Streaming: a non-empty window means
        # plan_chunk had capacity left after the backlog (engine.py:58-59), so the
        # plan's kv positions are the whole uncached queue.  Block baselines: the
        # block step recomputes the block's decoded (bd) / uncached (prefix) positions.
        if self.mode in ("bd", "prefix"):
            plan = ChunkPlan(kv_positions=plan_block(request, self.decoder.cfg.block_size, self.mode).kv_positions,
                             window=tuple(window))
        else:
            plan = ChunkPlan(kv_positions=tuple(request.uncached_queue), window=tuple(window))
        [c] = self.commits_batch([request], [plan])
        self._cache.pop(key, None)
        return c

    def consume(self, request, committed) -> None:
        fn = getattr(self.decoder.forward, "consume", None)
        if fn is not None:
            fn(request, committed)


def run_decode_batched(decoder: StreamingDecoder, batch: Sequence, chunk_size: int) -> tuple:
    """Batched twin of ``_Loop.run_decode``'s streaming branch: returns
    (computed_tokens, committed_tokens, summaries) for the iteration record."""
    summaries = decoder.step(batch, chunk_size)
    computed = sum(s.computed for s in summaries)
    committed = sum(len(s.commits) for s in summaries)
    return computed, committed, summaries
