"""One forward step over a batch of new-token rows, on the device.

Reference: model.py:126-193 (``forward_step`` / ``_forward_group``).  The
reference runs one group (message) at a time and never batches across messages;
here every row of every message in the step goes through one pass:

    embed -> per layer [ residual+RMSNorm -> QKV GEMM -> K1 rope_append (q rotated,
    K/V written into the message's pages) -> K5 split-KV attention over the
    K3-assembled page lists -> combine -> O GEMM -> residual+RMSNorm -> gate|up
    GEMM -> SiLU*up -> down GEMM ] -> final norm on the logit rows -> head GEMM.

New K/V are appended inside the step (before attention), so rows of the same
message see each other causally through the pool while batch peers — which are
never in each other's page lists — stay invisible, exactly as the reference's
mask [ones(T, n_ctx) | tril(T, T)] (model.py:166-168).  Dense projections are
cuBLAS GEMMs via torch (bf16 in, f32 accumulate); the residual stream is f32.
"""

from __future__ import annotations

import ctypes
import itertools
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .cache import DeviceKvCache, RotationTableDevice, cdiv, h2d
from .weights import DeviceWeights

RMS_EPS = 1e-6  # model.py:28


@dataclass
class CallRows:
    """Rows one message contributes to a step (tokens at consecutive positions)."""

    msg: int
    parents: list
    first_t: int  # within-message index of the first new token
    tokens: list
    pages: np.ndarray
    slots: np.ndarray
    offset: int  # message offset (position of token 0)


@dataclass
class StepPlan:
    calls: list
    logit_rows: np.ndarray  # row indices needing logits
    # pipelined decode: row r embeds sel_src[sel[r]] (a device-selected token of the previous
    # step, still unknown to the host) when sel[r] >= 0
    sel: np.ndarray | None = None
    sel_src: torch.Tensor | None = None

    @property
    def n_rows(self) -> int:
        return sum(len(c.tokens) for c in self.calls)


@dataclass
class Plan:
    """Host replica of K3's page-centric sizing (assemble.cu) for buffer capacities."""

    n_vis: int
    n_blk_rows: int
    n_items: int
    n_parts: int
    max_row_parts: int
    item_pages: int  # sum over items of pages (work estimate)


def plan_counts(calls: list, msg_len: np.ndarray, P: int, rpb: int, ppi: int,
                mode: int = 0) -> Plan:
    """Host replica of K3's sizing; mode 0 page-centric, mode 1 per-call (assemble.cu)."""
    if mode == 1:
        n_vis = n_blk = n_items = n_parts = item_pages = max_row = 0
        for c in calls:
            n = len(c.tokens)
            if n == 0:
                continue
            pp = sum(cdiv(int(msg_len[p]), P) for p in c.parents)
            n_vis += pp + (c.first_t + n - 1) // P + 1
            n_blk += n
            for b in range(0, n, rpb):
                nr = min(rpb, n - b)
                nvis = pp + (c.first_t + b + nr - 1) // P + 1
                ch = cdiv(nvis, ppi)
                n_items += ch
                n_parts += ch * nr
                item_pages += nvis
                max_row = max(max_row, ch)
        return Plan(n_vis, n_blk, n_items, n_parts, max_row, item_pages)
    groups: dict = {}
    for c in calls:
        for p in c.parents:
            groups[p] = groups.get(p, 0) + len(c.tokens)
    n_vis = n_blk = n_items = n_parts = item_pages = 0
    for p, rows in groups.items():
        pages = cdiv(int(msg_len[p]), P)
        n_vis += pages
        n_blk += rows
        if rows:
            ch = cdiv(pages, ppi)
            n_items += cdiv(rows, rpb) * ch
            n_parts += rows * ch
            item_pages += cdiv(rows, rpb) * pages
    max_row = 0
    for c in calls:
        n = len(c.tokens)
        if n == 0:
            continue
        par_ch = sum(cdiv(cdiv(int(msg_len[p]), P), ppi) for p in c.parents)
        t_last = c.first_t + n - 1
        n_vis += t_last // P + 1
        n_blk += n
        for b in range(0, n, rpb):
            nr = min(rpb, n - b)
            own_pages = (c.first_t + b + nr - 1) // P + 1
            ch = cdiv(own_pages, ppi)
            n_items += ch
            n_parts += ch * nr
            item_pages += own_pages
            max_row = max(max_row, par_ch + ch)
    return Plan(n_vis, n_blk, n_items, n_parts, max_row, item_pages)


_STEP_TAGS = itertools.count(1)  # K3 step tags (process-unique; int32 range is plenty)
K3_MAX_CALLS = 1024  # assemble.cu kMaxCalls
K3_MAX_PAIRS = 4096  # assemble.cu kMaxPairs (page-centric mode)
K3_MAX_PARENT_ID = (1 << 21) - 1  # parent ids are packed as (parent << 11 | call)


def split_plan(plan: StepPlan) -> list:
    """Cut a step into [(sub-plan, per-call mode)] pieces that fit K3's limits.

    Greedy in call order (the logit rows stay in call order, so the pieces' logits
    concatenate to the step's).  A piece takes the per-call mode when one of its calls
    alone has more than K3_MAX_PAIRS parents or a parent id does not fit the sort key."""
    calls = plan.calls
    pairs = [len(c.parents) for c in calls]
    big_id = any(p > K3_MAX_PARENT_ID for c in calls for p in c.parents)
    if len(calls) <= K3_MAX_CALLS and sum(pairs) <= K3_MAX_PAIRS:
        return [(plan, big_id)]
    starts = np.cumsum([0] + [len(c.tokens) for c in calls])
    logit_rows = np.asarray(plan.logit_rows, np.int64)
    out, i = [], 0
    while i < len(calls):
        j, npair = i, 0
        while (j < len(calls) and j - i < K3_MAX_CALLS
               and (j == i or npair + pairs[j] <= K3_MAX_PAIRS)):
            npair += pairs[j]
            j += 1
        lo, hi = starts[i], starts[j]
        sel = logit_rows[(logit_rows >= lo) & (logit_rows < hi)] - lo
        percall = npair > K3_MAX_PAIRS or any(
            p > K3_MAX_PARENT_ID for c in calls[i:j] for p in c.parents)
        sub_sel = None if plan.sel is None else np.asarray(plan.sel[lo:hi], np.int32)
        out.append((StepPlan(calls[i:j], sel.astype(np.int32), sub_sel, plan.sel_src), percall))
        i = j
    return out


class Runner:
    """Executes StepPlans for one (weights, cache) pair on the current stream."""

    def __init__(self, weights: DeviceWeights, cache: DeviceKvCache,
                 rotation: RotationTableDevice, split_activations: bool = True,
                 tp=None, tp_group=None) -> None:
        """tp: parallel.TPLayout for KV-head tensor parallelism (None = whole model here);
        the partial o_proj / down_proj outputs are all-reduced over tp_group (NCCL)."""
        self.w = weights
        self.cache = cache
        self.rot = rotation
        self.tp, self.tp_group = tp, tp_group
        # self.cfg: this rank's slice (heads, kv heads, ffn); self.d: the global model dim
        self.cfg = tp.local_config() if tp is not None else weights.config
        self.d = tp.model_dim if tp is not None else weights.config.model_dim
        self.dt = weights.torch_dtype
        self.dtc = nat.dtype_code(self.dt)
        self.pool_dtc = nat.dtype_code(cache.dtype)
        self.dev = cache.device
        G = self.cfg.n_heads // self.cfg.kv_heads
        self.rows_per_block = max(1, min(16, 64 // G))
        self.launches = 0  # our kernels launched (for bench accounting)
        self.h2d_bytes = 0  # per-step metadata uploads (bench e2e accounting)
        # When set to a list, attention launches are bracketed with CUDA events on the
        # launching stream and (start, end, algorithmic_bytes) tuples are appended.
        self.attn_events = None
        self.step_events = None  # when a list: (start, end) events around each step's GPU work
        # bf16 engines carry GEMM activations as hi/lo bf16 pairs (see choreo_b200.h)
        self.split = self.dt == torch.bfloat16 and split_activations
        # K7 weight-streaming linear for decode-sized bf16 steps (cuBLAS above 128 GEMM rows)
        self.k7 = self.dt == torch.bfloat16 and os.environ.get("CHOREO_K7", "1") != "0"
        self._k7_ws = self._k7_cnt = None
        # decode-sized bf16 steps run their layer loop in the native executor
        # (choreo_decode_layers: one library call per step instead of ~11 per layer)
        self.native_step = os.environ.get("CHOREO_NATIVE_STEP", "1") != "0"
        # ... or (CHOREO_CHAIN=1, one process per model) run the projections between two
        # attentions as ONE K8 layer-chain launch (choreo_layer_chain).  Measured in situ at
        # the 8B decode step: on par with the per-GEMM K7 sequence (4.10-4.12 vs 4.07 ms), so
        # K7 stays the default
        self.chain = (self.dt == torch.bfloat16 and (tp is None or tp.size == 1)
                      and os.environ.get("CHOREO_CHAIN", "0") == "1")
        self._chain_bufs = None
        self.q_bulk = os.environ.get("CHOREO_Q_BULK", "1") != "0"
        self.wide_k4 = os.environ.get("CHOREO_WIDE_K4", "1") != "0"
        # K5 v2 unit schedule of multi-wave steps (no effect on results): longest-first snake
        # deal (default) or unit w to CTA w mod grid (CHOREO_V2_LPT=0, for A/B timing)
        self.v2_lpt = os.environ.get("CHOREO_V2_LPT", "1") != "0"
        self._wptrs = None
        self._ev_free: list = []
        self._ev_pending: list = []  # (kind, event array, bytes per pair) awaiting readback
        self.attn_times: list = []  # (ms, algorithmic bytes) per timed attention launch
        # When True (native decode steps only), the four K7 launches of every layer are
        # bracketed with events too; (ms, bytes) land in linear_times.  The brackets cost the
        # GEMM its programmatic-launch overlap, so these times are conservative.
        self.time_linear = False
        self.linear_times: list = []
        # synchronise after K3 and check its overflow flag (tests set CHOREO_CHECK_ASSEMBLY=1;
        # the host sizes every buffer from plan_counts, so a flag here is a planner bug)
        self.check_assembly = os.environ.get("CHOREO_CHECK_ASSEMBLY", "0") == "1"

    def _weight_ptrs(self):
        if self._wptrs is None:
            L = len(self.w.layers)
            self._wptrs = {n: (ctypes.c_void_p * L)(*[lw[n].data_ptr() for lw in self.w.layers])
                           for n in ("attn_norm", "w_qkv", "wo", "ffn_norm", "w_gu", "w_down")}
        return self._wptrs

    def _retire_events(self, keep: int) -> None:
        """Read back native K5 timing events older than `keep` steps (they completed long
        ago, so this does not stall the launch pipeline) and recycle them."""
        while len(self._ev_pending) > keep:
            kind, arr, nbytes = self._ev_pending.pop(0)
            n = len(arr) // 2
            ms = (ctypes.c_float * n)()
            nat.events_elapsed(arr, n, ms)
            dst = self.attn_times if kind == "attn" else self.linear_times
            dst.extend((float(m), nbytes[i % len(nbytes)]) for i, m in enumerate(ms))
            self._ev_free.append(arr)

    def collect_attn_times(self) -> list:
        """(ms, algorithmic bytes) of every attention launch timed so far (both paths)."""
        self._retire_events(0)
        out = list(self.attn_times)
        if self.attn_events:
            out += [(a.elapsed_time(b), nb) for a, b, nb in self.attn_events]
        return out

    def _k7_ok(self, rows: int) -> bool:
        """K7 takes the step when its stacked GEMM input has <= 128 rows.  (K7 runs up to 256
        stacked rows, NX 256, but measured at the C3 header step -- 72 rows = 144 stacked --
        it is slower than cuBLAS there: every weight tile re-reads a 32 KB activation block
        per k-block and only 64 KB of weights fit in flight per SM.)"""
        return self.k7 and (2 * rows if self.split else rows) <= 128

    def _lin(self, a, w, rows: int):
        """f32 [rows, N] = a @ w^T through K7; a holds the step's GEMM input rows (hi/lo
        stacked when split; the halves are summed in K7's epilogue)."""
        if self._k7_ws is None:
            self._lin_buffers()
        n, k = w.shape
        y = torch.empty(rows, n, dtype=torch.float32, device=self.dev)
        nat.linear_skinny(a.data_ptr(), a.shape[0], int(self.split), w.data_ptr(), n, k,
                          y.data_ptr(), self._k7_ws.data_ptr(), self._k7_cnt.data_ptr(), 0,
                          torch.cuda.current_stream(self.dev).cuda_stream)
        self.launches += 1
        return y

    def _mm(self, a, w, out_f32: bool):
        if out_f32 and a.dtype != torch.float32:
            return torch.mm(a, w.t(), out_dtype=torch.float32)
        # the f32 parity variant needs true-f32 GEMMs (1e-4 contract): TF32 is pinned off
        # for this call whatever the caller set globally
        mm = torch.backends.cuda.matmul
        if not mm.allow_tf32:
            return torch.mm(a, w.t())
        mm.allow_tf32 = False
        try:
            return torch.mm(a, w.t())
        finally:
            mm.allow_tf32 = True

    def _attn_algorithmic_bytes(self, plan: StepPlan, msg_len, R: int, n_parts: int) -> int:
        """unique KV bytes the step's attention must read (each visible
        page once, valid slots only) + q read + partials written, for one layer."""
        cfg, P = self.cfg, self.cache.page_size
        seen: dict = {}
        for c in plan.calls:
            for p in c.parents:
                seen[p] = int(msg_len[p])
            own = c.first_t + len(c.tokens)
            seen[c.msg] = max(seen.get(c.msg, 0), own)
        toks = sum(seen.values())
        elt = self.cache.k_pool.element_size()
        return (2 * toks * cfg.kv_heads * cfg.head_dim * elt + R * cfg.n_heads * cfg.head_dim * 4
                + n_parts * cfg.n_heads * (cfg.head_dim + 1) * 4)

    def _native_layers(self, R, q, part_o, part_lse, attn, h, act, x, pos_d, page_d, slot_d, fat,
                       counts, n_items, row_part_off, row_part, attn_bytes, stream, v2=None):
        """All layers of a decode-sized step through choreo_decode_layers; returns the last
        layer's down_proj output (hi/lo summed)."""
        cfg, cache, dev = self.cfg, self.cache, self.dev
        L, d, hd = len(self.w.layers), self.d, cfg.head_dim
        n_qkv = (cfg.n_heads + 2 * cfg.kv_heads) * hd
        if self._k7_ws is None:
            self._lin_buffers()
        f32 = torch.float32
        qkv = torch.empty(R, n_qkv, dtype=f32, device=dev)
        ao = torch.empty(R, d, dtype=f32, device=dev)
        gu = torch.empty(R, 2 * cfg.ffn_dim, dtype=f32, device=dev)
        delta = torch.empty(R, d, dtype=f32, device=dev)
        wp = self._weight_ptrs()
        def events(n):
            for i, a in enumerate(self._ev_free):
                if len(a) == n:
                    return self._ev_free.pop(i)
            a = (ctypes.c_void_p * n)()
            nat.events_create(a, n)
            return a
        chain = self._chain_ok(R)
        ev = events(2 * L) if self.attn_events is not None else None
        lev = events(2 * (L + 1) if chain else 8 * L) if self.time_linear else None
        st = nat.DecodeStep(
            n_layers=L, d=d, n_heads=cfg.n_heads, n_kv=cfg.kv_heads, head_dim=hd,
            ffn_dim=cfg.ffn_dim, attn_norm=ctypes.cast(wp["attn_norm"], ctypes.c_void_p),
            w_qkv=ctypes.cast(wp["w_qkv"], ctypes.c_void_p), wo=ctypes.cast(wp["wo"], ctypes.c_void_p),
            ffn_norm=ctypes.cast(wp["ffn_norm"], ctypes.c_void_p),
            w_gu=ctypes.cast(wp["w_gu"], ctypes.c_void_p),
            w_down=ctypes.cast(wp["w_down"], ctypes.c_void_p), eps=RMS_EPS,
            k_pool=cache.k_pool.data_ptr(), v_pool=cache.v_pool.data_ptr(), n_pages=cache.n_pages,
            page_size=cache.page_size, cos_t=self.rot.cos.data_ptr(), sin_t=self.rot.sin.data_ptr(),
            max_delta=self.rot.max_delta, n_rows=R, split=int(self.split),
            n_items=n_items, pos=pos_d.data_ptr(),
            page=page_d.data_ptr(), slot=slot_d.data_ptr(), fat=nat.ptr(fat),
            counts=counts.data_ptr(), row_part_off=row_part_off.data_ptr(),
            row_part=row_part.data_ptr(), x=x.data_ptr(), delta_in=None, h=h.data_ptr(),
            qkv=qkv.data_ptr(), q=q.data_ptr(), part_o=part_o.data_ptr(),
            part_lse=part_lse.data_ptr(), attn=attn.data_ptr(), ao=ao.data_ptr(), gu=gu.data_ptr(),
            act=act.data_ptr(), delta=delta.data_ptr(), k7_ws=self._k7_ws.data_ptr(),
            k7_cnt=self._k7_cnt.data_ptr(),
            attn_events=ctypes.cast(ev, ctypes.c_void_p) if ev is not None else None,
            linear_events=ctypes.cast(lev, ctypes.c_void_p) if lev is not None else None)
        if self.q_bulk:  # RoPE writes K5 v2's Q record, K5 v2 bulk-copies it
            q_k5 = torch.empty(R, cfg.n_heads, 2, hd, dtype=torch.bfloat16, device=dev)
            st.q_k5 = q_k5.data_ptr()
        if v2 is not None:
            _, rowt_d, vis, blk_rows, items, order, tag = v2
            st.row_t, st.vis_page, st.vis_len, st.vis_own = (
                rowt_d.data_ptr(), vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr())
            st.blk_rows, st.items = blk_rows.data_ptr(), items.data_ptr()
            st.item_order = nat.ptr(order)
            st.k3_tag = tag
        if chain:
            cb = self._chain_buffers()
            h_b = torch.empty(2 * R if self.split else R, d, dtype=self.dt, device=dev)
            st.h_b, st.ssq_a, st.ssq_b = h_b.data_ptr(), cb["ssq_a"].data_ptr(), cb["ssq_b"].data_ptr()
            st.chain_ws, st.chain_counters = cb["ws"].data_ptr(), cb["counters"].data_ptr()
            st.chain_done = cb["done"].data_ptr()
            st.chain_events = ctypes.cast(lev, ctypes.c_void_p) if lev is not None else None
            nat.decode_layers(ctypes.byref(st), stream)
        elif self.tp is not None and self.tp.size > 1:
            # per layer: attention half, all-reduce o_proj partials, MLP half, all-reduce
            # down_proj partials (the collectives stay with torch.distributed / NCCL)
            for layer in range(L):
                st.layer_begin, st.layer_end, st.part = layer, layer + 1, 1
                st.delta_in = delta.data_ptr() if layer else None
                nat.decode_layers(ctypes.byref(st), stream)
                torch.distributed.all_reduce(ao, group=self.tp_group)
                st.part = 2
                nat.decode_layers(ctypes.byref(st), stream)
                torch.distributed.all_reduce(delta, group=self.tp_group)
        else:
            nat.decode_layers(ctypes.byref(st), stream)
        if ev is not None:
            self._ev_pending.append(("attn", ev, [attn_bytes]))
        if lev is not None:
            x_rows = (2 if self.split else 1) * R
            lb = {n: w.numel() * w.element_size() + x_rows * w.shape[1] * 2 + R * w.shape[0] * 4
                  for n, w in ((n, self.w.layers[0][n]) for n in ("w_qkv", "wo", "w_gu", "w_down"))}
            if chain:  # per chain launch: qkv(0); o, gate|up, down (+ next qkv) per layer
                rest = lb["wo"] + lb["w_gu"] + lb["w_down"]
                self._ev_pending.append(("linear", lev, [lb["w_qkv"]] + [rest + lb["w_qkv"]] * (L - 1)
                                         + [rest]))
            else:
                self._ev_pending.append(("linear", lev, [lb[n] for n in
                                                         ("w_qkv", "wo", "w_gu", "w_down")]))
        if ev is not None or lev is not None:
            self._retire_events(16)
        return None if chain else delta

    def _chain_ok(self, rows: int) -> bool:
        """K8 takes decode-sized steps of <= 128 rows (hi/lo: <= 256 stacked GEMM rows)."""
        cfg = self.cfg
        return (self.chain and self.native_step and rows <= 128 and self.d % 64 == 0
                and cfg.ffn_dim % 64 == 0 and (cfg.n_heads * cfg.head_dim) % 64 == 0)

    def _chain_buffers(self) -> dict:
        if self._chain_bufs is None:
            dev, tiles = self.dev, cdiv(self.d, 128)
            self._chain_bufs = {
                "ws": torch.empty(4 * 148 * 2 * 128 * 128, dtype=torch.float32, device=dev),
                "counters": torch.zeros(4 * 1024, dtype=torch.int32, device=dev),
                "done": torch.zeros(8, dtype=torch.int32, device=dev),
                "ssq_a": torch.empty(tiles * 128, dtype=torch.float32, device=dev),
                "ssq_b": torch.empty(tiles * 128, dtype=torch.float32, device=dev)}
        return self._chain_bufs

    def _lin_buffers(self) -> None:
        self._k7_ws = torch.empty(148 * 2 * 256 * 128, dtype=torch.float32, device=self.dev)
        n_max = max(self.w.out_head.shape[0], self.w.layers[0]["w_gu"].shape[0],
                    self.w.layers[0]["w_qkv"].shape[0], self.d)
        self._k7_cnt = torch.zeros(cdiv(n_max, 128) + 1, dtype=torch.int32, device=self.dev)

    def forward(self, plan: StepPlan) -> torch.Tensor | None:
        """Run one step; returns f32 logits [n_logit_rows, V] or None.

        K3 (assemble.cu) plans a step in one CTA with fixed shared-memory tables: at most
        K3_MAX_CALLS calls and, page-centric, K3_MAX_PAIRS (parent, call) pairs with parent
        ids < 2^21.  A step beyond those limits is cut here, on the host and before any
        launch, into sub-steps that each fit; the calls of one step never see each other
        (batch peers are invisible, reference masking.py:77-79), so running them as
        consecutive sub-steps gives the same K/V and logits.  A single call with more
        than K3_MAX_PAIRS parents runs with per-call page lists (mode 1), which have no
        pair limit."""
        chunks = split_plan(plan)
        if len(chunks) == 1:
            return self._forward_one(plan, force_percall=chunks[0][1])
        out = []
        for sub, percall in chunks:
            lg = self._forward_one(sub, force_percall=percall)
            if lg is not None:
                out.append(lg)
        return torch.cat(out) if out else None

    def _forward_one(self, plan: StepPlan, force_percall: bool = False) -> torch.Tensor | None:
        cfg, cache = self.cfg, self.cache
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        R = plan.n_rows
        H, Hk, hd, d = cfg.n_heads, cfg.kv_heads, cfg.head_dim, self.d
        P = cache.page_size
        cache.sync_tables()

        # ---- host-side packing of the step description (ints only) ----
        ids = np.concatenate([np.asarray(c.tokens, np.int32) for c in plan.calls])
        row_t = np.concatenate([c.first_t + np.arange(len(c.tokens), dtype=np.int32)
                                for c in plan.calls])
        pos = np.concatenate([c.offset + c.first_t + np.arange(len(c.tokens), dtype=np.int32)
                              for c in plan.calls])
        pages = np.concatenate([np.asarray(c.pages, np.int32) for c in plan.calls])
        slots = np.concatenate([np.asarray(c.slots, np.int32) for c in plan.calls])
        call_tab, parents, row_off = [], [], 0
        for c in plan.calls:
            call_tab += [c.msg, len(parents), len(c.parents), row_off, len(c.tokens)]
            parents += list(c.parents)
            row_off += len(c.tokens)
        n_calls = len(plan.calls)
        msg_len = cache.msg_len.host
        # prefill-sized steps run K4 (tcgen05, 128-row M tiles); decode-sized steps K5
        G = H // Hk
        # wide decode-sized steps (>= 64 rows, e.g. the parallel header step of 8 agents)
        # also run K4: its 256-vector items read each shared parent page once per 64 rows,
        # where K5 v2's 32-vector units re-read it once per 8 rows (measured: C3 header step
        # 6.5 -> 5.8 ms, tools/hdr_ab.sh)
        wide = R >= 64 and self.wide_k4
        use_k4 = (self.pool_dtc == nat.BF16 and P == 64 and hd in (64, 128) and G <= 128
                  and (max(len(c.tokens) for c in plan.calls) >= 64 or wide)
                  and os.environ.get("CHOREO_PREFILL_K4", "1") != "0")
        mode0 = max(len(c.tokens) for c in plan.calls) < 64 and not force_percall
        # decode-sized bf16 steps: K5 v2 (TMA page ring, <= 32 query vectors per item)
        v2 = (not use_k4 and mode0 and self.pool_dtc == nat.BF16 and P == 64
              and hd in (64, 128) and G <= 32 and os.environ.get("CHOREO_K5V2", "1") != "0")
        rpb = 256 // G if use_k4 else max(1, 32 // G) if v2 else self.rows_per_block
        # pages per item: about two waves of (2 CTAs/SM x 148 SMs) per layer, and at
        # most 512 partials per row for the combine
        # prefill-sized steps: per-call page lists (a row block already fills an M tile)
        mode = 1 if max(len(c.tokens) for c in plan.calls) >= 64 or force_percall else 0
        work = plan_counts(plan.calls, msg_len, P, rpb, 1, mode)
        ppi = max(1, cdiv(work.item_pages * Hk, (2 if use_k4 else 1 if v2 else 3) * 148))
        if v2:  # persistent CTAs: about one (item, kv head) unit per SM; unit record <= 32 pages
            ppi = min(max(ppi, 4), 32)
        if use_k4 and mode == 0:  # page-centric K4 items: long page runs keep its pipeline full
            ppi = max(ppi, 16)
        plan_ = plan_counts(plan.calls, msg_len, P, rpb, ppi, mode)
        if v2:  # grow items until the units fit one wave of CTAs; steps that still need more
            # waves (many workflows batched) deal them longest-first (K3 item_order; measured:
            # one wave of longer items beats a longest-first deal of shorter ones in situ)
            while plan_.n_items * Hk > 148 and ppi < 32:
                ppi = min(32, ppi + max(1, ppi // 4))
                plan_ = plan_counts(plan.calls, msg_len, P, rpb, ppi, mode)
        while plan_.max_row_parts > 512 and not (v2 and ppi >= 32):
            ppi *= 2
            plan_ = plan_counts(plan.calls, msg_len, P, rpb, ppi, mode)
        n_parts, n_items = plan_.n_parts, plan_.n_items
        # K4 writes final rows directly when no row is split across items
        direct = use_k4 and plan_.max_row_parts == 1 and self.dt == torch.bfloat16
        n_log = len(plan.logit_rows)

        sel = plan.sel if plan.sel is not None and (plan.sel >= 0).any() else None
        ints = np.concatenate([ids, row_t, pos, pages, slots, np.asarray(call_tab, np.int32),
                               np.asarray(parents + [0], np.int32),
                               np.asarray(plan.logit_rows, np.int32)]
                              + ([np.asarray(sel, np.int32)] if sel is not None else []))
        dints = h2d(ints, self.dev)
        self.h2d_bytes += ints.nbytes
        if self.step_events is not None:
            sev0 = torch.cuda.Event(enable_timing=True)
            sev0.record()
        attn_bytes = 0
        if self.attn_events is not None:
            attn_bytes = self._attn_algorithmic_bytes(plan, msg_len, R, n_parts)
        o = 0

        def take(n):
            nonlocal o
            t = dints[o:o + n]
            o += n
            return t

        ids_d, rowt_d, pos_d, page_d, slot_d = (take(R) for _ in range(5))
        calls_d = take(5 * n_calls)
        parents_d = take(len(parents) + 1)
        logit_d = take(n_log)
        sel_d = take(R) if sel is not None else None

        vis = torch.empty(3, max(plan_.n_vis, 1), dtype=torch.int32, device=self.dev)
        blk_rows = torch.empty(max(plan_.n_blk_rows, 1), dtype=torch.int32, device=self.dev)
        items = torch.empty(max(n_items, 1), 6, dtype=torch.int32, device=self.dev)
        row_part_off = torch.empty(R + 1, dtype=torch.int32, device=self.dev)
        row_part = torch.empty(max(n_parts, 1), dtype=torch.int32, device=self.dev)
        counts = torch.empty(6, dtype=torch.int32, device=self.dev)  # [4..5]: K3's step stamp
        # a process-unique tag per step: K3 stamps counts[4] with it once its outputs are
        # complete, and K5 v2 then reads them before its programmatic-dependency wait
        tag = next(_STEP_TAGS) if v2 else 0
        fat = (torch.empty(max(n_items, 1), 64, dtype=torch.int32, device=self.dev)
               if v2 and rpb <= 16 else None)
        order = (torch.empty(max(n_items, 1), dtype=torch.int32, device=self.dev)
                 if v2 and self.v2_lpt else None)
        nat.assemble_ex(cache.msg_len.dev.data_ptr(), cache.msg_pt.dev.data_ptr(),
                        cache.page_table.dev.data_ptr(), calls_d.data_ptr(), parents_d.data_ptr(),
                        n_calls, rowt_d.data_ptr(), R, None, 0, P, rpb, ppi, vis[0].data_ptr(),
                        vis[1].data_ptr(), vis[2].data_ptr(), blk_rows.data_ptr(),
                        items.data_ptr(), row_part_off.data_ptr(), row_part.data_ptr(),
                        counts.data_ptr(), plan_.n_vis, plan_.n_blk_rows, n_items, n_parts, mode,
                        nat.ptr(fat), nat.ptr(order), tag, stream)
        self.launches += 1
        self.last_assembly = (vis, blk_rows, items, row_part_off, row_part, counts, plan_, rowt_d)
        if self.check_assembly:  # debug/test: K3 must never report an overflow
            c = counts.cpu().tolist()
            if c[3] != 0 or c[1] != n_items:
                raise nat.NativeError(f"choreo_assemble overflow: counts {c}, planned items "
                                      f"{n_items}")

        S = 2 if self.split else 1  # stacked hi/lo activation rows
        sp = int(self.split)
        k7 = self._k7_ok(R)
        # GEMM outputs: K7 already summed the hi/lo halves (isp = 0); cuBLAS outputs keep
        # them stacked for the consumer to add (isp = sp)
        isp = 0 if k7 else sp
        mm = (lambda a, w: self._lin(a, w, R)) if k7 else (lambda a, w: self._mm(a, w, True))
        x = torch.empty(R, d, dtype=torch.float32, device=self.dev)
        if sel_d is not None:  # pipelined decode: ids of the previous step's device selection
            nat.embed_select(self.w.embed.data_ptr(), self.dtc, d, ids_d.data_ptr(),
                             sel_d.data_ptr(), plan.sel_src.data_ptr(), R, x.data_ptr(), stream)
        else:
            nat.embed(self.w.embed.data_ptr(), self.dtc, d, ids_d.data_ptr(), R, x.data_ptr(),
                      stream)
        q = torch.empty(R, H, hd, dtype=torch.float32, device=self.dev)
        part_o = torch.empty(max(n_parts, 1), H, hd, dtype=torch.float32, device=self.dev)
        part_lse = torch.empty(max(n_parts, 1), H, dtype=torch.float32, device=self.dev)
        attn = torch.empty(S * R, H * hd, dtype=self.dt, device=self.dev)
        h = torch.empty(S * R, d, dtype=self.dt, device=self.dev)
        act = torch.empty(S * R, cfg.ffn_dim, dtype=self.dt, device=self.dev)
        delta = None
        launches = 2
        native = (v2 and self.native_step and self.dt == torch.bfloat16
                  and (k7 or self._chain_ok(R)))
        if native:
            delta = self._native_layers(R, q, part_o, part_lse, attn, h, act, x, pos_d, page_d,
                                        slot_d, fat, counts, n_items, row_part_off, row_part,
                                        attn_bytes, stream,
                                        (v2, rowt_d, vis, blk_rows, items, order, tag))
            if self._chain_ok(R):  # prologue + qkv(0); per layer: K5, combine, K8 chain
                launches += 2 + 3 * len(self.w.layers)
            else:  # per layer: norm, K7 qkv, rope, K5, combine, K7 o, norm, K7 gate|up, K7 down
                launches += (9 if cfg.ffn_dim % 64 == 0 else 10) * len(self.w.layers)
        for layer, lw in enumerate([] if native else self.w.layers):
            nat.residual_rmsnorm(x.data_ptr(), nat.ptr(delta), nat.F32, isp,
                                 lw["attn_norm"].data_ptr(), self.dtc, R, d, RMS_EPS, h.data_ptr(),
                                 self.dtc, sp, None, 0, stream)
            qkv = mm(h, lw["w_qkv"])
            nat.rope_append(qkv.data_ptr(), nat.F32, qkv.shape[1], R, isp, pos_d.data_ptr(),
                            page_d.data_ptr(), slot_d.data_ptr(), q.data_ptr(),
                            cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), self.pool_dtc, layer,
                            Hk, cache.n_pages, P, H, hd, self.rot.cos.data_ptr(),
                            self.rot.sin.data_ptr(), self.rot.max_delta, stream)
            if self.attn_events is not None:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            if v2:
                nat.decode_attn_v2_ex(q.data_ptr(), cache.k_pool.data_ptr(),
                                      cache.v_pool.data_ptr(), cfg.n_layers, layer, Hk,
                                      cache.n_pages, P, H, hd, rowt_d.data_ptr(),
                                      vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr(),
                                      blk_rows.data_ptr(), items.data_ptr(), counts.data_ptr(),
                                      n_items, part_o.data_ptr(), part_lse.data_ptr(),
                                      nat.ptr(fat), 0, None, nat.ptr(order), tag, stream)
            elif use_k4:
                nat.prefill_attn(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                                 self.pool_dtc, cfg.n_layers, layer, Hk, cache.n_pages, P, H, hd,
                                 rowt_d.data_ptr(), vis[0].data_ptr(), vis[1].data_ptr(),
                                 vis[2].data_ptr(), blk_rows.data_ptr(), items.data_ptr(),
                                 counts.data_ptr(), n_items, part_o.data_ptr(),
                                 part_lse.data_ptr(), 0,
                                 attn.data_ptr() if direct else None, sp, R, stream)
            else:
                nat.attn_split(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                               self.pool_dtc, layer, Hk, cache.n_pages, P, H, hd,
                               rowt_d.data_ptr(), vis[0].data_ptr(), vis[1].data_ptr(),
                               vis[2].data_ptr(), blk_rows.data_ptr(), items.data_ptr(),
                               counts.data_ptr(), n_items, part_o.data_ptr(), part_lse.data_ptr(),
                               0, stream)
            if self.attn_events is not None:
                ev1.record()
                self.attn_events.append((ev0, ev1, attn_bytes))
            if not direct:
                nat.attn_combine(part_o.data_ptr(), part_lse.data_ptr(), row_part_off.data_ptr(),
                                 row_part.data_ptr(), R, H, hd, attn.data_ptr(), self.dtc, sp,
                                 stream)
            ao = mm(attn, lw["wo"])
            if self.tp is not None and self.tp.size > 1:  # row-parallel o_proj: sum partials
                torch.distributed.all_reduce(ao, group=self.tp_group)
            nat.residual_rmsnorm(x.data_ptr(), ao.data_ptr(), nat.F32, isp,
                                 lw["ffn_norm"].data_ptr(), self.dtc, R, d, RMS_EPS, h.data_ptr(),
                                 self.dtc, sp, None, 0, stream)
            if k7 and cfg.ffn_dim % 64 == 0:  # K7 with SiLU(gate)*up in its epilogue
                nat.linear_gate_up_silu(h.data_ptr(), h.shape[0], sp, lw["w_gu"].data_ptr(),
                                        cfg.ffn_dim, d, act.data_ptr(), self._k7_ws.data_ptr(),
                                        self._k7_cnt.data_ptr(), stream)
                self.launches += 1
            else:
                gu = mm(h, lw["w_gu"])  # f32 pre-activations (parity)
                nat.silu_mul(gu.data_ptr(), nat.F32, isp, R, cfg.ffn_dim, act.data_ptr(),
                             self.dtc, sp, stream)
            delta = mm(act, lw["w_down"])
            if self.tp is not None and self.tp.size > 1:  # row-parallel down_proj
                torch.distributed.all_reduce(delta, group=self.tp_group)
            launches += 6
        if delta is not None:  # the K8 chain already added the last down_proj into x
            nat.residual_rmsnorm(x.data_ptr(), delta.data_ptr(), nat.F32, isp, None, 0, R, d,
                                 RMS_EPS, None, 0, 0, None, 0, stream)
            launches += 1
        self.launches += launches
        logits = None
        if n_log:
            xn = torch.empty(S * n_log, d, dtype=self.dt, device=self.dev)
            nat.residual_rmsnorm(x.data_ptr(), None, 0, 0, self.w.out_norm.data_ptr(), self.dtc,
                                 R, d, RMS_EPS, xn.data_ptr(), self.dtc, sp, logit_d.data_ptr(),
                                 n_log, stream)
            self.launches += 1
            if self._k7_ok(n_log):
                logits = self._lin(xn, self.w.out_head, n_log)
            else:
                logits = self._mm(xn, self.w.out_head, out_f32=True)
                if self.split:
                    logits = logits[:n_log] + logits[n_log:]
        if self.step_events is not None:
            sev1 = torch.cuda.Event(enable_timing=True)
            sev1.record()
            self.step_events.append((sev0, sev1))
        return logits
