"""Drop-in choreography Engine over the device cache (reference engine.py:133-468).

Same public surface and semantics as the reference ``Engine``: ``prefill``,
``prefill_parallel``, ``decode``, ``decode_parallel``, ``message_text``,
``message_token_count``, ``generated_token_ids``, ``clone``, ``stats`` /
``last_stats``, ``kind``, ``seed``, ``config``, ``record_logits`` and a ``cache``
with the reference's inspection surface.  All validation runs on the host mirror
before any device work (ids are never burned by a failed call).

What differs is the schedule, never the result:
* every step is ONE batched forward over all rows of all messages in it
  (the reference loops over groups, model.py:138-142);
* a parallel decode encodes all headers in the first step (the reference feeds
  one header token per step, engine.py:452-455).  Each message's tokens only
  depend on its own tokens and its parents, so outputs are identical; the
  reference's physical interleaving is reproduced in the cache's views;
* greedy selection runs on the device (K6) over the generatable ids.
CallStats FLOPs follow the reference's analytic accounting per op exactly.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native as nat
from .cache import DeviceKvCache, RotationTableDevice, h2d
from .config import EOS_MSG, ModelConfig
from .errors import (CapacityError, EmptyHeaderError, InvalidCallError, OffsetConflictError,
                     UnknownMessageError, WindowOverflowError)
from .model import CallRows, Runner, StepPlan
from .tokenizer import decode_tokens, encode_text, frame_header, frame_message, generatable_mask
from .weights import DeviceWeights, WeightSet


@dataclass(frozen=True)
class SamplingParams:
    """engine.py:45-69."""

    mode: str = "greedy"
    temperature: float = 0.7
    top_p: float = 0.95
    seed: int = 0
    max_tokens: int = 64

    def __post_init__(self) -> None:
        if self.mode not in ("greedy", "temperature"):
            raise InvalidCallError(f"unknown sampling mode {self.mode!r}")
        if self.mode == "temperature" and self.temperature <= 0:
            raise InvalidCallError("temperature must be > 0")
        if not 0 < self.top_p <= 1:
            raise InvalidCallError("top_p must be in (0, 1]")
        if self.max_tokens < 0:
            raise InvalidCallError("max_tokens must be >= 0")


@dataclass(frozen=True)
class PrefillCall:
    message: str
    parents: Sequence[int] = ()
    offsets: Sequence[int | None] | None = None
    new_offset: int | None = None


@dataclass(frozen=True)
class DecodeCall:
    header: str
    parents: Sequence[int] = ()
    offsets: Sequence[int | None] | None = None
    new_offset: int | None = None
    sampling: SamplingParams = field(default_factory=SamplingParams)


@dataclass
class CallStats:
    """engine.py:93-106."""

    op: str
    ids: list
    prefill_flops: int = 0
    decode_flops: int = 0
    tokens_encoded: int = 0
    cache_hit_tokens: int = 0
    repositioned_tokens: int = 0
    ttft: dict = field(default_factory=dict)
    wall: float = 0.0
    logits: dict | None = None


def encode_flops(config: ModelConfig, t_new: int, ctx: int, rows: str) -> int:
    """Analytic FLOPs of one group (model.py:218-235), GQA-aware projections."""
    if t_new == 0:
        return 0
    d, L = config.model_dim, config.n_layers
    nrow = {"all": t_new, "last": 1, "none": 0}[rows]
    return (L * 2 * t_new * (2 * d * d + 2 * d * config.kv_dim) + L * 4 * t_new * d * (ctx + t_new)
            + L * 6 * t_new * d * config.ffn_dim + 2 * nrow * d * config.vocab_size)


def resolve_calls(calls, new_lens, length_of, window: int):
    """Validate a batch's parents/offsets and lay it out (engine.py:203-245).

    ``length_of(msg)`` returns a message's token count, or None if unknown.
    Omitted offsets default to right after the preceding parent (first to 0),
    new_offset to right after the last parent; a parent shared within the batch
    must get one offset.  Returns (agreed {parent: offset}, [(parents, new_offset)]).
    Raises before any mutation.
    """
    agreed: dict[int, int] = {}
    layouts = []
    for call, new_len in zip(calls, new_lens):
        parents = [int(p) for p in call.parents]
        if len(set(parents)) != len(parents):
            raise InvalidCallError(f"duplicate parents {parents}")
        lens = [length_of(p) for p in parents]
        for p, n in zip(parents, lens):
            if n is None:
                raise UnknownMessageError(f"unknown parent id {p}")
        offsets = list(call.offsets) if call.offsets is not None else [None] * len(parents)
        if len(offsets) != len(parents):
            raise InvalidCallError(
                f"offsets length {len(offsets)} != parents length {len(parents)}")
        prev_end = 0
        for p, plen, off in zip(parents, lens, offsets):
            o = prev_end if off is None else int(off)
            if o < 0:
                raise InvalidCallError(f"negative offset {o} for parent {p}")
            if o + plen > window:
                raise WindowOverflowError(f"parent {p} (len {plen}) does not fit at offset {o}")
            if p in agreed and agreed[p] != o:
                raise OffsetConflictError(
                    f"parent {p} placed at both {agreed[p]} and {o} in one batch")
            agreed[p] = o
            prev_end = o + plen
        new_off = int(call.new_offset) if call.new_offset is not None else prev_end
        if new_off < 0:
            raise InvalidCallError(f"negative new_offset {new_off}")
        if new_off + new_len > window:
            raise WindowOverflowError(f"new message (len {new_len}) does not fit at offset {new_off}")
        layouts.append((parents, new_off))
    return agreed, layouts


class _Dec:
    """Per-message decode progress (engine.py:109-130)."""

    __slots__ = ("mid", "call", "hdr", "new_off", "parents", "n_par", "forced", "generated",
                 "appended", "sel", "done", "finishing", "last_row")

    def __init__(self, mid, call, hdr, new_off, parents, n_par, forced):
        self.mid, self.call, self.hdr, self.new_off = mid, call, hdr, new_off
        self.parents, self.n_par, self.forced = parents, n_par, forced
        self.generated: list[int] = []
        self.appended = 0
        self.sel = 0
        self.done = False
        self.finishing = False
        self.last_row = None


class Engine:
    """Cache-choreography engine on one B200: paged global KV cache + sm_100a kernels."""

    kind = "choreo"

    def __init__(self, weights, *, capacity: int = 65536, seed: int = 0,
                 record_logits: bool = False, dtype=None, device=None, page_size: int = 64,
                 split_activations: bool = True, tp=None, tp_group=None) -> None:
        """tp / tp_group: KV-head tensor parallelism (parallel.TPLayout); weights must then
        be this rank's shard (parallel.shard_weights or DeviceWeights.random(tp=...))."""
        nat.load()  # fail loudly without the CUDA extension
        device = torch.device(device or "cuda")
        if isinstance(weights, WeightSet):
            dtype = dtype or torch.bfloat16
            weights = DeviceWeights.from_host(weights, dtype=dtype, device=device)
        self.weights: DeviceWeights = weights
        self.config: ModelConfig = tp.config if tp is not None else weights.config
        self.tp, self.tp_group = tp, tp_group
        self.seed = int(seed)
        self.record_logits = record_logits
        # free-running decode steps are enqueued before the previous step's tokens are read
        # back (the selected ids flow to the next step on the device; _decode_loop)
        self.pipeline = True
        self.device = device
        cache_cfg = tp.local_config() if tp is not None else self.config
        self.cache = DeviceKvCache(cache_cfg, capacity=capacity, dtype=weights.torch_dtype,
                                   device=device, page_size=page_size)
        self.rotation = RotationTableDevice(self.config, device)
        self._runner = Runner(self.weights, self.cache, self.rotation, split_activations, tp,
                              tp_group)
        self._generatable = generatable_mask(self.config.vocab_size)
        # temperature sampling on the device (K6b); False: the host NumPy sampler
        self.device_sampling = self.config.vocab_size >= 258
        self._next_id = 0
        self.stats: list[CallStats] = []
        self.d2h_bytes = 0

    # -- public API (engine.py:153-199) ------------------------------------------------

    def prefill(self, call: PrefillCall) -> int:
        return self._prefill_batch([call], op="prefill")[0]

    def prefill_parallel(self, calls: Sequence[PrefillCall]) -> list[int]:
        return self._prefill_batch(list(calls), op="prefill_parallel")

    def decode(self, call: DecodeCall, force_tokens=None) -> int:
        return self._decode_batch([call], [force_tokens], op="decode")[0]

    def decode_parallel(self, calls: Sequence[DecodeCall], force_tokens=None) -> list[int]:
        forces = list(force_tokens) if force_tokens is not None else [None] * len(calls)
        if len(forces) != len(calls):
            raise InvalidCallError("force_tokens length must match calls")
        return self._decode_batch(list(calls), forces, op="decode_parallel")

    def message_text(self, message_id: int) -> str:
        return self.cache.message_span(message_id).text

    def message_token_count(self, message_id: int) -> int:
        return self.cache.message_length(message_id)

    def generated_token_ids(self, message_id: int) -> list[int]:
        span = self.cache.message_span(message_id)
        if span.kind != "decoded":
            raise InvalidCallError(f"message {message_id} was not decoded")
        return [int(t) for t in span.token_ids[len(frame_header(span.header)):]]

    def clone(self) -> "Engine":
        other = Engine.__new__(Engine)
        other.weights, other.config, other.seed = self.weights, self.config, self.seed
        other.record_logits, other.device = self.record_logits, self.device
        other.cache = self.cache.clone()
        other.rotation = self.rotation
        other.tp, other.tp_group = self.tp, self.tp_group
        other._runner = Runner(self.weights, other.cache, self.rotation, self._runner.split,
                               self.tp, self.tp_group)
        other._generatable = self._generatable
        other.device_sampling = self.device_sampling
        other.pipeline = self.pipeline
        other._next_id = self._next_id
        other.stats = []
        other.d2h_bytes = 0
        return other

    def reset(self) -> None:
        """Empty the cache and restart message ids (pool storage is reused).

        Not in the reference API: lets benchmarks run many workflow instances on
        one resident engine without reallocating the HBM pool."""
        self.cache.reset()
        self._next_id = 0
        self.stats = []

    @property
    def last_stats(self) -> CallStats:
        return self.stats[-1]

    @property
    def kernel_launches(self) -> int:
        return self._runner.launches

    # -- validation and layout (engine.py:203-258) ---------------------------------------

    def _resolve_calls(self, calls, new_lens):
        return resolve_calls(calls, new_lens, self.cache.message_length_or_none,
                             self.config.context_window)

    def _check_capacity(self, n_tokens: int) -> None:
        if self.cache.token_count + n_tokens > self.cache.capacity:
            raise CapacityError(f"{n_tokens} new tokens exceed capacity {self.cache.capacity} "
                                f"(token_count {self.cache.token_count})")

    def _alloc_id(self) -> int:
        self._next_id += 1
        return self._next_id - 1

    def _parent_tokens(self, parents) -> int:
        return sum(self.cache.message_length(p) for p in parents)

    # -- prefill (engine.py:262-294) --------------------------------------------------------

    def _prefill_batch(self, calls: list, op: str) -> list[int]:
        t0 = time.perf_counter()
        if not calls:
            return []
        framed = [frame_message(c.message) for c in calls]
        agreed, layouts = self._resolve_calls(calls, [len(f) for f in framed])
        self._check_capacity(sum(len(f) for f in framed))
        stats = CallStats(op=op, ids=[])
        stats.repositioned_tokens = self.cache.reposition_many(agreed, self.rotation)
        ids = [self._alloc_id() for _ in calls]
        stats.ids = ids
        rows = []
        for mid, call, toks, (parents, new_off) in zip(ids, calls, framed, layouts):
            self.cache.register_message(mid, "prefilled", new_off, text=call.message,
                                        max_tokens=len(toks))
            n_vis = self._parent_tokens(parents)
            pages, slots = self.cache.reserve_slots(mid, toks)
            rows.append(CallRows(mid, parents, 0, toks, pages, slots, new_off))
            stats.prefill_flops += encode_flops(self.config, len(toks), n_vis, "none")
            stats.cache_hit_tokens += n_vis
            stats.tokens_encoded += len(toks)
        self._runner.forward(StepPlan(rows, np.zeros(0, np.int32)))
        for mid, toks in zip(ids, framed):
            self.cache.log_append(mid, 0, len(toks))
        torch.cuda.current_stream(self.device).synchronize()
        stats.wall = time.perf_counter() - t0
        self.stats.append(stats)
        return ids

    # -- decode (engine.py:298-463) ---------------------------------------------------------

    def _decode_batch(self, calls: list, forces: list, op: str) -> list[int]:
        t0 = time.perf_counter()
        if not calls:
            return []
        for call in calls:
            if not call.header:
                raise EmptyHeaderError("decode header must be non-empty")
        headers = [frame_header(c.header) for c in calls]
        agreed, layouts = self._resolve_calls(calls, [len(h) for h in headers])
        self._check_capacity(sum(len(h) for h in headers))
        stats = CallStats(op=op, ids=[], logits={} if self.record_logits else None)
        stats.repositioned_tokens = self.cache.reposition_many(agreed, self.rotation)
        ids = [self._alloc_id() for _ in calls]
        stats.ids = ids
        states = []
        W = self.config.context_window
        for mid, call, hdr, force, (parents, new_off) in zip(ids, calls, headers, forces, layouts):
            cap = min(W - new_off, len(hdr) + call.sampling.max_tokens)
            self.cache.register_message(mid, "decoded", new_off, header=call.header,
                                        max_tokens=max(cap, len(hdr)))
            n_par = self._parent_tokens(parents)
            forced = list(encode_text(force)) if isinstance(force, str) else (
                None if force is None else [int(t) for t in force])
            states.append(_Dec(mid, call, hdr, new_off, parents, n_par, forced))
            stats.cache_hit_tokens += n_par
            if self.record_logits:
                stats.logits[mid] = []
        lone = len(states) == 1
        firsts = [self.cache.message_length(s.mid) for s in states]
        try:
            self._decode_loop(states, stats, t0, lone)
        finally:
            counts = [self.cache.message_length(s.mid) - f for s, f in zip(states, firsts)]
            if lone:
                self.cache.log_append(states[0].mid, firsts[0], counts[0])
            else:
                self.cache.log_interleaved([s.mid for s in states], firsts, counts)
            for s in states:
                self.cache.set_text(s.mid, s.call.header + decode_tokens(s.generated))
        # like the reference, a decode call returns with its messages fully encoded in the
        # cache (teacher-forced steps never synchronise mid-call, so without this the next
        # call's TTFT would absorb this call's queued steps)
        torch.cuda.current_stream(self.device).synchronize()
        stats.wall = time.perf_counter() - t0
        self.stats.append(stats)
        return ids

    def _decode_loop(self, states: list, stats: CallStats, t0: float, lone: bool) -> None:
        """Encode pending tokens for all active messages per step, then select.

        Event order per message is the reference's: encode header, select,
        [encode token, select]*, with the stop rules of engine.py:394-413/448-463.

        Pipelined (``self.pipeline``; free-running messages selected on the device, no host
        logits): the step that encodes a message's selected token is enqueued BEFORE the
        host reads that token back -- its embedding row takes the id straight from the
        selection kernel's output (choreo_embed_select) -- and the host resolves the
        previous step's tokens while the GPU runs the next one, so the per-step token
        read-back no longer leaves the GPU idle.  A message the host then sees stop (EOS)
        had one token encoded speculatively: its slot is unreserved (past the message's
        length, so no later step can see it), and that row's accounting and selection are
        dropped: tokens, cache layout and statistics equal the synchronous run's, values up
        to summation order (the undone row was part of that step's batch).
        """
        pending = {s.mid: list(s.hdr) for s in states}
        pipeline = self.pipeline and not self.record_logits and self.device_sampling
        prev = None  # unresolved device selection of the previous step
        while True:
            # ---- rows of this step: known tokens, and (pipelined) one device-selected token
            # for each message of the unresolved selection that may still accept it
            spec = {}
            if prev is not None:
                for s, k, i in prev["free"]:
                    if not s.done and self._may_accept(s):
                        spec[s.mid] = i
            active = [s for s in states if not s.done and (pending[s.mid] or s.mid in spec)]
            room = self.cache.capacity - self.cache.token_count
            if prev is not None and sum(len(pending[s.mid]) or 1 for s in active) > room:
                # not every row fits: settle the previous selection first, then run the
                # reference's capacity order on known tokens
                self._resolve(prev, stats, t0, pending, None)
                prev, spec = None, {}
                active = [s for s in states if not s.done and pending[s.mid]]
            if not active:
                if prev is None:
                    return
                self._resolve(prev, stats, t0, pending, None)
                prev = None
                continue
            # capacity for the whole step first: the reference runs the step's forward and
            # then appends message by message, so the messages before the first one that
            # does not fit get their K/V and the append of that one raises (cache.py:114-117,
            # engine.py:430-433).  Same here: encode the prefix that fits, then raise.
            n_fit = 0
            for s in active:
                if len(pending[s.mid]) > room:
                    break
                room -= len(pending[s.mid])
                n_fit += 1
            if n_fit < len(active):
                self._encode_only(active[:n_fit], pending)
                self._check_capacity(len(pending[active[n_fit].mid]))
            calls, logit_rows, owners, r = [], [], [], 0
            sel = np.full(0, -1, np.int32)
            sel_rows = []
            spec_rows = {}  # mid -> (token index in the message, flops added)
            for s in active:
                is_spec = s.mid in spec
                toks = [0] if is_spec else pending[s.mid]
                first = s.appended
                pages, slots = self.cache.reserve_slots(s.mid, toks)
                calls.append(CallRows(s.mid, s.parents, first, toks, pages, slots, s.new_off))
                if is_spec:
                    sel_rows.append((r, spec[s.mid]))
                r += len(toks)
                # FLOP accounting as the reference would have executed it
                fl = 0
                if lone or len(states) == 1:
                    if first == 0:
                        fl = encode_flops(self.config, len(toks), s.n_par, "last")
                    else:
                        fl = encode_flops(self.config, 1, s.n_par + first, "all")
                else:
                    for j in range(len(toks)):
                        fl += encode_flops(self.config, 1, s.n_par + first + j, "all")
                stats.decode_flops += fl
                stats.tokens_encoded += len(toks)
                s.appended += len(toks)
                if is_spec:
                    spec_rows[s.mid] = (first, fl)
                    # the token, if accepted, may be the message's last (max_tokens)
                    if len(s.generated) + 1 >= s.call.sampling.max_tokens:
                        s.finishing = True
                if not s.finishing:
                    logit_rows.append(r - 1)
                    owners.append(s)
            plan = StepPlan(calls, np.asarray(logit_rows, np.int32))
            if sel_rows:
                plan.sel = np.full(r, -1, np.int32)
                for row, i in sel_rows:
                    plan.sel[row] = i
                plan.sel_src = prev["out"]
            logits = self._runner.forward(plan)
            for s in active:
                pending[s.mid] = []
                if s.finishing:
                    s.done = True
            cur = None
            if owners:
                cur = self._select(owners, logits, stats, t0, pending, pipeline)
            if prev is not None:
                # the GPU runs this step while the host settles the previous one
                void = self._resolve(prev, stats, t0, pending, spec_rows)
                if void and cur is not None:  # their selections in this step are moot
                    cur["free"] = [e for e in cur["free"] if e[0].mid not in void]
            prev = cur if cur is not None and cur["free"] else None

    def _select(self, owners: list, logits, stats: CallStats, t0: float, pending: dict,
                pipeline: bool):
        """Select one token per owner row: forced tokens directly, free ones on the device
        (K6 greedy / K6b nucleus).  Pipelined, the free tokens stay on the device and are
        returned unresolved (copied to pinned host memory behind an event); otherwise they
        are read back and applied now.  Selection indices are assigned at launch."""
        stream = torch.cuda.current_stream(self.device).cuda_stream
        n_own = len(owners)
        ks = []
        for s in owners:
            ks.append(s.sel)
            s.sel += 1
        free = [s for s in owners if s.forced is None]
        want_g = any(s.call.sampling.mode == "greedy" for s in free)
        want_n = any(s.call.sampling.mode != "greedy" for s in free) and self.device_sampling
        out = None
        if want_g or want_n:
            out = torch.empty(2, n_own, dtype=torch.int32, device=self.device)
            if want_g:  # K6 greedy over every owner row (non-greedy rows ignored)
                nat.select_greedy(logits.data_ptr(), n_own, logits.shape[1], logits.shape[1],
                                  0, out[0].data_ptr(), stream)
                self._runner.launches += 1
            if want_n:  # K6b nucleus: the reference's f64 algorithm + Philox stream
                params = np.array([[s.call.sampling.temperature, s.call.sampling.top_p]
                                   for s in owners], np.float64)
                m64 = 0xFFFFFFFFFFFFFFFF
                keys = np.array([[self.seed & m64, s.call.sampling.seed & m64, s.mid, k]
                                 for s, k in zip(owners, ks)], np.uint64).view(np.int64)
                pd, kd = h2d(params, self.device), h2d(keys, self.device)
                nat.select_nucleus(logits.data_ptr(), n_own, logits.shape[1],
                                   logits.shape[1], pd.data_ptr(), kd.data_ptr(),
                                   out[1].data_ptr(), stream)
                self._runner.launches += 1
        # flat index of each free owner's token in `out` (greedy row 0, nucleus row 1)
        free_idx = [(s, k, (0 if s.call.sampling.mode == "greedy" else 1) * n_own + i)
                    for i, (s, k) in enumerate(zip(owners, ks)) if s.forced is None]
        if pipeline and out is not None and len(free_idx) == len([s for s in free]):
            # a ring of pinned read-back buffers (a buffer is reused two steps later, after
            # its tokens were read)
            self._pin_i = (getattr(self, "_pin_i", 0) + 1) % 3
            ring = getattr(self, "_pin", None)
            if ring is None or ring[0].numel() < 2 * n_own:
                ring = self._pin = [torch.empty(max(64, 2 * n_own), dtype=torch.int32,
                                                pin_memory=True) for _ in range(3)]
            host = ring[self._pin_i][:2 * n_own]
            flat = out.view(-1)
            host.copy_(flat, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self.d2h_bytes += out.nbytes
            cur = {"free": free_idx, "out": flat, "host": host, "event": ev}
        else:
            cur = None
        host_logits = None
        toks = None
        if out is not None and cur is None:
            toks = out.view(-1).cpu().numpy()
            self.d2h_bytes += out.nbytes
        if self.record_logits or (not self.device_sampling and any(
                s.forced is None and s.call.sampling.mode != "greedy" for s in owners)):
            hl = logits.double().cpu().numpy()
            self.d2h_bytes += logits.nbytes
            host_logits = hl
        elif out is None and any(k == 0 for k in ks):
            # all forced: the host already knows the tokens; synchronise only at a
            # message's first selection so its TTFT is the time its logits exist
            torch.cuda.current_stream(self.device).synchronize()
        for i, (s, k) in enumerate(zip(owners, ks)):
            if stats.logits is not None:
                stats.logits[s.mid].append(host_logits[i].copy())
            if s.forced is not None:
                tok = s.forced[k] if k < len(s.forced) else None
            elif cur is not None:
                continue  # resolved with the next step in flight (_resolve)
            elif s.call.sampling.mode == "greedy":
                tok = int(toks[i])
            elif self.device_sampling:
                tok = int(toks[n_own + i])
            else:
                tok = _sample_nucleus(host_logits[i], self._generatable, s.call.sampling,
                                      self.seed, s.mid, k)
            self._accept(s, k, tok, stats, t0, pending)
        return cur

    def _accept(self, s: _Dec, k: int, tok, stats: CallStats, t0: float, pending: dict,
                spec_index=None) -> bool:
        """Apply selection k of message s (engine.py:394-413).  spec_index: the message's
        token index already encoded with this token (pipelined step), patched or undone."""
        if k == 0:
            stats.ttft[s.mid] = time.perf_counter() - t0
        if tok is None or tok == EOS_MSG or not self._may_accept(s):
            s.done = True
            return False
        s.generated.append(tok)
        if spec_index is not None:
            self.cache.set_token(s.mid, spec_index, tok)
        else:
            pending[s.mid] = [tok]
        if len(s.generated) >= s.call.sampling.max_tokens:
            s.finishing = True
        return True

    def _resolve(self, prev: dict, stats: CallStats, t0: float, pending: dict,
                 spec_rows) -> set:
        """Read back a pipelined selection and apply it.  Messages whose token the current
        step already encoded (spec_rows: mid -> (token index, flops)) keep it if accepted;
        if the token stops the message, the encoding is undone (slot unreserved, accounting
        subtracted).  Returns the mids whose current-step rows were undone."""
        prev["event"].synchronize()
        toks = prev["host"].numpy()
        void = set()
        for s, k, i in prev["free"]:
            sp = spec_rows.get(s.mid) if spec_rows else None
            if sp is not None:
                s.appended -= 1  # _may_accept sees the count at selection time
            ok = self._accept(s, k, int(toks[i]), stats, t0, pending,
                              spec_index=None if sp is None else sp[0])
            if sp is None:
                continue
            if ok:
                s.appended += 1
            else:
                self.cache.unreserve_last(s.mid)
                stats.decode_flops -= sp[1]
                stats.tokens_encoded -= 1
                s.finishing = False
                s.done = True
                void.add(s.mid)
        return void

    def _encode_only(self, states: list, pending: dict) -> None:
        """Encode (append) the pending tokens of `states` without selecting: the part of a
        step that precedes a capacity failure."""
        calls = []
        for s in states:
            toks = pending[s.mid]
            pages, slots = self.cache.reserve_slots(s.mid, toks)
            calls.append(CallRows(s.mid, s.parents, s.appended, toks, pages, slots, s.new_off))
            s.appended += len(toks)
            pending[s.mid] = []
        if calls:
            self._runner.forward(StepPlan(calls, np.zeros(0, np.int32)))

    def _may_accept(self, s: _Dec) -> bool:
        """engine.py:394-399."""
        if len(s.generated) >= s.call.sampling.max_tokens:
            return False
        return s.new_off + s.appended < self.config.context_window


def _stream_uniform(engine_seed: int, sampling_seed: int, msg_id: int, sel_index: int) -> float:
    """Counter-based Philox draw keyed (engine seed, sampling seed) (engine.py:388-392)."""
    key = np.array([engine_seed & 0xFFFFFFFFFFFFFFFF, sampling_seed & 0xFFFFFFFFFFFFFFFF],
                   dtype=np.uint64)
    counter = np.array([sel_index, msg_id, 0, 0], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(counter=counter, key=key)).random()


def _sample_nucleus(logits: np.ndarray, generatable: np.ndarray, params: SamplingParams,
                    engine_seed: int, msg_id: int, sel_index: int) -> int:
    """Temperature + top-p over generatable ids, prob-desc / id-asc (engine.py:374-386)."""
    z = np.where(generatable, logits / params.temperature, -np.inf)
    z = z - z.max()
    probs = np.exp(z)
    probs /= probs.sum()
    order = np.lexsort((np.arange(len(probs)), -probs))
    csum = np.cumsum(probs[order])
    cut = min(int(np.searchsorted(csum, params.top_p, side="left")), len(order) - 1)
    kept = order[:cut + 1]
    kcs = np.cumsum(probs[kept] / probs[kept].sum())
    u = _stream_uniform(engine_seed, params.seed, msg_id, sel_index)
    return int(kept[min(int(np.searchsorted(kcs, u, side="right")), len(kept) - 1)])
