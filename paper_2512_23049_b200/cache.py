"""Global KV cache rebuilt for HBM: a paged K/V pool plus a message table.

Reference: cache.py:51-204 (GlobalKvCache).  What changes:

* K/V live in two device pools ``[layer][kv_head][page][slot][head_dim]`` (bf16,
  or f32 for the parity variant).  Every page belongs to one message and a
  message's tokens fill its page chain in within-message order, so the visible
  set of any call is an exact page subset (+ a causal cut in its own pages).
* The message table (length, page-chain offset, page table) is mirrored on the
  device for the assembler kernel (K3); the host keeps the authoritative copy
  and uploads dirty ranges before a step.
* Physical (append) order — the reference's ``msg_ids/positions/token_ids``
  arrays and ``keys/values`` — is kept as an append log and materialised on
  demand (compat views), so tests and tools that inspect the reference layout
  keep working, including the step-synchronous interleaving of parallel decode.
* Repositioning is destructive as in the reference (cache.py:139-160): the
  position-update kernel (K2) rotates the message's cached keys in place by
  delta = new offset - current offset, all layers in one launch.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _native as nat
from .config import ModelConfig
from .errors import CapacityError, UnknownMessageError, WindowOverflowError


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def h2d(arr: np.ndarray, device) -> torch.Tensor:
    """Host array -> device tensor without a host sync: staged through pinned memory
    (torch's caching host allocator keeps the buffer alive until the copy ran)."""
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if torch.device(device).type != "cuda":
        return t.clone()
    return t.pin_memory().to(device, non_blocking=True)


@dataclass
class MessageSpan:
    """Where one message lives (reference cache.py:28-39)."""

    message_id: int
    kind: str
    offset: int
    length: int
    physical: np.ndarray
    token_ids: np.ndarray
    text: str
    header: str | None = None


@dataclass
class _Entry:
    kind: str
    offset: int
    text: str
    header: str | None
    pt: int  # offset of this message's page chain in the page table
    pt_cap: int  # page-table entries reserved
    tokens: list = field(default_factory=list)
    pages: list = field(default_factory=list)
    phys: list = field(default_factory=list)  # physical indices (reference append order)

    @property
    def length(self) -> int:
        return len(self.tokens)


class RotationTableDevice:
    """cos/sin over deltas [-W, W], computed in f64 then cast to f32 (tensor.py:103-107)."""

    def __init__(self, config: ModelConfig, device) -> None:
        hd, W = config.head_dim, config.context_window
        inv = config.rope_base ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
        ang = np.arange(-W, W + 1, dtype=np.float64)[:, None] * inv[None, :]
        self.max_delta = W
        self.cos = torch.from_numpy(np.cos(ang).astype(np.float32)).to(device)
        self.sin = torch.from_numpy(np.sin(ang).astype(np.float32)).to(device)


class _Grow:
    """Growable host int32/int64 array with a device mirror and a dirty range."""

    def __init__(self, n: int, device, fill: int = 0) -> None:
        self.host = np.full(max(n, 16), fill, dtype=np.int32)
        self.fill = fill
        self.device = device
        self.dev = torch.from_numpy(self.host.copy()).to(device)
        self.lo, self.hi = len(self.host), 0
        self.generation = 0

    def ensure(self, n: int) -> None:
        if n <= len(self.host):
            return
        new = max(n, 2 * len(self.host))
        h = np.full(new, self.fill, dtype=np.int32)
        h[:len(self.host)] = self.host
        self.host = h
        self.dev = torch.from_numpy(h.copy()).to(self.device)
        self.lo, self.hi = len(h), 0
        self.generation += 1

    def set(self, i: int, v: int) -> None:
        self.host[i] = v
        self.lo, self.hi = min(self.lo, i), max(self.hi, i + 1)

    def set_range(self, i: int, vals) -> None:
        vals = np.asarray(vals, dtype=np.int32)
        self.host[i:i + len(vals)] = vals
        if len(vals):
            self.lo, self.hi = min(self.lo, i), max(self.hi, i + len(vals))

    def sync(self) -> None:
        if self.hi > self.lo:
            self.dev[self.lo:self.hi].copy_(h2d(self.host[self.lo:self.hi], self.device),
                                            non_blocking=True)
            self.lo, self.hi = len(self.host), 0


class DeviceKvCache:
    """Paged, message-addressed K/V store in HBM with reference-compatible views."""

    def __init__(self, config: ModelConfig, capacity: int = 65536, dtype=torch.bfloat16,
                 device=None, page_size: int = 64) -> None:
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.config = config
        self.capacity = int(capacity)
        self.dtype = dtype
        self.device = torch.device(device or "cuda")
        self.page_size = int(page_size)
        self.n_pages = 0
        self.k_pool = self.v_pool = None
        self._free: list[int] = []
        self.generation = 0  # bumps whenever pool storage moves (graphs must be recaptured)
        self._grow_pool(max(4, cdiv(min(self.capacity, 1 << 20), self.page_size) // 2 + 8))
        self._messages: dict[int, _Entry] = {}
        self.msg_len = _Grow(64, self.device)
        self.msg_pt = _Grow(64, self.device)
        self.page_table = _Grow(1024, self.device, fill=-1)
        self._pt_next = 0
        self.token_count = 0
        self._log: list[tuple[int, int, int]] = []  # (msg, first token idx, count)
        self._nphys = 0
        self._views = None

    # -- pool ---------------------------------------------------------------------

    def _grow_pool(self, n_pages: int) -> None:
        cfg = self.config
        shape = (cfg.n_layers, cfg.kv_heads, n_pages, self.page_size, cfg.head_dim)
        k = torch.zeros(shape, dtype=self.dtype, device=self.device)
        v = torch.zeros(shape, dtype=self.dtype, device=self.device)
        if self.k_pool is not None:
            k[:, :, :self.n_pages].copy_(self.k_pool)
            v[:, :, :self.n_pages].copy_(self.v_pool)
        self._free = list(range(n_pages - 1, self.n_pages - 1, -1)) + self._free
        self.k_pool, self.v_pool, self.n_pages = k, v, n_pages
        self.generation += 1

    def alloc_page(self) -> int:
        if not self._free:
            self._grow_pool(self.n_pages + max(16, self.n_pages // 2))
        return self._free.pop()

    @property
    def pool_bytes(self) -> int:
        return 2 * self.k_pool.numel() * self.k_pool.element_size()

    # -- message registry -----------------------------------------------------------

    def register_message(self, message_id: int, kind: str, offset: int, text: str = "",
                         header: str | None = None, max_tokens: int | None = None) -> None:
        if message_id in self._messages:
            raise ValueError(f"message {message_id} already registered")
        cap = cdiv(max(1, max_tokens if max_tokens is not None else self.config.context_window),
                   self.page_size)
        e = _Entry(kind=kind, offset=int(offset), text=text, header=header, pt=self._pt_next,
                   pt_cap=cap)
        self._pt_next += cap
        self.page_table.ensure(self._pt_next)
        self.msg_len.ensure(message_id + 1)
        self.msg_pt.ensure(message_id + 1)
        self.msg_pt.set(message_id, e.pt)
        self.msg_len.set(message_id, 0)
        self._messages[message_id] = e

    def set_text(self, message_id: int, text: str) -> None:
        self._entry(message_id).text = text

    def _entry(self, message_id: int) -> _Entry:
        try:
            return self._messages[message_id]
        except KeyError:
            raise UnknownMessageError(f"unknown message id {message_id}") from None

    def __contains__(self, message_id: int) -> bool:
        return message_id in self._messages

    def message_ids(self) -> list[int]:
        return list(self._messages)

    def message_length(self, message_id: int) -> int:
        return self._entry(message_id).length

    def message_length_or_none(self, message_id: int) -> int | None:
        e = self._messages.get(message_id)
        return None if e is None else e.length

    def message_offset(self, message_id: int) -> int:
        return self._entry(message_id).offset

    # -- slots for new tokens -----------------------------------------------------------

    def reserve_slots(self, message_id: int, tokens) -> tuple[np.ndarray, np.ndarray]:
        """Extend a message by len(tokens) tokens; returns (page, slot) per new token.

        Capacity is the reference's token-count limit (cache.py:114-117).  Physical
        order is recorded separately (log_append / log_interleaved).
        """
        e = self._entry(message_id)
        n = len(tokens)
        if self.token_count + n > self.capacity:
            raise CapacityError(f"append of {n} tokens exceeds capacity {self.capacity} "
                                f"(token_count {self.token_count})")
        if e.offset + e.length + n > self.config.context_window:
            raise WindowOverflowError(f"position outside context window [0, {self.config.context_window})")
        P = self.page_size
        first = e.length
        need = cdiv(first + n, P)
        while len(e.pages) < need:
            if len(e.pages) >= e.pt_cap:
                self._relocate_chain(e, max(2 * e.pt_cap, need))
            pg = self.alloc_page()
            self.page_table.set(e.pt + len(e.pages), pg)
            e.pages.append(pg)
        idx = np.arange(first, first + n)
        pages = np.asarray(e.pages, dtype=np.int32)[idx // P]
        slots = (idx % P).astype(np.int32)
        e.tokens.extend(int(t) for t in tokens)
        self.msg_len.set(message_id, e.length)
        self.token_count += n
        self._views = None
        return pages, slots

    def set_token(self, message_id: int, index: int, token: int) -> None:
        """Record the id of a token reserved before its value was known on the host (a
        pipelined decode step encodes the device-selected token of the previous step)."""
        self._entry(message_id).tokens[index] = int(token)
        self._views = None

    def unreserve_last(self, message_id: int) -> None:
        """Undo the last reserve_slots of one token: a pipelined decode step encoded the
        device-selected token of a message the host then saw stop (EOS, window, limit).
        The slot lies past the message's length again, so nothing can see it; its page
        stays with the message."""
        e = self._entry(message_id)
        e.tokens.pop()
        self.msg_len.set(message_id, e.length)
        self.token_count -= 1
        self._views = None

    def release_prefix_pages(self, message_id: int, n_tokens: int) -> int:
        """Return the pages holding only tokens [0, n_tokens) of a message to the pool (the
        re-encoding comparator's dead prompt copies).  The message must never be read
        below n_tokens again; its page-table entries for them become -1.  Returns the
        number of pages released."""
        e = self._entry(message_id)
        P = self.page_size
        n = len(e.pages) if n_tokens >= e.length else n_tokens // P
        freed = 0
        for i in range(n):
            if e.pages[i] >= 0:
                self._free.append(e.pages[i])
                e.pages[i] = -1
                self.page_table.set(e.pt + i, -1)
                self.token_count -= min(P, e.length - i * P)
                freed += 1
        return freed

    def _relocate_chain(self, e: _Entry, cap: int) -> None:
        e.pt, e.pt_cap = self._pt_next, cap
        self._pt_next += cap
        self.page_table.ensure(self._pt_next)
        self.page_table.set_range(e.pt, e.pages)
        mid = next(m for m, x in self._messages.items() if x is e)
        self.msg_pt.set(mid, e.pt)

    def log_append(self, message_id: int, first: int, count: int) -> None:
        """Record tokens [first, first+count) of a message as physically contiguous."""
        if count <= 0:
            return
        e = self._entry(message_id)
        start = self._nphys
        self._nphys += count
        e.phys.extend(range(start, start + count))
        if self._log and self._log[-1][0] == message_id and \
                self._log[-1][1] + self._log[-1][2] == first:
            m, f, c = self._log[-1]
            self._log[-1] = (m, f, c + count)
        else:
            self._log.append((message_id, first, count))
        self._views = None

    def log_interleaved(self, message_ids: list[int], firsts: list[int], counts: list[int]) -> None:
        """Physical order of a step-synchronous parallel decode (engine.py:437-441).

        Step s appends token s of every message still active, in call order.
        """
        for s in range(max(counts, default=0)):
            for m, f, c in zip(message_ids, firsts, counts):
                if s < c:
                    self.log_append(m, f + s, 1)

    def sync_tables(self) -> None:
        self.msg_len.sync()
        self.msg_pt.sync()
        self.page_table.sync()

    # -- repositioning (K2) ------------------------------------------------------------

    def reposition_many(self, moves: dict, rotation: RotationTableDevice, stream=None) -> int:
        """Move messages to new offsets; rotates their cached keys by the deltas.

        Validation first (window), then one K2 launch for all moved pages.
        Returns the number of moved tokens (engine.py:247-252).
        """
        W = self.config.context_window
        for m, o in moves.items():
            e = self._entry(m)
            if o < 0:
                raise ValueError("offset must be >= 0")
            if o + e.length > W:
                raise WindowOverflowError(f"message {m} (len {e.length}) does not fit at {o}")
        pages, lens, deltas, moved = [], [], [], 0
        P = self.page_size
        for m, o in moves.items():
            e = self._entry(m)
            delta = int(o) - e.offset
            if delta == 0:
                continue
            if abs(delta) > W:
                from .errors import DeltaRangeError
                raise DeltaRangeError(f"delta {delta} outside [-{W}, {W}]")
            for i, pg in enumerate(e.pages):
                pages.append(pg)
                lens.append(min(P, e.length - i * P))
                deltas.append(delta)
            e.offset = int(o)
            moved += e.length
        if pages:
            self._views = None
            arr = h2d(np.asarray([pages, lens, deltas], dtype=np.int32), self.device)
            cfg = self.config
            nat.rerotate(self.k_pool.data_ptr(), nat.dtype_code(self.dtype), cfg.n_layers,
                         cfg.kv_heads, self.n_pages, P, cfg.head_dim, arr[0].data_ptr(),
                         arr[1].data_ptr(), arr[2].data_ptr(), len(pages),
                         rotation.cos.data_ptr(), rotation.sin.data_ptr(), rotation.max_delta,
                         stream or torch.cuda.current_stream(self.device).cuda_stream)
        return moved

    # -- reference-compatible views --------------------------------------------------------

    def _build_views(self) -> dict:
        if self._views is not None:
            return self._views
        n = self._nphys
        mid = np.empty(n, np.int64)
        idx = np.empty(n, np.int64)
        at = 0
        for m, f, c in self._log:
            mid[at:at + c] = m
            idx[at:at + c] = np.arange(f, f + c)
            at += c
        pos = np.empty(n, np.int64)
        tok = np.empty(n, np.int64)
        page = np.empty(n, np.int64)
        P = self.page_size
        for m, e in self._messages.items():
            sel = mid == m
            if not sel.any():
                continue
            ii = idx[sel]
            pos[sel] = e.offset + ii
            tok[sel] = np.asarray(e.tokens, np.int64)[ii]
            page[sel] = np.asarray(e.pages, np.int64)[ii // P]
        self._views = {"msg_ids": mid, "positions": pos, "token_ids": tok, "page": page,
                       "slot": idx % P}
        return self._views

    @property
    def msg_ids(self) -> np.ndarray:
        return self._build_views()["msg_ids"]

    @property
    def positions(self) -> np.ndarray:
        return self._build_views()["positions"]

    @property
    def token_ids(self) -> np.ndarray:
        return self._build_views()["token_ids"]

    def _gather(self, pool) -> np.ndarray:
        v = self._build_views()
        page = torch.from_numpy(v["page"]).to(self.device)
        slot = torch.from_numpy(v["slot"]).to(self.device)
        g = pool[:, :, page, slot]  # (L, Hkv, n, hd)
        return g.permute(0, 2, 1, 3).to(torch.float64).cpu().numpy()

    @property
    def keys(self) -> np.ndarray:
        """(L, token_count, Hkv, hd) in physical order, float64 (reference cache.keys layout)."""
        return self._gather(self.k_pool)

    @property
    def values(self) -> np.ndarray:
        return self._gather(self.v_pool)

    def message_span(self, message_id: int) -> MessageSpan:
        e = self._entry(message_id)
        return MessageSpan(message_id=message_id, kind=e.kind, offset=e.offset, length=e.length,
                           physical=np.asarray(e.phys, np.int64),
                           token_ids=np.asarray(e.tokens, np.int64), text=e.text, header=e.header)

    def dump_jsonl(self, path: str | Path) -> None:
        v = self._build_views()
        with open(path, "w", encoding="utf-8") as fh:
            for i in range(len(v["msg_ids"])):
                fh.write(json.dumps({"physical_index": i, "m": int(v["msg_ids"][i]),
                                     "j": int(v["positions"][i]),
                                     "token_id": int(v["token_ids"][i])}) + "\n")

    def reset(self) -> None:
        """Drop every message and free every page; pool storage is kept (no realloc)."""
        self._free = list(range(self.n_pages - 1, -1, -1))
        self._messages = {}
        self.msg_len = _Grow(64, self.device)
        self.msg_pt = _Grow(64, self.device)
        self.page_table = _Grow(1024, self.device, fill=-1)
        self._pt_next = 0
        self.token_count = 0
        self._log = []
        self._nphys = 0
        self._views = None

    def clone(self) -> "DeviceKvCache":
        """Deep copy: pools (device copy), page tables and host metadata."""
        other = DeviceKvCache.__new__(DeviceKvCache)
        other.config, other.capacity, other.dtype = self.config, self.capacity, self.dtype
        other.device, other.page_size, other.n_pages = self.device, self.page_size, self.n_pages
        other.k_pool, other.v_pool = self.k_pool.clone(), self.v_pool.clone()
        other._free = list(self._free)
        other.generation = 0
        other._messages = {m: _Entry(e.kind, e.offset, e.text, e.header, e.pt, e.pt_cap,
                                     list(e.tokens), list(e.pages), list(e.phys))
                           for m, e in self._messages.items()}
        for name in ("msg_len", "msg_pt", "page_table"):
            src = getattr(self, name)
            g = _Grow.__new__(_Grow)
            g.host, g.fill, g.device = src.host.copy(), src.fill, src.device
            g.dev = torch.from_numpy(g.host.copy()).to(src.device)
            g.lo, g.hi, g.generation = len(g.host), 0, 0
            setattr(other, name, g)
        other._pt_next = self._pt_next
        other.token_count = self.token_count
        other._log = list(self._log)
        other._nphys = self._nphys
        other._views = None
        return other
