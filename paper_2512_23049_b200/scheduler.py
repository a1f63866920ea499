"""Cross-workflow batching scheduler (no reference counterpart,
SPEC.md:404 leaves scheduling to the caller).

Many independent choreographed workflows share one ``Engine`` (one global cache, one set
of weights on one GPU).  Each workflow is a generator that yields its next engine request
and receives the message ids back::

    def workflow(rng):
        a, b = yield Prefill([PrefillCall("..."), PrefillCall("...")])
        (c,) = yield Decode([DecodeCall("Agent:", parents=[b, a])], force_tokens=None)
        return c

``BatchScheduler.run`` advances all workflows in lock step: every tick it merges the
pending prefill requests of all workflows into ONE ``prefill_parallel`` and the pending
decode requests into ONE ``decode_parallel``, so the device runs a single forward per step
for all workflows — one K7 weight stream and one K5 launch serve every agent of every
workflow (weights are read once per step instead of once per workflow).

Semantics are unchanged: a message's tokens depend only on its own tokens and its
parents (reference masking.py:36-40), and workflows never share messages unless the
caller makes them, so each workflow's greedy and teacher-forced tokens and logits are
exactly what it would get alone.  Message ids (and so the physical cache layout) are
allocated across the merged calls, and temperature sampling draws its Philox counter from
the message id (reference engine.py:388-392), so sampled tokens are a valid draw but not
the solo run's draw.  Calls are
validated by the engine before any mutation; if merging makes two workflows place a
shared parent at different offsets (``OffsetConflictError``) the tick falls back to one
engine call per workflow.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Generator, Sequence

from .errors import OffsetConflictError


@dataclass
class Prefill:
    calls: Sequence[Any]


@dataclass
class Decode:
    calls: Sequence[Any]
    force_tokens: Sequence[Any] | None = None


@dataclass
class TickStats:
    kind: str
    workflows: int
    calls: int
    merged: bool
    ttft: dict = field(default_factory=dict)


class BatchScheduler:
    """Lock-step batching of workflow generators over one engine."""

    def __init__(self, engine) -> None:
        self.engine = engine
        self.ticks: list[TickStats] = []

    def run(self, workflows: Sequence[Generator]) -> list:
        results: list = [None] * len(workflows)
        pending: dict[int, Any] = {}
        for i, wf in enumerate(workflows):
            self._advance(i, wf, None, pending, results, first=True)
        while pending:
            for kind in (Prefill, Decode):
                batch = {i: r for i, r in pending.items() if isinstance(r, kind)}
                if not batch:
                    continue
                for i, ids in self._issue(kind, batch).items():
                    del pending[i]
                    self._advance(i, workflows[i], ids, pending, results)
        return results

    # -- internals ---------------------------------------------------------------------

    @staticmethod
    def _advance(i, wf, value, pending, results, first=False) -> None:
        try:
            req = next(wf) if first else wf.send(value)
        except StopIteration as stop:
            results[i] = stop.value
            return
        if not isinstance(req, (Prefill, Decode)):
            raise TypeError(f"workflow {i} yielded {type(req).__name__}, not Prefill/Decode")
        pending[i] = req

    def _call(self, kind, calls, forces):
        if kind is Prefill:
            return self.engine.prefill_parallel(calls)
        return self.engine.decode_parallel(calls, force_tokens=forces)

    def _issue(self, kind, batch: dict) -> dict:
        order = sorted(batch)
        calls, forces, spans = [], [], []
        for i in order:
            req = batch[i]
            spans.append((i, len(calls), len(req.calls)))
            calls += list(req.calls)
            if kind is Decode:
                f = req.force_tokens
                forces += list(f) if f is not None else [None] * len(req.calls)
        try:
            ids = self._call(kind, calls, forces if kind is Decode else None)
            self._record(kind, len(order), len(calls), True)
            return {i: ids[a:a + n] for i, a, n in spans}
        except OffsetConflictError:
            # a parent shared across workflows at different offsets: one call per workflow
            out = {}
            for i, a, n in spans:
                f = forces[a:a + n] if kind is Decode else None
                out[i] = self._call(kind, calls[a:a + n], f)
                self._record(kind, 1, n, False)
            return out

    def _record(self, kind, n_wf, n_calls, merged) -> None:
        st = self.engine.last_stats
        self.ticks.append(TickStats("prefill" if kind is Prefill else "decode", n_wf, n_calls,
                                    merged, dict(st.ttft) if kind is Decode else {}))
