"""Workflow scripts and traces over the Engine API (reference script.py:39-398, subset).

A script is {"name", "sampling"?, "steps": [{"op": prefill|prefill_parallel|
decode|decode_parallel, ...}]} with parents named by earlier steps.  ``run_script``
replays it through any engine with the reference call surface and returns a
``Trace`` whose ``forcing()`` teacher-forces a replay (script.py:201-204).
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from .engine import DecodeCall, PrefillCall, SamplingParams
from .errors import ScriptError, TraceMismatchError

OPS = ("prefill", "prefill_parallel", "decode", "decode_parallel")


@dataclass
class MessageResult:
    name: str
    message_id: int
    text: str
    token_count: int
    generated: list | None
    ttft: float | None = None


@dataclass
class StepRecord:
    index: int
    name: str
    op: str
    messages: list
    prefill_flops: int = 0
    decode_flops: int = 0
    tokens_encoded: int = 0
    cache_hit_tokens: int = 0
    repositioned_tokens: int = 0
    wall: float = 0.0
    logits: dict | None = None


@dataclass
class Trace:
    script_name: str
    engine: str
    seed: int
    config: dict
    steps: list = field(default_factory=list)

    def messages(self) -> list:
        return [m for s in self.steps for m in s.messages]

    def message(self, name: str) -> MessageResult:
        for m in self.messages():
            if m.name == name:
                return m
        raise KeyError(name)

    def forcing(self) -> dict:
        return {m.name: list(m.generated) for m in self.messages() if m.generated is not None}

    def ttft_values(self) -> list:
        return [m.ttft for m in self.messages() if m.ttft is not None]

    def total(self, name: str) -> int:
        return sum(getattr(s, name) for s in self.steps)

    def to_jsonl(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(json.dumps({"kind": "trace", "script": self.script_name,
                                 "engine": self.engine, "seed": self.seed,
                                 "config": self.config}, sort_keys=True) + "\n")
            for s in self.steps:
                d = asdict(s)
                d["logits"] = None if s.logits is None else {
                    k: [list(map(float, r)) for r in v] for k, v in s.logits.items()}
                fh.write(json.dumps(d, sort_keys=True) + "\n")


    @classmethod
    def from_jsonl(cls, path) -> "Trace":
        """Inverse of to_jsonl (reference script.py:235-262 reads the same layout)."""
        lines = [json.loads(x) for x in Path(path).read_text(encoding="utf-8").splitlines() if x]
        if not lines or lines[0].get("kind") != "trace":
            raise ScriptError(f"{path}: not a trace file")
        head = lines[0]
        tr = cls(head["script"], head["engine"], head["seed"], head["config"])
        for d in lines[1:]:
            msgs = [MessageResult(**m) for m in d.pop("messages")]
            tr.steps.append(StepRecord(messages=msgs, **d))
        return tr


def diff_traces(a: Trace, b: Trace, *, compare_logits: bool = False,
                atol: float = 1e-9) -> list[str]:
    """What two runs of one script disagree on (reference script.py:348-379).

    Structural differences (other script, other steps / message names) raise
    TraceMismatchError; engine kind, walls and cost counters are not compared.  Returns one
    line per content difference (text, token count, generated ids, optionally logits
    beyond ``atol``); empty when the runs are equivalent.
    """
    if a.script_name != b.script_name:
        raise TraceMismatchError(f"scripts differ: {a.script_name!r} / {b.script_name!r}")
    if len(a.steps) != len(b.steps):
        raise TraceMismatchError(f"{len(a.steps)} vs {len(b.steps)} steps")
    out: list[str] = []
    for sa, sb in zip(a.steps, b.steps):
        if (sa.name, sa.op) != (sb.name, sb.op) or len(sa.messages) != len(sb.messages):
            raise TraceMismatchError(f"step {sa.index} differs in structure")
        for ma, mb in zip(sa.messages, sb.messages):
            if ma.name != mb.name:
                raise TraceMismatchError(f"step {sa.name}: message {ma.name} vs {mb.name}")
            if ma.text != mb.text:
                out.append(f"{ma.name}: text {ma.text!r} != {mb.text!r}")
            if ma.token_count != mb.token_count:
                out.append(f"{ma.name}: token count {ma.token_count} != {mb.token_count}")
            if list(ma.generated or []) != list(mb.generated or []):
                out.append(f"{ma.name}: generated ids differ")
        if compare_logits and (sa.logits is not None or sb.logits is not None):
            if sa.logits is None or sb.logits is None:
                out.append(f"{sa.name}: logits recorded on one side only")
                continue
            for name in sorted(set(sa.logits) | set(sb.logits)):
                ra, rb = sa.logits.get(name), sb.logits.get(name)
                if ra is None or rb is None or len(ra) != len(rb):
                    out.append(f"{name}: logits row counts differ")
                    continue
                for i, (x, y) in enumerate(zip(ra, rb)):
                    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
                    err = float(np.abs(x - y).max()) if x.shape == y.shape and x.size else 0.0
                    if x.shape != y.shape or err > atol:
                        out.append(f"{name}: logits row {i} differ (max abs {err:.3e})")
                        break
    return out


def validate_script(script: dict) -> None:
    if not isinstance(script, dict) or "steps" not in script or "name" not in script:
        raise ScriptError("script needs 'name' and 'steps'")
    seen: set = set()
    for step in script["steps"]:
        op = step.get("op")
        if op not in OPS:
            raise ScriptError(f"bad op {op!r}")
        items = step.get("calls", []) if op.endswith("_parallel") else [step]
        for it in items:
            for p in it.get("parents", []):
                if p not in seen:
                    raise ScriptError(f"unknown parent {p!r}")
        for it in items:
            if it["name"] in seen:
                raise ScriptError(f"duplicate name {it['name']!r}")
            seen.add(it["name"])


def sampling_from_dict(obj, default: SamplingParams | None = None) -> SamplingParams:
    base = default or SamplingParams()
    if not obj:
        return base
    d = asdict(base)
    d.update(obj)
    return SamplingParams(**d)


def run_script(engine, script: dict, force: dict | None = None) -> Trace:
    """script.py:265-298."""
    validate_script(script)
    force = dict(force or {})
    default = sampling_from_dict(script.get("sampling"))
    ids: dict = {}
    trace = Trace(script["name"], engine.kind, engine.seed, engine.config.to_dict())

    def pcall(o):
        return PrefillCall(o["content"], [ids[p] for p in o.get("parents", [])],
                           o.get("offsets"), o.get("new_offset"))

    def dcall(o):
        return DecodeCall(o["header"], [ids[p] for p in o.get("parents", [])], o.get("offsets"),
                          o.get("new_offset"), sampling_from_dict(o.get("sampling"), default))

    for index, step in enumerate(script["steps"]):
        op = step["op"]
        if op == "prefill":
            names, mids = [step["name"]], [engine.prefill(pcall(step))]
        elif op == "prefill_parallel":
            names = [c["name"] for c in step["calls"]]
            mids = engine.prefill_parallel([pcall(c) for c in step["calls"]])
        elif op == "decode":
            names = [step["name"]]
            mids = [engine.decode(dcall(step), force_tokens=force.get(step["name"], step.get("force")))]
        else:
            names = [c["name"] for c in step["calls"]]
            mids = engine.decode_parallel([dcall(c) for c in step["calls"]],
                                          force_tokens=[force.get(c["name"], c.get("force"))
                                                        for c in step["calls"]])
        ids.update(zip(names, mids))
        st = engine.last_stats
        dec = op in ("decode", "decode_parallel")
        msgs = [MessageResult(n, m, engine.message_text(m), engine.message_token_count(m),
                              engine.generated_token_ids(m) if dec else None, st.ttft.get(m))
                for n, m in zip(names, mids)]
        logits = None
        if st.logits is not None:
            by_id = dict(zip(mids, names))
            logits = {by_id[m]: rows for m, rows in st.logits.items()}
        trace.steps.append(StepRecord(index, step["name"], op, msgs, st.prefill_flops,
                                      st.decode_flops, st.tokens_encoded, st.cache_hit_tokens,
                                      st.repositioned_tokens, st.wall, logits))
    return trace


def load_script(path) -> dict:
    return json.loads(Path(path).read_text(encoding="utf-8"))
