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
    """One produced message of a trace; serialised with the reference's keys
    (script.py:126-145: id, tokens)."""

    name: str
    message_id: int
    text: str
    token_count: int
    generated: list | None = None
    ttft: float | None = None

    def to_dict(self) -> dict:
        return {"name": self.name, "id": self.message_id, "text": self.text,
                "tokens": self.token_count, "generated": self.generated, "ttft": self.ttft}

    @classmethod
    def from_dict(cls, d: dict) -> "MessageResult":
        return cls(d["name"], d["id"], d["text"], d["tokens"], d.get("generated"),
                   d.get("ttft"))


_COUNTERS = ("prefill_flops", "decode_flops", "tokens_encoded", "cache_hit_tokens",
             "repositioned_tokens")


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

    def to_dict(self) -> dict:
        """Reference layout (script.py:161-171): ``logits`` only when recorded."""
        d = {"index": self.index, "name": self.name, "op": self.op,
             "messages": [m.to_dict() for m in self.messages], "wall": self.wall}
        d.update({k: getattr(self, k) for k in _COUNTERS})
        if self.logits is not None:
            d["logits"] = {k: [[float(x) for x in row] for row in rows]
                           for k, rows in self.logits.items()}
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "StepRecord":
        return cls(d["index"], d["name"], d["op"],
                   [MessageResult.from_dict(m) for m in d["messages"]],
                   *(d.get(k, 0) for k in _COUNTERS), d.get("wall", 0.0), d.get("logits"))


@dataclass
class Trace:
    script_name: str
    engine: str
    seed: int
    config: dict
    steps: list = field(default_factory=list)
    meta: dict = field(default_factory=dict)

    def messages(self) -> list:
        return [m for s in self.steps for m in s.messages]

    def message(self, name: str) -> MessageResult:
        for m in self.messages():
            if m.name == name:
                return m
        raise KeyError(f"no message named {name!r} in trace")

    def forcing(self) -> dict:
        return {m.name: list(m.generated) for m in self.messages() if m.generated is not None}

    def ttft_values(self) -> list:
        return [m.ttft for m in self.messages() if m.ttft is not None]

    def total(self, name: str) -> int:
        return sum(getattr(s, name) for s in self.steps)

    def total_wall(self) -> float:
        return sum(s.wall for s in self.steps)

    def canonical(self) -> dict:
        """Timing-free rendering (script.py:215-224)."""
        steps = []
        for s in self.steps:
            d = s.to_dict()
            d["wall"] = 0.0
            d["messages"] = [dict(m, ttft=None) for m in d["messages"]]
            steps.append(d)
        return {"script": self.script_name, "engine": self.engine, "seed": self.seed,
                "config": self.config, "meta": self.meta, "steps": steps}

    def to_jsonl(self, path) -> None:
        """One header line {kind, script, engine, seed, config, meta}, then one line per
        step -- the reference's file layout (script.py:226-233), readable by its
        ``Trace.from_jsonl`` and ``choreo diff``."""
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(json.dumps({"kind": "trace", "script": self.script_name,
                                 "engine": self.engine, "seed": self.seed,
                                 "config": self.config, "meta": self.meta},
                                sort_keys=True) + "\n")
            for s in self.steps:
                fh.write(json.dumps(s.to_dict(), sort_keys=True) + "\n")

    @classmethod
    def from_jsonl(cls, path) -> "Trace":
        """Reads traces written by either engine; malformed files raise ScriptError
        (script.py:235-251)."""
        try:
            text = Path(path).read_text(encoding="utf-8")
        except OSError as exc:
            raise ScriptError(f"{path}: {exc}") from exc
        lines = [x for x in text.splitlines() if x.strip()]
        if not lines:
            raise ScriptError(f"{path}: empty trace file")
        try:
            head = json.loads(lines[0])
            if not isinstance(head, dict) or head.get("kind") != "trace":
                raise ScriptError(f"{path}: not a trace file")
            steps = [StepRecord.from_dict(json.loads(x)) for x in lines[1:]]
            return cls(head["script"], head["engine"], head["seed"], head.get("config", {}),
                       steps, head.get("meta", {}))
        except (json.JSONDecodeError, KeyError, TypeError, AttributeError) as exc:
            raise ScriptError(f"{path}: malformed trace: {exc}") from exc


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


_SAMPLING_KEYS = {"mode", "temperature", "top_p", "seed", "max_tokens"}


def _nonempty_str(x) -> bool:
    return isinstance(x, str) and bool(x)


def validate_script(script) -> None:
    """Every malformed script raises ScriptError before any engine call (the checks of
    reference script.py:39-123: names, ops, parallel call lists, content / header
    types, parents produced by earlier steps, offsets, new_offset, force, sampling)."""
    if not isinstance(script, dict):
        raise ScriptError("script must be a JSON object")
    if not _nonempty_str(script.get("name")):
        raise ScriptError("script needs a non-empty 'name'")
    if "sampling" in script:
        _check_sampling(script["sampling"], "script")
    steps = script.get("steps")
    if not isinstance(steps, list) or not steps:
        raise ScriptError("script needs a non-empty 'steps' list")
    seen: set = set()
    for i, step in enumerate(steps):
        if not isinstance(step, dict):
            raise ScriptError(f"step {i}: must be an object")
        if not _nonempty_str(step.get("name")):
            raise ScriptError(f"step {i}: needs a non-empty 'name'")
        where = f"step {i} ({step['name']})"
        if step["name"] in seen:
            raise ScriptError(f"{where}: duplicate name")
        op = step.get("op")
        if op not in OPS:
            raise ScriptError(f"{where}: unknown op {op!r}")
        lone = op in ("prefill", "decode")
        calls = [step] if lone else step.get("calls")
        if not isinstance(calls, list) or not calls:
            raise ScriptError(f"{where}: parallel op needs a non-empty 'calls' list")
        if not lone and not all(isinstance(c, dict) and _nonempty_str(c.get("name"))
                                for c in calls):
            raise ScriptError(f"{where}: every call needs a non-empty 'name'")
        names = [c["name"] for c in calls] + ([] if lone else [step["name"]])
        if len(set(names)) != len(names):
            raise ScriptError(f"{where}: duplicate names within the step")
        if set(names) & seen:
            raise ScriptError(f"{where}: duplicate name {sorted(set(names) & seen)}")
        for c in calls:
            _check_call(c, op, seen, where)
        seen |= set(names)


def _check_call(call: dict, op: str, produced: set, where: str) -> None:
    key = "content" if op.startswith("prefill") else "header"
    if not isinstance(call.get(key), str):
        raise ScriptError(f"{where}: missing or non-string '{key}'")
    parents = call.get("parents", [])
    if not isinstance(parents, list):
        raise ScriptError(f"{where}: 'parents' must be a list of names")
    for p in parents:
        if not isinstance(p, str):
            raise ScriptError(f"{where}: parent {p!r} is not a name")
        if p not in produced:
            raise ScriptError(f"{where}: parent {p!r} is not produced by an earlier step")
    offs = call.get("offsets")
    if offs is not None and (not isinstance(offs, list) or len(offs) != len(parents) or any(
            not (o is None or (isinstance(o, int) and not isinstance(o, bool))) for o in offs)):
        raise ScriptError(f"{where}: 'offsets' must match parents (ints or nulls)")
    no = call.get("new_offset")
    if no is not None and (not isinstance(no, int) or isinstance(no, bool)):
        raise ScriptError(f"{where}: 'new_offset' must be an int")
    if "sampling" in call:
        _check_sampling(call["sampling"], where)
    force = call.get("force")
    if force is not None and not isinstance(force, str) and not (
            isinstance(force, list) and all(isinstance(t, int) for t in force)):
        raise ScriptError(f"{where}: 'force' must be a string or a token id list")


def _check_sampling(obj, where: str) -> None:
    if not isinstance(obj, dict):
        raise ScriptError(f"{where}: 'sampling' must be an object")
    bad = set(obj) - _SAMPLING_KEYS
    if bad:
        raise ScriptError(f"{where}: unknown sampling keys {sorted(bad)}")


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
    """script.py:29-36: invalid JSON and invalid scripts raise ScriptError."""
    try:
        obj = json.loads(Path(path).read_text(encoding="utf-8"))
    except json.JSONDecodeError as exc:
        raise ScriptError(f"{path}: invalid JSON: {exc}") from exc
    validate_script(obj)
    return obj
