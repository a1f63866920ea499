"""Trace files and trace diffing (reference script.py:226-262, 348-379) on the reference's
own recorded runs (tests/golden/ref_runs_f64.json): jsonl round trip, equivalence, content
differences reported per message, structural mismatches raised, cost fields ignored."""

import copy
import json
import os

import pytest

from paper_2512_23049_b200.__main__ import main
from paper_2512_23049_b200.errors import TraceMismatchError
from paper_2512_23049_b200.script import MessageResult, StepRecord, Trace, diff_traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _trace(script="branching", engine="choreo"):
    run = json.load(open(os.path.join(GOLD, "ref_runs_f64.json")))[script]
    tr = Trace(script, engine, 0, {"n_layers": 4})
    for st in run["steps"]:
        msgs = [MessageResult(m["name"], m["id"], m["text"], m["tokens"], m["generated"])
                for m in st["messages"]]
        tr.steps.append(StepRecord(st["index"], st["name"], st["op"], msgs, st["prefill_flops"],
                                   st["decode_flops"], st["tokens_encoded"],
                                   st["cache_hit_tokens"], st["repositioned_tokens"]))
    return tr


def test_jsonl_round_trip_and_self_equivalence(tmp_path):
    tr = _trace()
    p = tmp_path / "t.jsonl"
    tr.to_jsonl(p)
    back = Trace.from_jsonl(p)
    assert back.script_name == tr.script_name and len(back.steps) == len(tr.steps)
    assert back.forcing() == tr.forcing()
    assert diff_traces(tr, back) == []


def test_cost_fields_and_engine_kind_are_ignored():
    a, b = _trace(), _trace(engine="baseline")
    for s in b.steps:
        s.prefill_flops += 7
        s.cache_hit_tokens = 0
        s.wall = 3.0
    assert diff_traces(a, b) == []


def test_content_differences_are_listed():
    a = _trace()
    b = copy.deepcopy(a)
    dec = next(m for s in b.steps for m in s.messages if m.generated)
    dec.generated = list(dec.generated[:-1]) + [dec.generated[-1] ^ 1]
    dec.text += "!"
    diffs = diff_traces(a, b)
    assert any("generated ids differ" in d for d in diffs)
    assert any("text" in d for d in diffs)


def test_structural_mismatch_raises():
    a = _trace()
    with pytest.raises(TraceMismatchError):
        diff_traces(a, _trace("tot"))
    b = copy.deepcopy(a)
    b.steps.pop()
    with pytest.raises(TraceMismatchError):
        diff_traces(a, b)


def test_logit_tolerance():
    a = _trace()
    b = copy.deepcopy(a)
    a.steps[-1].logits = {"x": [[0.0, 1.0]]}
    b.steps[-1].logits = {"x": [[0.0, 1.0 + 1e-6]]}
    assert diff_traces(a, b, compare_logits=True, atol=1e-5) == []
    assert diff_traces(a, b, compare_logits=True, atol=1e-9)


def test_cli_diff_exit_codes(tmp_path, capsys):
    a = _trace()
    b = copy.deepcopy(a)
    pa, pb = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    a.to_jsonl(pa)
    b.to_jsonl(pb)
    assert main(["diff", str(pa), str(pb)]) == 0
    b.steps[-1].messages[-1].text = "changed"
    b.to_jsonl(pb)
    assert main(["diff", str(pa), str(pb)]) == 1
    assert "difference" in capsys.readouterr().out
