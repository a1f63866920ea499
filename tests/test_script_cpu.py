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


REF_TRACE = os.path.join(GOLD, "ref_trace_branching.jsonl")


def test_reads_a_trace_written_by_the_reference(tmp_path):
    """tests/golden/ref_trace_branching.jsonl was written by the reference's own
    Trace.to_jsonl (make_golden.py `trace`): it loads, equals the recorded run, and our
    writer reproduces its layout key for key (so the reference's `diff` reads ours)."""
    tr = Trace.from_jsonl(REF_TRACE)
    assert tr.script_name == "branching" and tr.meta == {}
    assert diff_traces(tr, _trace()) == []
    assert tr.steps[-1].logits  # recorded logits come back
    p = tmp_path / "ours.jsonl"
    tr.to_jsonl(p)
    ref_lines = [json.loads(x) for x in open(REF_TRACE)]
    our_lines = [json.loads(x) for x in open(p)]

    def keys(d):
        return {k: (keys(v) if isinstance(v, dict) and k != "logits" else
                    [keys(m) for m in v] if k == "messages" else None) for k, v in d.items()}
    assert [keys(d) for d in our_lines] == [keys(d) for d in ref_lines]
    assert diff_traces(Trace.from_jsonl(p), tr, compare_logits=True, atol=0.0) == []


@pytest.mark.parametrize("text", ["", "not json\n", '{"kind": "other"}\n',
                                  '{"kind": "trace"}\n',
                                  '{"kind": "trace", "script": "s", "engine": "e", "seed": 0}\n'
                                  '{"index": 0}\n'])
def test_malformed_trace_raises_script_error(tmp_path, text):
    from paper_2512_23049_b200.errors import ScriptError
    p = tmp_path / "bad.jsonl"
    p.write_text(text)
    with pytest.raises(ScriptError):
        Trace.from_jsonl(p)


@pytest.mark.parametrize("mutate", [
    lambda s: s.update(name=""),
    lambda s: s.update(steps=[]),
    lambda s: s["steps"][0].update(name=""),
    lambda s: s["steps"][0].update(op="encode"),
    lambda s: s["steps"][0].update(content=5),
    lambda s: s["steps"][1].update(parents=["nope"]),
    lambda s: s["steps"][1].update(parents="u1"),
    lambda s: s["steps"][1].update(offsets=[0, 1]),
    lambda s: s["steps"][1].update(offsets=["0"]),
    lambda s: s["steps"][1].update(new_offset=1.5),
    lambda s: s["steps"][1].update(sampling={"temp": 1}),
    lambda s: s["steps"][1].update(force=[1, "a"]),
    lambda s: s.update(sampling=[]),
    lambda s: s["steps"].append(dict(s["steps"][0])),
    lambda s: s["steps"].append({"name": "par", "op": "decode_parallel", "calls": []}),
    lambda s: s["steps"].append({"name": "par", "op": "decode_parallel",
                                 "calls": [{"name": "x", "header": "h"},
                                           {"name": "x", "header": "h"}]}),
])
def test_validate_script_rejects_malformed_scripts_up_front(mutate):
    """The reference's script checks (script.py:39-123): every malformed script raises
    ScriptError before any engine call."""
    from paper_2512_23049_b200.errors import ScriptError
    from paper_2512_23049_b200.script import validate_script
    script = json.load(open(os.path.join(GOLD, "scripts", "branching.json")))
    validate_script(copy.deepcopy(script))
    assert script["steps"][1].get("parents")
    mutate(script)
    with pytest.raises(ScriptError):
        validate_script(script)
