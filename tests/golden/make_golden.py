"""Generate the golden vectors that pin oracle/choreo_oracle.py to the reference.

Runs ONLY in the build container, where the read-only reference package lives
at /root/reference/pkg/src (it does not exist on the GPU box, so nothing at
test/bench time may import it).  Everything it writes is committed under
tests/golden/ and is small:

  ref_pins.json           reference fixture goldens (weights sha256, mask panels,
                          conversation trace) + rope-table digests + C1 result
  scripts/*.json          the 10 reference fixture scripts (inputs), verbatim
  ref_runs_<variant>.json per-script reference traces + cache metadata
  ref_logits_<variant>.npz per-selection logits recorded by the reference
                          (record_logits=True), key "<script>/<message>"
  ref_baseline_runs.json  the same scripts through the reference BaselineEngine
  ref_baseline_logits.npz (re-encoding comparator, f64 weights): traces with its
                          cost counters (flops, tokens encoded, trie hits) + logits
  ref_sampling_runs.json  temperature / top-p runs of the scripts with free decodes,
  ref_sampling_logits.npz f64 weights, three (temperature, top_p, seed) settings: the
                          reference's sampled tokens and the logits each selection saw
                          (engine.py:374-392 -- pins K6b and the oracle's nucleus())
  ref_trace_branching.jsonl  a trace file written by the reference's Trace.to_jsonl

variants: "f64"  = init_weights(DEFAULT_CONFIG) as the reference builds it;
          "bf16" = the same weights rounded to bfloat16 (RNE) and upcast, the
                   weight set both sides share for the bf16 GPU parity runs.

Usage:  python tests/golden/make_golden.py [part ...]   (parts: core sampling trace;
        default all)
"""

from __future__ import annotations

import hashlib
import json
import shutil
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(HERE.parent.parent))

from choreo.baseline import BaselineEngine  # noqa: E402  (reference, read-only)
from choreo.config import DEFAULT_CONFIG  # noqa: E402
from choreo.engine import DecodeCall, Engine, PrefillCall, SamplingParams  # noqa: E402
from choreo.model import WeightSet, LayerWeights, init_weights  # noqa: E402
from choreo.script import run_script  # noqa: E402
from choreo.tensor import RotationTable  # noqa: E402

from oracle.choreo_oracle import round_weights  # noqa: E402

SCRIPTS = ["branching", "bsm", "conversation", "doc_qa", "maditer", "madpar",
           "multiqa_chained", "multiqa_parallel", "multiqa_serial", "tot"]

# C1: three prefilled messages at offset 0, then a decode that
# reads C then A, skipping B, with a gap of 5 and A moved by +37.
C1_TEXTS = {"A": "System: answer the question using the notes.",
            "B": "Note: the river is long.",
            "C": "Question: which river is long?"}


def ref_weights(variant: str) -> WeightSet:
    w = init_weights(DEFAULT_CONFIG)
    if variant == "f64":
        return w
    as_dict = {"embed": w.embed, "out_norm": w.out_norm, "out_head": w.out_head,
               "layers": [{k: getattr(lw, k) for k in ("attn_norm", "wq", "wk", "wv", "wo",
                                                         "ffn_norm", "w_gate", "w_up", "w_down")}
                          for lw in w.layers]}
    r = round_weights(as_dict, variant)
    return WeightSet(config=w.config, embed=r["embed"], out_norm=r["out_norm"],
                     out_head=r["out_head"],
                     layers=[LayerWeights(**lw) for lw in r["layers"]])


def run_c1(weights: WeightSet) -> dict:
    eng = Engine(weights, seed=0, record_logits=True)
    a = eng.prefill(PrefillCall(C1_TEXTS["A"]))
    b = eng.prefill(PrefillCall(C1_TEXTS["B"]))
    c = eng.prefill(PrefillCall(C1_TEXTS["C"]))
    m = eng.decode(DecodeCall("Answer:", parents=[c, a], offsets=[0, 37],
                              sampling=SamplingParams(max_tokens=16)))
    n = eng.cache.token_count
    return {"ids": [a, b, c, m], "generated": eng.generated_token_ids(m),
            "text": eng.message_text(m),
            "msg_ids": eng.cache.msg_ids[:n].tolist(),
            "positions": eng.cache.positions[:n].tolist(),
            "token_ids": eng.cache.token_ids[:n].tolist(),
            "repositioned": eng.last_stats.repositioned_tokens,
            "logits": np.stack(eng.last_stats.logits[m])}


def _trace_steps(trace, name: str, logits: dict) -> list:
    steps = []
    for s in trace.steps:
        d = s.to_dict()
        d.pop("wall", None)
        lg = d.pop("logits", None) or {}
        for msg_name, rows in lg.items():
            logits[f"{name}/{msg_name}"] = np.asarray(rows, dtype=np.float64)
        for m in d["messages"]:
            m.pop("ttft", None)
        steps.append(d)
    return steps


def run_variant(variant: str) -> tuple[dict, dict]:
    weights = ref_weights(variant)
    runs, logits = {}, {}
    for name in SCRIPTS:
        script = json.loads((REF / "fixtures" / "scripts" / f"{name}.json").read_text())
        eng = Engine(weights, seed=0, record_logits=True)
        trace = run_script(eng, script)
        n = eng.cache.token_count
        runs[name] = {"steps": _trace_steps(trace, name, logits),
                      "msg_ids": eng.cache.msg_ids[:n].tolist(),
                      "positions": eng.cache.positions[:n].tolist(),
                      "token_ids": eng.cache.token_ids[:n].tolist()}
    c1 = run_c1(weights)
    logits["C1/answer"] = c1.pop("logits")
    runs["C1"] = c1
    return runs, logits


def run_baseline() -> tuple[dict, dict]:
    weights = ref_weights("f64")
    runs, logits = {}, {}
    for name in SCRIPTS:
        script = json.loads((REF / "fixtures" / "scripts" / f"{name}.json").read_text())
        for cache in (True, False):
            key = name if cache else f"{name}@nocache"
            eng = BaselineEngine(weights, seed=0, prefix_cache=cache, record_logits=cache)
            runs[key] = {"steps": _trace_steps(run_script(eng, script), key, logits)}
    return runs, logits


SAMPLING_SCRIPTS = ["branching", "bsm", "conversation", "maditer", "tot"]
SAMPLING_SETTINGS = [(0.7, 0.95, 1), (1.3, 0.5, 2), (0.9, 1.0, 3)]


def run_sampling() -> tuple[dict, dict]:
    """The scripts with free decodes, every decode sampled with temperature + top-p."""
    weights = ref_weights("f64")
    runs, logits = {}, {}
    for t, top_p, seed in SAMPLING_SETTINGS:
        for name in SAMPLING_SCRIPTS:
            script = json.loads((REF / "fixtures" / "scripts" / f"{name}.json").read_text())
            script["sampling"] = dict(script.get("sampling", {}), mode="temperature",
                                      temperature=t, top_p=top_p, seed=seed)
            key = f"{name}@T{t}_p{top_p}_s{seed}"
            eng = Engine(weights, seed=0, record_logits=True)
            trace = run_script(eng, script)
            runs[key] = {"script": name, "sampling": script["sampling"],
                         "steps": _trace_steps(trace, key, logits)}
    return runs, logits


def write_ref_trace() -> None:
    """A trace file in the reference's own jsonl layout (read by tests/test_script_cpu)."""
    script = json.loads((REF / "fixtures" / "scripts" / "branching.json").read_text())
    eng = Engine(ref_weights("f64"), seed=0, record_logits=True)
    run_script(eng, script).to_jsonl(HERE / "ref_trace_branching.jsonl")


def main() -> None:
    parts = set(sys.argv[1:]) or {"core", "sampling", "trace"}
    if "sampling" in parts:
        runs, logits = run_sampling()
        (HERE / "ref_sampling_runs.json").write_text(json.dumps(runs, sort_keys=True) + "\n")
        np.savez_compressed(HERE / "ref_sampling_logits.npz", **logits)
        print("sampling selections:", sum(len(v) for v in logits.values()))
    if "trace" in parts:
        write_ref_trace()
    if "core" not in parts:
        return
    (HERE / "scripts").mkdir(exist_ok=True)
    for name in SCRIPTS:
        shutil.copyfile(REF / "fixtures" / "scripts" / f"{name}.json",
                        HERE / "scripts" / f"{name}.json")
    pins = {
        "weights_default_seed0": json.loads(
            (REF / "fixtures" / "golden" / "weights_default_seed0.json").read_text()),
        "conversation_reference": json.loads(
            (REF / "fixtures" / "golden" / "conversation_reference.json").read_text()),
        "mask_prefill_parallel": json.loads(
            (REF / "fixtures" / "masks" / "prefill_parallel.json").read_text()),
        "mask_decode_parallel": json.loads(
            (REF / "fixtures" / "masks" / "decode_parallel.json").read_text()),
        "rope_tables": {},
        "c1_texts": C1_TEXTS,
    }
    for hd, W, base in ((16, 2048, 10000.0), (8, 256, 10000.0), (128, 4096, 500000.0)):
        t = RotationTable(hd, W, base)
        pins["rope_tables"][f"{hd}_{W}_{base}"] = {
            "cos_sha256": hashlib.sha256(t.cos.tobytes()).hexdigest(),
            "sin_sha256": hashlib.sha256(t.sin.tobytes()).hexdigest()}
    # rotation known-answer vectors: rotate(k, delta) for a fixed random k
    rng = np.random.default_rng(1234)
    t = RotationTable(16, 2048)
    k = rng.standard_normal((5, 4, 16))
    pins["rotation_kat"] = {"k": k.tolist(), "deltas": [-2048, -37, 0, 1, 37, 2048],
                            "out": [t.rotate(k, dl).tolist() for dl in (-2048, -37, 0, 1, 37, 2048)]}
    for variant in ("f64", "bf16"):
        runs, logits = run_variant(variant)
        (HERE / f"ref_runs_{variant}.json").write_text(json.dumps(runs, sort_keys=True) + "\n")
        np.savez_compressed(HERE / f"ref_logits_{variant}.npz", **logits)
        print(variant, "selections:", sum(len(v) for v in logits.values()))
    runs, logits = run_baseline()
    (HERE / "ref_baseline_runs.json").write_text(json.dumps(runs, sort_keys=True) + "\n")
    np.savez_compressed(HERE / "ref_baseline_logits.npz", **logits)
    print("baseline selections:", sum(len(v) for v in logits.values()))
    (HERE / "ref_pins.json").write_text(json.dumps(pins, sort_keys=True, indent=1) + "\n")


if __name__ == "__main__":
    main()
