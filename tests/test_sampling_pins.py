"""Temperature / top-p sampling pinned to the reference (CPU only).

tests/golden/ref_sampling_*.{json,npz} are the reference Engine's own runs of the fixture
scripts with free decodes, every decode sampled (engine.py:374-392) under three
(temperature, top_p, seed) settings, with the f64 logits each selection saw
(make_golden.py `sampling`).  Here the oracle's ``nucleus`` and the engine's host
sampler must reproduce every sampled token from those logits, and the oracle replays
the whole runs end to end.  The device sampler K6b is pinned to the same goldens in
tests/test_gpu_sampling.py.
"""

import json
import os

import numpy as np
import pytest

from oracle import choreo_oracle as O

from paper_2512_23049_b200.engine import SamplingParams, _sample_nucleus
from paper_2512_23049_b200.tokenizer import generatable_mask

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RUNS = json.load(open(os.path.join(GOLD, "ref_sampling_runs.json")))
LOGITS = np.load(os.path.join(GOLD, "ref_sampling_logits.npz"))
EOS = 257


def selections(key):
    """(msg_id, sel_index, logits row, reference outcome) for every selection of a run;
    outcome is the sampled token, or EOS/None for the selection that ended the message."""
    run = RUNS[key]
    script = json.load(open(os.path.join(GOLD, "scripts", f"{run['script']}.json")))
    forced = {c["name"] for st in script["steps"] for c in st.get("calls", [st]) if "force" in c}
    for st in run["steps"]:
        for m in st["messages"]:
            if m["generated"] is None or m["name"] in forced:
                continue
            rows = LOGITS[f"{key}/{m['name']}"]
            for k, row in enumerate(rows):
                yield m["id"], k, row, (m["generated"][k] if k < len(m["generated"]) else None)


def test_goldens_cover_the_three_settings():
    assert len(RUNS) == 15
    n = sum(1 for k in RUNS for _ in selections(k))
    assert n > 850
    got = {(r["sampling"]["temperature"], r["sampling"]["top_p"], r["sampling"]["seed"])
           for r in RUNS.values()}
    assert got == {(0.7, 0.95, 1), (1.3, 0.5, 2), (0.9, 1.0, 3)}


@pytest.mark.parametrize("key", sorted(RUNS))
def test_oracle_and_host_sampler_reproduce_reference_tokens(key):
    sp = RUNS[key]["sampling"]
    gen = generatable_mask(512)
    so = O.Sampling(mode="temperature", temperature=sp["temperature"], top_p=sp["top_p"],
                    seed=sp["seed"], max_tokens=sp["max_tokens"])
    sh = SamplingParams(mode="temperature", temperature=sp["temperature"], top_p=sp["top_p"],
                        seed=sp["seed"], max_tokens=sp["max_tokens"])
    n_tok = 0
    for mid, k, row, want in selections(key):
        a = O.nucleus(row, O.sampler_mask(512), so, 0, mid, k)
        b = _sample_nucleus(row, gen, sh, 0, mid, k)
        assert a == b
        if want is not None:
            assert a == want, (mid, k)
            n_tok += 1
        else:  # the selection that stopped the message: EOS, or the max_tokens cut
            assert a == EOS or k == sp["max_tokens"]
    assert n_tok > 0


@pytest.mark.parametrize("key", sorted(RUNS))
def test_oracle_replays_sampled_runs(key):
    run = RUNS[key]
    script = json.load(open(os.path.join(GOLD, "scripts", f"{run['script']}.json")))
    script["sampling"] = run["sampling"]
    eng = O.Oracle(O.init_weights(O.TINY), O.TINY, record_logits=True)
    recs = O.run_script(eng, script)
    for got, want in zip(recs, run["steps"], strict=True):
        for gm, wm in zip(got["messages"], want["messages"], strict=True):
            assert (gm["id"], gm["generated"], gm["text"], gm["tokens"]) == \
                (wm["id"], wm["generated"], wm["text"], wm["tokens"])
        for name, rows in (got["logits"] or {}).items():
            np.testing.assert_allclose(np.stack(rows), LOGITS[f"{key}/{name}"], rtol=0,
                                       atol=1e-12)
