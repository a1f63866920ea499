"""Pin the CPU oracle to the reference before trusting it (CPU only).

Golden vectors come from two places, both committed under tests/golden/:
- the reference's own fixtures (weights sha256, Fig. 2 mask panels, the
  canonical conversation trace), copied verbatim by make_golden.py;
- outputs of the reference run in the build container by make_golden.py
  (per-script traces, cache metadata and recorded logits, for f64 weights and
  for bf16-rounded weights, plus the C1 choreography).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import choreo_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


PINS = _load("ref_pins.json")
SCRIPTS = sorted(n[:-5] for n in os.listdir(os.path.join(GOLD, "scripts")))


def _weights(variant):
    w = O.init_weights(O.TINY)
    return w if variant == "f64" else O.round_weights(w, variant)


def test_weights_sha_matches_reference_fixture():
    assert O.weights_sha256(O.init_weights(O.TINY), O.TINY) == \
        PINS["weights_default_seed0"]["sha256"]


def test_weight_file_roundtrip():
    w = O.init_weights(O.SMALL)
    shape, w2 = O.parse_weights_file(O.weights_file_bytes(w, O.SMALL))
    assert shape == O.SMALL
    np.testing.assert_array_equal(w2["layers"][1]["w_down"],
                                  w["layers"][1]["w_down"].astype(np.float32))


@pytest.mark.parametrize("key", sorted(PINS["rope_tables"]))
def test_rope_tables_bitwise(key):
    hd, W, base = key.split("_")
    c, s = O.rope_tables(int(hd), int(W), float(base))
    assert hashlib.sha256(c.tobytes()).hexdigest() == PINS["rope_tables"][key]["cos_sha256"]
    assert hashlib.sha256(s.tobytes()).hexdigest() == PINS["rope_tables"][key]["sin_sha256"]


def test_rotation_known_answers():
    kat = PINS["rotation_kat"]
    rot = O.Rotor(O.TINY)
    k = np.asarray(kat["k"])
    for dl, want in zip(kat["deltas"], kat["out"]):
        np.testing.assert_array_equal(rot.by_delta(k, dl), np.asarray(want))
    with pytest.raises(O.OracleError):
        rot.by_delta(k, 2049)


def test_prefill_mask_panel():
    eng = O.Oracle(O.init_weights(O.SMALL), O.SMALL)
    par = [eng.prefill({"message": t}) for t in "abc"]
    st = eng.store
    batch = [(100, j) for j in range(3)] + [(101, j) for j in range(3)]
    m = O.dense_mask(batch, st.mid[:st.n], st.pos[:st.n], {100: (par[0],), 101: (par[1], par[2])})
    assert m.astype(int).tolist() == PINS["mask_prefill_parallel"]["mask"]


def test_decode_mask_panel():
    st = O.Store(O.SMALL, 64)
    z = np.zeros((O.SMALL.n_layers, 1, O.SMALL.kv_heads, O.SMALL.head_dim))
    for m in range(3):
        st.msgs[m] = O.Msg("prefilled", 0, "", None)
        for j in range(2):
            st.append(m, [0], [j], z, z)
    for m in (3, 4, 5):
        st.msgs[m] = O.Msg("decoded", 2, "", "x")
    for m in (3, 4, 5):
        st.append(m, [0], [2], z, z)
    m = O.dense_mask([(mm, 3) for mm in (3, 4, 5)], st.mid[:st.n], st.pos[:st.n],
                     {mm: (mm - 3,) for mm in (3, 4, 5)})
    assert m.astype(int).tolist() == PINS["mask_decode_parallel"]["mask"]


def test_conversation_reference_trace():
    ref = PINS["conversation_reference"]
    script = _load("scripts/conversation.json")
    recs = O.run_script(O.Oracle(O.init_weights(O.TINY), O.TINY), script)
    assert len(recs) == len(ref["steps"])
    for got, want in zip(recs, ref["steps"]):
        for key in ("prefill_flops", "decode_flops", "tokens_encoded", "cache_hit_tokens",
                    "repositioned_tokens"):
            assert got[key] == want[key], (got["name"], key)
        for gm, wm in zip(got["messages"], want["messages"]):
            assert gm["generated"] == wm["generated"]
            assert gm["text"] == wm["text"] and gm["tokens"] == wm["tokens"]


@pytest.mark.parametrize("variant", ["f64", "bf16"])
@pytest.mark.parametrize("script", SCRIPTS)
def test_fixture_script_matches_reference(variant, script):
    runs = _load(f"ref_runs_{variant}.json")[script]
    logits = np.load(os.path.join(GOLD, f"ref_logits_{variant}.npz"))
    eng = O.Oracle(_weights(variant), O.TINY, record_logits=True)
    recs = O.run_script(eng, _load(f"scripts/{script}.json"))
    for got, want in zip(recs, runs["steps"], strict=True):
        for key in ("prefill_flops", "decode_flops", "tokens_encoded", "cache_hit_tokens",
                    "repositioned_tokens"):
            assert got[key] == want[key], (got["name"], key)
        for gm, wm in zip(got["messages"], want["messages"], strict=True):
            assert (gm["id"], gm["generated"], gm["text"], gm["tokens"]) == \
                (wm["id"], wm["generated"], wm["text"], wm["tokens"])
        for name, rows in (got["logits"] or {}).items():
            np.testing.assert_allclose(np.stack(rows), logits[f"{script}/{name}"], rtol=0, atol=1e-12)
    st = eng.store
    assert st.mid[:st.n].tolist() == runs["msg_ids"]
    assert st.pos[:st.n].tolist() == runs["positions"]
    assert st.tok[:st.n].tolist() == runs["token_ids"]


def run_c1(eng):
    t = PINS["c1_texts"]
    a = eng.prefill({"message": t["A"]})
    b = eng.prefill({"message": t["B"]})
    c = eng.prefill({"message": t["C"]})
    m = eng.decode({"header": "Answer:", "parents": [c, a], "offsets": [0, 37],
                    "sampling": O.Sampling(max_tokens=16)})
    return [a, b, c, m]


@pytest.mark.parametrize("variant", ["f64", "bf16"])
def test_c1_choreography_matches_reference(variant):
    want = _load(f"ref_runs_{variant}.json")["C1"]
    logits = np.load(os.path.join(GOLD, f"ref_logits_{variant}.npz"))["C1/answer"]
    eng = O.Oracle(_weights(variant), O.TINY, record_logits=True)
    ids = run_c1(eng)
    assert ids == want["ids"]
    assert eng.generated(ids[3]) == want["generated"]
    assert eng.stats[-1].repositioned_tokens == want["repositioned"]
    st = eng.store
    assert st.pos[:st.n].tolist() == want["positions"]
    assert st.mid[:st.n].tolist() == want["msg_ids"]
    np.testing.assert_allclose(np.stack(eng.stats[-1].logits[ids[3]]), logits, rtol=0, atol=1e-12)


def test_gqa_reduces_to_mha():
    mha = O.Shape(n_layers=2, n_heads=4, head_dim=8, ffn_dim=32, vocab_size=300, context_window=128)
    same = O.Shape(n_layers=2, n_heads=4, head_dim=8, ffn_dim=32, vocab_size=300,
                   context_window=128, n_kv_heads=4)
    w1, w2 = O.init_weights(mha), O.init_weights(same)
    assert O.weights_sha256(w1, mha) == O.weights_sha256(w2, same)
    outs = []
    for shape, w in ((mha, w1), (same, w2)):
        e = O.Oracle(w, shape, record_logits=True)
        a = e.prefill({"message": "parent text"})
        m = e.decode({"header": "Q:", "parents": [a], "offsets": [3],
                      "sampling": O.Sampling(max_tokens=4)})
        outs.append(np.stack(e.stats[-1].logits[m]))
    np.testing.assert_array_equal(outs[0], outs[1])


def test_gqa_parallel_equals_lone():
    shape = O.Shape(n_layers=2, n_heads=4, head_dim=8, ffn_dim=32, vocab_size=300,
                    context_window=128, n_kv_heads=2)
    e = O.Oracle(O.init_weights(shape), shape, record_logits=True)
    a = e.prefill({"message": "first parent"})
    b = e.prefill({"message": "second parent"})
    calls = [{"header": "A:", "parents": [a], "offsets": [20], "sampling": O.Sampling(max_tokens=5)},
             {"header": "B:", "parents": [b, a], "offsets": [0, 20], "sampling": O.Sampling(max_tokens=5)}]
    par, lone = e.clone(), e.clone()
    pids = par.decode_batch(calls)
    for i, c in enumerate(calls):
        m = lone.decode(c)
        assert m == pids[i]
        assert lone.generated(m) == par.generated(m)
        np.testing.assert_allclose(np.stack(lone.stats[-1].logits[m]),
                                   np.stack(par.stats[-1].logits[m]), rtol=0, atol=1e-10)
