"""Re-encoding comparator (BaselineEngine) on the B200 against the reference's own
BaselineEngine (golden traces + logits recorded from it, tests/golden/make_golden.py).

Cost counters (prefill/decode FLOPs, tokens encoded, trie hits) must match exactly,
generated tokens exactly, logits within the f32 tolerance (1e-4).  The remaining
tests follow the reference's test_baseline.py behaviours.
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2512_23049_b200 as P  # noqa: E402
from paper_2512_23049_b200.baseline import BaselineEngine  # noqa: E402
from paper_2512_23049_b200.script import run_script  # noqa: E402
from paper_2512_23049_b200.tokenizer import frame_header, frame_message  # noqa: E402

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SCRIPTS = sorted(n[:-5] for n in os.listdir(os.path.join(GOLD, "scripts")))
with open(os.path.join(GOLD, "ref_baseline_runs.json")) as fh:
    RUNS = json.load(fh)
LOGITS = np.load(os.path.join(GOLD, "ref_baseline_logits.npz"))

_W = {}


def _weights(mode="f32"):
    if mode not in _W:
        ws = P.init_weights(P.DEFAULT_CONFIG)
        if mode == "f32":
            _W[mode] = P.DeviceWeights.from_host(ws, dtype=torch.float32)
        else:
            _W[mode] = P.DeviceWeights.from_host(ws.rounded("bf16"), dtype=torch.bfloat16)
    return _W[mode]


def _script(name):
    with open(os.path.join(GOLD, "scripts", f"{name}.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("cache", [True, False])
@pytest.mark.parametrize("script", SCRIPTS)
def test_fixture_scripts_match_reference_baseline(script, cache):
    key = script if cache else f"{script}@nocache"
    want = RUNS[key]
    eng = BaselineEngine(_weights(), prefix_cache=cache, record_logits=cache)
    trace = run_script(eng, _script(script))
    assert trace.engine == "baseline"
    worst = 0.0
    for got, ws in zip(trace.steps, want["steps"], strict=True):
        for k in ("prefill_flops", "decode_flops", "tokens_encoded", "cache_hit_tokens",
                  "repositioned_tokens"):
            assert getattr(got, k) == ws[k], (got.name, k)
        for gm, wm in zip(got.messages, ws["messages"], strict=True):
            assert (gm.message_id, gm.generated, gm.text, gm.token_count) == \
                (wm["id"], wm["generated"], wm["text"], wm["tokens"])
        for name, rows in (got.logits or {}).items():
            ref = LOGITS[f"{key}/{name}"]
            assert len(rows) == len(ref)
            worst = max(worst, float(np.abs(np.stack(rows) - ref).max()))
    assert worst <= 1e-4, f"max |dlogit| {worst:.3e}"


def _small_weights(dtype=torch.float32):
    cfg = P.ModelConfig(n_layers=2, n_heads=2, head_dim=8, ffn_dim=64, vocab_size=512,
                        context_window=256)
    return P.DeviceWeights.from_host(P.init_weights(cfg), dtype=dtype)


def test_offsets_and_new_offset_are_ignored():
    w = _small_weights()

    def run(**layout):
        e = BaselineEngine(w, record_logits=True)
        a = e.prefill(P.PrefillCall("context one"))
        b = e.prefill(P.PrefillCall("context two"))
        m = e.decode(P.DecodeCall("Q:", parents=[a, b], sampling=P.SamplingParams(max_tokens=5),
                                  **layout))
        return e.generated_token_ids(m), e.last_stats.logits[m]

    t0, l0 = run()
    t1, l1 = run(offsets=[40, 7], new_offset=99)
    assert t0 == t1
    for x, y in zip(l0, l1):
        assert np.array_equal(x, y)


def test_repeat_decode_reencodes_only_last_header_token():
    e = BaselineEngine(_small_weights())
    a = e.prefill(P.PrefillCall("shared long context here"))
    call = P.DecodeCall("Ans:", parents=[a], sampling=P.SamplingParams(max_tokens=4))
    m1 = e.decode(call)
    first = e.last_stats
    known = len(frame_message("shared long context here")) + len(frame_header("Ans:"))
    assert first.cache_hit_tokens == 0
    assert first.tokens_encoded == known + len(e.generated_token_ids(m1))
    m2 = e.decode(call)
    second = e.last_stats
    assert e.generated_token_ids(m2) == e.generated_token_ids(m1)
    assert second.cache_hit_tokens == known - 1
    assert second.prefill_flops == 0
    assert second.tokens_encoded == 1 + len(e.generated_token_ids(m2))
    assert second.decode_flops < first.decode_flops


@pytest.mark.parametrize("mode,tol", [("f32", 1e-4), ("bf16", 2e-2)])
def test_matches_choreo_engine_on_a_chain(mode, tol):
    """On a chain with default offsets both engines see the same tokens at the same
    positions, so outputs agree (reference test_baseline.py:83-103)."""
    w = _weights(mode)
    base = BaselineEngine(w, record_logits=True)
    cho = P.Engine(w, record_logits=True)
    out = {}
    for e in (cho, base):
        sys_ = e.prefill(P.PrefillCall("You answer briefly."))
        a1 = e.decode(P.DecodeCall("A:", parents=[sys_], sampling=P.SamplingParams(max_tokens=6)))
        u = e.prefill(P.PrefillCall("more?", parents=[sys_, a1]) if e.kind == "choreo"
                      else P.PrefillCall("more?"))
        a2 = e.decode(P.DecodeCall("A:", parents=[sys_, a1, u],
                                   sampling=P.SamplingParams(max_tokens=6)))
        out[e.kind] = ((e.message_text(a1), e.message_text(a2)),
                       [np.stack(e.stats[i].logits[m]) for i, m in ((1, a1), (3, a2))])
    assert out["choreo"][0] == out["baseline"][0]
    for g, c in zip(out["baseline"][1], out["choreo"][1]):
        assert float(np.abs(g - c).max()) <= tol


def test_parallel_decode_is_sequential_lone_decodes():
    w = _small_weights()
    calls = [P.DecodeCall("L:", sampling=P.SamplingParams(max_tokens=4)),
             P.DecodeCall("R:", sampling=P.SamplingParams(max_tokens=4))]
    par = BaselineEngine(w)
    ids_par = par.decode_parallel(calls)
    seq = BaselineEngine(w)
    ids_seq = [seq.decode(c) for c in calls]
    assert ids_par == ids_seq
    for m in ids_par:
        assert par.message_text(m) == seq.message_text(m)


def test_error_contract():
    w = _small_weights()
    e = BaselineEngine(w)
    a = e.prefill(P.PrefillCall("ctx"))
    n_before = len(e.messages)
    with pytest.raises(P.EmptyHeaderError):
        e.decode(P.DecodeCall("", parents=[a]))
    with pytest.raises(P.UnknownMessageError):
        e.decode(P.DecodeCall("Q:", parents=[77]))
    with pytest.raises(P.WindowOverflowError):
        e.decode(P.DecodeCall("x" * w.config.context_window))
    with pytest.raises(P.InvalidCallError):
        e.decode_parallel([P.DecodeCall("A:")], force_tokens=[None, None])
    with pytest.raises(P.EmptyHeaderError):
        e.decode_parallel([P.DecodeCall("ok", parents=[a]), P.DecodeCall("")])
    assert len(e.messages) == n_before
    assert e.prefill(P.PrefillCall("next")) == a + 1
    with pytest.raises(P.InvalidCallError):
        e.generated_token_ids(a)
    with pytest.raises(P.UnknownMessageError):
        e.message_text(41)


def test_forced_decode_and_ttft():
    e = BaselineEngine(_small_weights())
    m = e.decode(P.DecodeCall("Say:"), force_tokens="ok")
    assert e.message_text(m) == "Say:ok"
    st = e.last_stats
    assert st.ttft[m] > 0 and st.wall >= st.ttft[m]


def test_tensor_core_paths_long_prompt_bf16():
    """Prompts long enough to route the re-encode through K4 (tcgen05) and trie hits
    that copy K/V pages: outputs equal the choreo engine's on the same chain."""
    cfg = P.ModelConfig(n_layers=2, n_heads=4, head_dim=64, ffn_dim=256, vocab_size=512,
                        context_window=2048)
    w = P.DeviceWeights.from_host(P.init_weights(cfg).rounded("bf16"), dtype=torch.bfloat16)
    text = " ".join(f"fact {i} is {i * 7 % 13}." for i in range(60))
    base = BaselineEngine(w, record_logits=True)
    cho = P.Engine(w, record_logits=True)
    res = {}
    for e in (cho, base):
        s = e.prefill(P.PrefillCall(text))
        m1 = e.decode(P.DecodeCall("Q1:", parents=[s], sampling=P.SamplingParams(max_tokens=8)))
        m2 = e.decode(P.DecodeCall("Q2:", parents=[s], sampling=P.SamplingParams(max_tokens=8)))
        res[e.kind] = [np.stack(e.stats[i].logits[m]) for i, m in ((1, m1), (2, m2))]
    # prompt + the shared header prefix [BOS_MSG, 'Q'] came from the trie
    assert base.stats[2].cache_hit_tokens == len(frame_message(text)) + 2
    for g, c in zip(res["baseline"], res["choreo"]):
        assert float(np.abs(g - c).max()) <= 2e-2


@pytest.mark.parametrize("prefix_cache", [True, False])
def test_storage_is_bounded_by_distinct_tokens(prefix_cache):
    """re-encoded prompts must not accumulate.  300 decodes that re-read the same
    ~200-token prompt (≈ 70K re-encoded tokens, past the old 64K store limit) neither raise
    CapacityError nor grow the pool: after the first, every decode's pages go back."""
    eng = BaselineEngine(_weights(), prefix_cache=prefix_cache)
    ids = [eng.prefill(P.PrefillCall(t * 20)) for t in ("abcd ", "efgh ")]
    first = None
    for i in range(300):
        m = eng.decode(P.DecodeCall("Q:", parents=ids, sampling=P.SamplingParams(max_tokens=4)))
        if first is None:
            first = eng.generated_token_ids(m)
            pages_after_first = eng.store.n_pages - len(eng.store._free)
        assert eng.generated_token_ids(m) == first
    assert eng.store.n_pages - len(eng.store._free) == (pages_after_first if prefix_cache else 0)
    assert eng.stats[-1].cache_hit_tokens == (len(frame_message("abcd " * 20)) * 2
                                              + len(frame_header("Q:")) - 1 if prefix_cache else 0)
