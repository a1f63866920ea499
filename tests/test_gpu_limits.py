"""K3 planning limits on the B200.

assemble.cu plans a step in one CTA with fixed tables (1024 calls, 4096 (parent, call)
pairs page-centric).  Steps beyond those limits are cut on the host before any launch
(model.split_plan); these tests drive the engine past each limit and compare with the
oracle, with CHOREO_CHECK_ASSEMBLY on so any K3 overflow flag raises.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import choreo_oracle as O  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = {
    # the reference's tiny model in f32 (SIMT split-KV path)
    "tiny_f32": (O.TINY, "f32", torch.float32, 1e-4),
    # hd 64 GQA in bf16 (K5 v2 page-centric decode, K7 projections)
    "gqa64_bf16": (O.Shape(n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, ffn_dim=128,
                           vocab_size=300, context_window=2048, rope_base=500000.0),
                   "bf16", torch.bfloat16, 2e-2),
}


def _pair(name, capacity=1 << 16):
    shape, rk, dt, tol = SHAPES[name]
    cfg = P.ModelConfig(**{k: getattr(shape, k) for k in shape.__dataclass_fields__})
    ref = O.Oracle(O.round_weights(O.init_weights(shape), rk), shape, capacity=capacity,
                   record_logits=True)
    ws = P.init_weights(cfg)
    ws = ws.rounded("bf16") if rk == "bf16" else ws
    eng = P.Engine(P.DeviceWeights.from_host(ws, dtype=dt), capacity=capacity,
                   record_logits=True)
    eng._runner.check_assembly = True
    return ref, eng, tol


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_parallel_decode_beyond_k3_pair_limit(name):
    """64 agents x 70 shared parents = 4480 (parent, call) pairs > 4096: the step is cut
    into sub-steps; tokens and logits equal the oracle's, physical layout bit-exact."""
    ref, eng, tol = _pair(name)
    texts = [f"m{i}" for i in range(70)]
    for t in texts:
        ref.prefill({"message": t})
    ids = eng.prefill_parallel([P.PrefillCall(t) for t in texts])
    assert ids == list(range(70))
    parents = list(range(70))[::-1]  # reordered, default offsets (shared => one layout)
    sp_o, sp_p = O.Sampling(max_tokens=3), P.SamplingParams(max_tokens=3)
    ref_ids = ref.decode_batch([{"header": f"A{i}:", "parents": parents, "sampling": sp_o}
                                for i in range(64)])
    got = eng.decode_parallel([P.DecodeCall(f"A{i}:", parents=parents, sampling=sp_p)
                               for i in range(64)],
                              force_tokens=[ref.generated(m) for m in ref_ids])
    assert got == ref_ids
    worst = 0.0
    for m in got:
        a = np.stack(eng.stats[-1].logits[m])
        b = np.stack(ref.stats[-1].logits[m])
        assert a.shape == b.shape
        worst = max(worst, float(np.abs(a - b).max()))
    assert worst <= tol, worst
    n = eng.cache.token_count
    assert eng.cache.msg_ids[:n].tolist() == ref.store.mid[:n].tolist()
    assert eng.cache.positions[:n].tolist() == ref.store.pos[:n].tolist()


def test_prefill_parallel_beyond_k3_call_limit():
    """1030 calls in one prefill_parallel (> 1024 K3 call slots): cut into two sub-steps;
    the cached K/V equal the oracle's and every message is contiguous in call order."""
    ref, eng, tol = _pair("tiny_f32")
    texts = [f"n{i:04d}" for i in range(1030)]
    eng.prefill(P.PrefillCall("root message"))
    ref.prefill({"message": "root message"})
    ids = eng.prefill_parallel([P.PrefillCall(t, parents=[0]) for t in texts])
    ref_ids = ref.prefill_batch([{"message": t, "parents": [0]} for t in texts])
    assert ids == ref_ids
    n = eng.cache.token_count
    assert n == ref.store.n
    assert eng.cache.msg_ids[:n].tolist() == ref.store.mid[:n].tolist()
    assert eng.cache.positions[:n].tolist() == ref.store.pos[:n].tolist()
    np.testing.assert_allclose(eng.cache.keys, ref.store.K[:, :n], rtol=0, atol=1e-4)
    np.testing.assert_allclose(eng.cache.values, ref.store.V[:, :n], rtol=0, atol=1e-4)
    # and a decode over the last of them still matches
    m = eng.decode(P.DecodeCall("Q:", parents=[ids[-1], 0], sampling=P.SamplingParams(max_tokens=4)))
    mr = ref.decode({"header": "Q:", "parents": [ref_ids[-1], 0],
                     "sampling": O.Sampling(max_tokens=4)})
    assert eng.generated_token_ids(m) == ref.generated(mr)


def test_single_call_with_more_parents_than_pair_limit():
    """One decode over 4200 parents (more than K3's 4096 page-centric pairs on its own)
    runs with per-call page lists; tokens and logits equal the oracle's."""
    ref, eng, tol = _pair("tiny_f32", capacity=1 << 15)
    # two-token messages (BOS, EOS framing of the empty string is not allowed: use 1 char)
    cfg_w = eng.config.context_window
    n_par = 4200
    assert 3 * n_par > cfg_w  # the window cannot hold them at distinct offsets:
    # overlap them (every parent at offset 0 is legal, reference test_engine.py:73-82)
    texts = [chr(97 + i % 26) for i in range(n_par)]
    ids = eng.prefill_parallel([P.PrefillCall(t) for t in texts])
    ref.prefill_batch([{"message": t} for t in texts])
    sp_o, sp_p = O.Sampling(max_tokens=3), P.SamplingParams(max_tokens=3)
    offs = [0] * n_par
    mr = ref.decode({"header": "Z:", "parents": ids, "offsets": offs, "sampling": sp_o})
    m = eng.decode(P.DecodeCall("Z:", parents=ids, offsets=offs, sampling=sp_p))
    assert eng.generated_token_ids(m) == ref.generated(mr)
    a = np.stack(eng.last_stats.logits[m])
    b = np.stack(ref.stats[-1].logits[mr])
    assert float(np.abs(a - b).max()) <= tol


def test_capacity_failure_mid_step_keeps_the_prefix_like_the_reference():
    """A parallel decode step that runs out of capacity appends the messages before the
    one that does not fit, then raises CapacityError (reference engine.py:430-433 +
    cache.py:114-117) -- no slot is left reserved without its K/V."""
    shape = O.TINY
    cap = 5 + 4 + 2 * 2 + 1
    ref = O.Oracle(O.round_weights(O.init_weights(shape), "f32"), shape, capacity=cap)
    eng = P.Engine(P.DeviceWeights.from_host(P.init_weights(P.DEFAULT_CONFIG),
                                             dtype=torch.float32), capacity=cap)
    force = [[65, 66, 67, 68], [70, 71, 72, 73]]
    ref.prefill({"message": "abc"})
    a = eng.prefill(P.PrefillCall("abc"))
    with pytest.raises(O.OracleError):
        ref.decode_batch([{"header": "A", "parents": [0]}, {"header": "B", "parents": [0]}],
                         force)
    with pytest.raises(P.CapacityError):
        eng.decode_parallel([P.DecodeCall("A", parents=[a]), P.DecodeCall("B", parents=[a])],
                            force_tokens=force)
    n = eng.cache.token_count
    assert n == ref.store.n == cap
    assert eng.cache.msg_ids[:n].tolist() == ref.store.mid[:n].tolist()
    assert eng.cache.token_ids[:n].tolist() == ref.store.tok[:n].tolist()
    np.testing.assert_allclose(eng.cache.keys, ref.store.K[:, :n], rtol=0, atol=1e-4)
    np.testing.assert_allclose(eng.cache.values, ref.store.V[:, :n], rtol=0, atol=1e-4)
