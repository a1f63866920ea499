"""Device temperature / top-p sampling (K6b) pinned to the reference's own sampled runs.

Goldens: tests/golden/ref_sampling_* (make_golden.py `sampling`): the reference Engine
(engine.py:374-392) sampling every free decode of five fixture scripts under three
(temperature, top_p, seed) settings, with the f64 logits of every selection.
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import choreo_oracle as O  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from paper_2512_23049_b200 import _native as nat  # noqa: E402
from paper_2512_23049_b200.script import run_script  # noqa: E402

from .test_sampling_pins import LOGITS, RUNS, selections  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_k6b_reproduces_reference_sampled_tokens():
    """Every recorded selection through K6b (one launch for all 884 rows): the token equals
    the oracle's nucleus() on the same (f32) logits and the reference's sampled token."""
    rows, params, keys, want, mids = [], [], [], [], []
    for key in sorted(RUNS):
        sp = RUNS[key]["sampling"]
        for mid, k, row, tok in selections(key):
            rows.append(row)
            params.append((sp["temperature"], sp["top_p"]))
            keys.append((0, sp["seed"], mid, k))
            want.append(tok)
            mids.append((key, mid, k))
    lg32 = np.stack(rows).astype(np.float32)
    n, V = lg32.shape
    dev = torch.from_numpy(lg32).cuda()
    pd = torch.from_numpy(np.asarray(params, np.float64)).cuda()
    kd = torch.from_numpy(np.asarray(keys, np.uint64).view(np.int64)).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.select_nucleus(dev.data_ptr(), n, V, V, pd.data_ptr(), kd.data_ptr(), out.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
    got = out.cpu().tolist()
    gen = O.sampler_mask(V)
    for i in range(n):
        sp = O.Sampling(mode="temperature", temperature=params[i][0], top_p=params[i][1],
                        seed=keys[i][1])
        assert got[i] == O.nucleus(lg32[i].astype(np.float64), gen, sp, 0, keys[i][2],
                                   keys[i][3]), mids[i]
        if want[i] is not None:
            assert got[i] == want[i], mids[i]


@pytest.mark.parametrize("key", sorted(RUNS))
def test_engine_free_run_sampling_matches_reference(key):
    """The f32 engine with device sampling replays the reference's sampled runs: the same
    tokens, texts and token counts for every message; logits within 1e-4."""
    run = RUNS[key]
    script = json.load(open(os.path.join(GOLD, "scripts", f"{run['script']}.json")))
    script["sampling"] = run["sampling"]
    eng = P.Engine(P.DeviceWeights.from_host(P.init_weights(P.DEFAULT_CONFIG),
                                             dtype=torch.float32), record_logits=True)
    assert eng.device_sampling
    trace = run_script(eng, script)
    worst = 0.0
    for got, want in zip(trace.steps, run["steps"], strict=True):
        for gm, wm in zip(got.messages, want["messages"], strict=True):
            assert (gm.message_id, gm.generated, gm.text, gm.token_count) == \
                (wm["id"], wm["generated"], wm["text"], wm["tokens"])
        for name, rows in (got.logits or {}).items():
            worst = max(worst, float(np.abs(np.stack(rows) - LOGITS[f"{key}/{name}"]).max()))
    assert worst <= 1e-4
