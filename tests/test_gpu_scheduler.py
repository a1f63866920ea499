"""Cross-workflow batching on the B200: workflows merged by BatchScheduler into one
engine call per step produce what each produces alone (same tokens; logits within the
dtype tolerance), over C4-style layouts (reordered parent subsets, gaps, overlaps)."""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2512_23049_b200 as P  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import c4_workflow  # noqa: E402

pytestmark = pytest.mark.gpu

SMALL = dict(n_prefill=5, n_rounds=3, n_dec=3, pre_len=(20, 90), dec_len=(10, 40))


def _run(dw, seeds, merged: bool):
    out = {}
    if merged:
        eng = P.Engine(dw, record_logits=True)
        wfs = [c4_workflow(eng, P, s, **SMALL) for s in seeds]
        res = P.BatchScheduler(eng).run(wfs)
        engines = [eng] * len(seeds)
    else:
        res, engines = [], []
        for s in seeds:
            eng = P.Engine(dw, record_logits=True)
            res.append(P.BatchScheduler(eng).run([c4_workflow(eng, P, s, **SMALL)])[0])
            engines.append(eng)
    for s, ids, eng in zip(seeds, res, engines):
        logits = {}
        for st in eng.stats:
            if st.logits:
                logits.update(st.logits)
        out[s] = [(eng.generated_token_ids(m), np.stack(logits[m])) for m in ids]
    return out


@pytest.mark.parametrize("mode", ["bf16", "f32"])
def test_batched_workflows_match_lone_runs(mode):
    cfg = P.ModelConfig(n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, ffn_dim=256,
                        vocab_size=300, context_window=4096, rope_base=500000.0)
    ws = P.init_weights(cfg)
    if mode == "bf16":
        dw = P.DeviceWeights.from_host(ws.rounded("bf16"), dtype=torch.bfloat16)
    else:
        dw = P.DeviceWeights.from_host(ws, dtype=torch.float32)
    seeds = [11, 12, 13]
    a = _run(dw, seeds, merged=True)
    b = _run(dw, seeds, merged=False)
    tol = 2e-2 if mode == "bf16" else 1e-4
    for s in seeds:
        for (ta, la), (tb, lb) in zip(a[s], b[s], strict=True):
            assert ta == tb
            assert la.shape == lb.shape
            assert float(np.abs(la - lb).max()) <= tol
