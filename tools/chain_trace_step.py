"""In-situ K8 timeline: one 8B decode step (C3 round 2, 8 agents) through the engine with the
-DCHOREO_TRACE library (build it with `python tools/chain_trace.py --build`).  Prints, per
chain launch, its start / end (us from the step's first launch) and the gap to the previous
launch's end (where K5 v2 + combine run), plus per-phase first/last MMA medians."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_23049_b200 import _native as nat  # noqa: E402

nat.LIB_PATH = os.path.join(ROOT, "tools", "_trace", "_choreo_b200.so")
lib = nat.load()
import paper_2512_23049_b200 as P  # noqa: E402
from bench import workflow_inputs  # noqa: E402

cfg = P.PRESETS["llama-3.1-8b"]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536)
sys_text, q, forced = workflow_inputs(0, 8, 2)
s = eng.prefill(P.PrefillCall(sys_text))
qq = eng.prefill(P.PrefillCall(q))
calls = [P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq], sampling=P.SamplingParams(max_tokens=512))
         for i in range(8)]
prev = eng.decode_parallel(calls, force_tokens=[f[:300] for f in forced[0]])
placed, cur = {}, 224
for m in prev:
    placed[m] = cur
    cur += eng.message_token_count(m)
calls = []
for i in range(8):
    others = [m for j, m in enumerate(prev) if j != i]
    calls.append(P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq] + others,
                              offsets=[0, 64] + [placed[m] for m in others], new_offset=cur,
                              sampling=P.SamplingParams(max_tokens=512)))
tr = torch.zeros(64 * 148 * 48, dtype=torch.int64, device="cuda")
lib.choreo_chain_set_trace.argtypes = [ctypes.c_void_p]
orig = eng._runner.forward
state = {"n": 0}


def fwd(plan):
    state["n"] += 1
    if state["n"] == 4:  # a decode step in the middle of the round
        torch.cuda.synchronize()
        assert lib.choreo_chain_set_trace(tr.data_ptr()) == 0
        out = orig(plan)
        torch.cuda.synchronize()
        lib.choreo_chain_set_trace(None)
        return out
    return orig(plan)


eng._runner.forward = fwd
eng.decode_parallel(calls, force_tokens=[f[:8] for f in forced[1]])
t = tr.cpu().numpy().reshape(64, 148, 48).astype(np.float64)
n_l = int((t[:, :, 0] > 0).any(axis=1).sum())
t0 = t[0, :, 0][t[0, :, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
prev_end = None
tot_chain = 0.0
for L in range(n_l):
    st, en = np.nanmin(rel[L, :, 0]), np.nanmax(rel[L, :, 25])
    tot_chain += en - st
    ph = []
    for k, nm in enumerate(["o", "gu", "d", "qkv"]):
        a, b = rel[L, :, 3 + 6 * k], rel[L, :, 4 + 6 * k]
        if not np.all(np.isnan(a)):
            ph.append(f"{nm} {np.nanmedian(a):6.1f}-{np.nanmedian(b):6.1f}")
    gap = "" if prev_end is None else f"gap {st - prev_end:5.1f}"
    print(f"launch {L:2d}: {st:7.1f} -> {en:7.1f} ({en - st:5.1f} us) {gap}  " + "  ".join(ph))
    prev_end = en
print(f"chain time {tot_chain:.1f} us of {prev_end:.1f} us")
