"""In-situ K5 v2 timeline: one 8B decode step (C3 round 2, 8 agents) with the -DCHOREO_TRACE
library (`python tools/chain_trace.py --build`).  Per stamp, the median over the 32 layer
launches of (median over CTAs of the stamp - the launch's first CTA start), in us."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_23049_b200 import _native as nat  # noqa: E402

nat.LIB_PATH = os.path.join(ROOT, "tools", "_trace", "_choreo_b200.so")
lib = nat.load()
import paper_2512_23049_b200 as P  # noqa: E402
from bench import workflow_inputs  # noqa: E402

WF = int(os.environ.get("WF", "1"))
cfg = P.PRESETS["llama-3.1-8b"]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536 * WF)
sched_calls = []
for wf in range(WF):
    sys_text, q, forced = workflow_inputs(wf, 8, 2)
    s = eng.prefill(P.PrefillCall(sys_text))
    qq = eng.prefill(P.PrefillCall(q))
    calls = [P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq],
                          sampling=P.SamplingParams(max_tokens=512)) for i in range(8)]
    prev = eng.decode_parallel(calls, force_tokens=[f[:300] for f in forced[0]])
    placed, cur = {}, 224
    for m in prev:
        placed[m] = cur
        cur += eng.message_token_count(m)
    sched_calls += [(P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq] + [m for j, m in enumerate(prev) if j != i],
                                  offsets=[0, 64] + [placed[m] for j, m in enumerate(prev) if j != i],
                                  new_offset=cur, sampling=P.SamplingParams(max_tokens=512)),
                     forced[1][i][:8]) for i in range(8)]
tr = torch.zeros(64 * 148 * 16, dtype=torch.int64, device="cuda")
lib.choreo_dv_set_trace.argtypes = [ctypes.c_void_p]
orig = eng._runner.forward
st = {"n": 0}


def fwd(plan):
    st["n"] += 1
    if st["n"] == 4:
        torch.cuda.synchronize()
        assert lib.choreo_dv_set_trace(tr.data_ptr()) == 0
        out = orig(plan)
        torch.cuda.synchronize()
        lib.choreo_dv_set_trace(None)
        return out
    return orig(plan)


eng._runner.forward = fwd
eng.decode_parallel([c for c, _ in sched_calls], force_tokens=[f for _, f in sched_calls])
t = tr.cpu().numpy().reshape(64, 148, 16).astype(np.float64)
n_l = int((t[:, :, 0] > 0).any(axis=1).sum())
if n_l == 0:
    sys.exit("no K5 v2 launch traced")
names = ["init", "pdl_wait", "prod 1st TMA", "loader unit0", "cons unit0", "cons page0",
         "cons last page", "merge_full", "merge unit0", "merge end", "-", "cons end",
         "loader items in", "loader Q in", "loader start"]
rows = []
for L in range(n_l):
    t0 = t[L, :, 0][t[L, :, 0] > 0].min()
    rel = np.where(t[L] > 0, (t[L] - t0) / 1e3, np.nan)
    rows.append([np.nanmedian(rel[:, i]) if np.any(~np.isnan(rel[:, i])) else np.nan
                 for i in range(15)] + [np.nanmax(rel[:, 11])])
rows = np.array(rows)
print(f"{n_l} launches, WF={WF}; medians over launches of per-CTA medians (us from launch start)")
for i, nm in enumerate(names):
    if nm != "-":
        print(f"  {nm:16s} {np.nanmedian(rows[:, i]):7.2f}")
print(f"  {'last CTA end':16s} {np.nanmedian(rows[:, 15]):7.2f}")
starts = [t[L, :, 0][t[L, :, 0] > 0].min() for L in range(n_l)]
print("  layer period (us):", np.round(np.median(np.diff(starts)) / 1e3, 2))
