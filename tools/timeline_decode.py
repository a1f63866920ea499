"""In-situ kernel timeline of 8B decode steps (C3 round 2, 8 agents) from CUPTI (torch.profiler),
with programmatic-dependent-launch overlap intact (ncu serialises kernels, this does not).

python tools/timeline_decode.py [--steps 2]
Prints per kernel name: count, average duration (with PDL a kernel starts early and waits
in griddepcontrol.wait, so this over-counts), and the critical-path share: how far each
kernel moves the completion front (its end minus the latest end before it).
"""
import argparse
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from bench import workflow_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()

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
calls = [P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq] + [m for j, m in enumerate(prev) if j != i],
                      offsets=[0, 64] + [placed[m] for j, m in enumerate(prev) if j != i],
                      new_offset=cur, sampling=P.SamplingParams(max_tokens=512))
         for i in range(8)]
orig = eng._runner.forward
st = {"n": 0, "prof": None}


def fwd(plan):
    st["n"] += 1
    if st["n"] == 3:
        torch.cuda.synchronize()
        st["prof"] = profile(activities=[ProfilerActivity.CUDA])
        st["prof"].__enter__()
    out = orig(plan)
    if st["n"] == 2 + args.steps:
        torch.cuda.synchronize()
        st["prof"].__exit__(None, None, None)
    return out


eng._runner.forward = fwd
eng.decode_parallel(calls, force_tokens=[f[:4 + args.steps] for f in forced[1]])
torch.cuda.synchronize()
ev = [e for e in st["prof"].events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
kern = [e for e in ev if "Memcpy" not in e.name and "Memset" not in e.name]
dur, cnt, crit = defaultdict(float), defaultdict(int), defaultdict(float)
for i, e in enumerate(kern):
    nm = e.name.split("(")[0].replace("void ", "").replace("choreo::", "")[:48]
    dur[nm] += e.time_range.end - e.time_range.start
    cnt[nm] += 1
    if i > 0:  # how far this kernel moved the step's completion front
        crit[nm] += e.time_range.end - max(k.time_range.end for k in kern[max(0, i - 3):i])
span = kern[-1].time_range.end - kern[0].time_range.start
print(f"{args.steps} steps: {span:.1f} us from first kernel start to last kernel end "
      f"({span / args.steps:.1f} us/step), {len(kern)} kernels")
print(f"{'kernel':50s} {'n':>5s} {'avg us':>8s} {'end - prev end avg':>22s} {'share':>6s}")
for nm in sorted(dur, key=lambda k: -crit[k]):
    print(f"{nm:50s} {cnt[nm]:5d} {dur[nm] / cnt[nm]:8.2f} {crit[nm] / cnt[nm]:22.2f} "
          f"{100 * crit[nm] / span:5.1f}%")
