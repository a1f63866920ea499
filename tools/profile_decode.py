"""Profile window for ncu: build the 8B engine, run one warm debate round, then
bracket N decode steps of round 2 with cudaProfilerStart/Stop.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python tools/profile_decode.py --steps 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from bench import workflow_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--agents", type=int, default=8)
ap.add_argument("--model", default="llama-3.1-8b")
args = ap.parse_args()

cfg = P.PRESETS[args.model]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536)
sys_text, q, forced = workflow_inputs(0, args.agents, 2)
s = eng.prefill(P.PrefillCall(sys_text))
qq = eng.prefill(P.PrefillCall(q))
calls = [P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq], sampling=P.SamplingParams(max_tokens=512))
         for i in range(args.agents)]
prev = eng.decode_parallel(calls, force_tokens=[f[:300] for f in forced[0]])
base = 224
placed, cur = {}, base
for m in prev:
    placed[m] = cur
    cur += eng.message_token_count(m)
calls = []
for i in range(args.agents):
    others = [m for j, m in enumerate(prev) if j != i]
    calls.append(P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq] + others,
                              offsets=[0, 64] + [placed[m] for m in others], new_offset=cur,
                              sampling=P.SamplingParams(max_tokens=512)))


class Hook:
    n = 0


orig = eng._runner.forward


def fwd(plan):
    Hook.n += 1
    first = 1 if os.environ.get("PROFILE_HEADER") else 3  # 1: the header step itself
    if Hook.n == first:  # else skip the header step and the first decode step
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    out = orig(plan)
    if Hook.n == first - 1 + args.steps:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    return out


eng._runner.forward = fwd
eng.decode_parallel(calls, force_tokens=[f[:2 + args.steps] for f in forced[1]])
torch.cuda.synchronize()
print("profiled steps:", args.steps, "launches/step:", eng.kernel_launches)
