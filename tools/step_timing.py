"""Host vs device time per decode step (C3 round 2, 8B shape): is the step host-bound?

python tools/step_timing.py [--steps 64]   (env CHOREO_NATIVE_STEP / CHOREO_K7 toggle paths)
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from bench import workflow_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--agents", type=int, default=8)
args = ap.parse_args()

cfg = P.PRESETS["llama-3.1-8b"]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536)
sys_text, q, forced = workflow_inputs(0, args.agents, 2)
s = eng.prefill(P.PrefillCall(sys_text))
qq = eng.prefill(P.PrefillCall(q))
calls = [P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq], sampling=P.SamplingParams(max_tokens=512))
         for i in range(args.agents)]
prev = eng.decode_parallel(calls, force_tokens=[f[:300] for f in forced[0]])
placed, cur = {}, 224
for m in prev:
    placed[m] = cur
    cur += eng.message_token_count(m)
calls = []
for i in range(args.agents):
    others = [m for j, m in enumerate(prev) if j != i]
    calls.append(P.DecodeCall(f"Agent {i + 1}:", parents=[s, qq] + others,
                              offsets=[0, 64] + [placed[m] for m in others], new_offset=cur,
                              sampling=P.SamplingParams(max_tokens=512)))
host, evs = [], []
orig = eng._runner.forward


def fwd(plan):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    out = orig(plan)
    host.append(time.perf_counter() - t0)
    b.record()
    evs.append((a, b))
    return out


eng._runner.forward = fwd
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.decode_parallel(calls, force_tokens=[f[:args.steps] for f in forced[1]])
t_enq = time.perf_counter() - t0
torch.cuda.synchronize()
wall = time.perf_counter() - t0
dev = [a.elapsed_time(b) for a, b in evs[2:]]
gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(2, len(evs) - 1)]
print(f"native={os.environ.get('CHOREO_NATIVE_STEP', '1')} k7={os.environ.get('CHOREO_K7', '1')} "
      f"steps={len(evs)} host_fwd_ms={1e3 * statistics.median(host[2:]):.3f} "
      f"dev_step_ms={statistics.median(dev):.3f} gap_ms={statistics.median(gaps):.3f} "
      f"enqueue_s={t_enq:.3f} wall_s={wall:.3f} wall_per_step_ms={1e3 * wall / len(evs):.3f}")
