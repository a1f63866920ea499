"""Kernel breakdown of the C3 header step (the 72-row first forward of each decode_parallel,
which sets TTFT) at 8B bf16, from CUPTI (torch.profiler).  Per kernel name: launches,
summed duration (PDL early starts included) and device critical-path time: end minus the
later of the latest earlier end and the kernel's own start, so host gaps the profiler's
overhead opens between launches are not charged to anyone (sum = device-busy union)."""
import os
import sys
import time
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from bench import run_debate, workflow_inputs  # noqa: E402

cfg = P.PRESETS["llama-3.1-8b"]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536)
orig = eng._runner.forward
state = {"n": 0, "prof": None, "host": []}


def fwd(plan):
    if plan.n_rows <= 8:
        return orig(plan)
    state["n"] += 1
    torch.cuda.synchronize()
    if state["n"] == 3:  # third header step: warm caches, cuBLAS heuristics settled
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            t0 = time.perf_counter()
            out = orig(plan)
            state["host"].append((time.perf_counter() - t0) * 1e3)
            torch.cuda.synchronize()
        state["prof"] = prof
        return out
    t0 = time.perf_counter()
    out = orig(plan)
    state["host"].append((time.perf_counter() - t0) * 1e3)
    return out


eng._runner.forward = fwd
run_debate(eng, P, workflow_inputs(0, 8, 3), 8, 3)
evs = [e for e in state["prof"].events() if e.device_type == torch.autograd.DeviceType.CUDA
       and e.device_time_total > 0 and "Memcpy" not in e.name and "Memset" not in e.name
       and "sleep" not in e.name and "spin" not in e.name]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
t1 = max(e.time_range.end for e in evs)
agg = defaultdict(lambda: [0, 0.0, 0.0])
front = t0
for e in evs:
    a = agg[e.name[:64]]
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
    if e.time_range.end > front:
        a[2] += e.time_range.end - max(front, e.time_range.start)
        front = e.time_range.end
busy = sum(v[2] for v in agg.values())
print(f"header step: span {t1 - t0:.1f} us, device-busy {busy:.1f} us, {len(evs)} kernels, "
      f"host enqueue ms {['%.2f' % h for h in state['host']]}")
print(f"  {'kernel':64s} {'n':>5s} {'sum us':>9s} {'crit us':>9s}  share")
for k, (n, us, cr) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"  {k:64s} {n:5d} {us:9.1f} {cr:9.1f} {100 * cr / busy:5.1f}%")
