"""Host side of the C3 header step (8B bf16): where the host spends the step and how long the
GPU waits for its first kernel.  Events: forward entry -> just before choreo_assemble (host
preparation the GPU idles through) -> forward return -> device done; plus a cProfile of one
header forward (top functions by cumulative time)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from paper_2512_23049_b200 import _native as nat  # noqa: E402
from bench import run_debate, workflow_inputs  # noqa: E402

cfg = P.PRESETS["llama-3.1-8b"]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536)
orig = eng._runner.forward
orig_asm = nat.assemble_ex
rec, marks, state = [], {}, {"n": 0}


def asm(*a):
    if "pre" not in marks:
        marks["pre_t"] = time.perf_counter()
        marks["pre"] = torch.cuda.Event(enable_timing=True)
        marks["pre"].record()
    return orig_asm(*a)


nat.assemble_ex = asm


def fwd(plan):
    if plan.n_rows <= 8:
        return orig(plan)
    state["n"] += 1
    torch.cuda.synchronize()
    marks.clear()
    e0, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    t0 = time.perf_counter()
    e0.record()
    if state["n"] == 4:
        pr = cProfile.Profile()
        pr.enable()
        out = orig(plan)
        pr.disable()
        state["prof"] = pr
    else:
        out = orig(plan)
    t2 = time.perf_counter()
    e2.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    rec.append((plan.n_rows, (marks["pre_t"] - t0) * 1e3, e0.elapsed_time(marks["pre"]),
                (t2 - t0) * 1e3, e0.elapsed_time(e2), (t3 - t0) * 1e3))
    return out


eng._runner.forward = fwd
run_debate(eng, P, workflow_inputs(0, 8, 3), 8, 3)
for r in rec:
    print("rows=%d host_prep_ms=%.3f gpu_idle_to_first_ms=%.3f host_fwd_ms=%.2f "
          "dev_at_return_ms=%.2f wall_ms=%.2f" % r)
pstats.Stats(state["prof"]).sort_stats("cumulative").print_stats(22)
