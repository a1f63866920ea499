"""Host vs device time of the header step (first forward of a decode_parallel) at 8B."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
if os.environ.get("BLAS"):
    torch.backends.cuda.preferred_blas_library(os.environ["BLAS"])
import paper_2512_23049_b200 as P
from bench import workflow_inputs, run_debate

cfg = P.PRESETS["llama-3.1-8b"]
w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16)
eng = P.Engine(w, capacity=65536)
rec = []
orig = eng._runner.forward
def fwd(plan):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); a.record()
    out = orig(plan)
    h = time.perf_counter() - t0
    b.record(); torch.cuda.synchronize()
    rec.append((plan.n_rows, h * 1e3, a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    return out
eng._runner.forward = fwd
run_debate(eng, P, workflow_inputs(0, 8, 3), 8, 3)
for r in rec:
    if r[0] > 8:
        print("rows=%d host_ms=%.2f dev_ms=%.2f wall_ms=%.2f" % r)
