"""Where does the host time of a decode step go?  (C3 round 2, 8B, teacher-forced)

cProfile over 32 decode steps of one decode_parallel, plus wall time of the native
executor call alone (choreo_decode_layers) per step.
python tools/host_profile.py
"""
import cProfile
import os
import pstats
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from paper_2512_23049_b200 import _native as nat  # noqa: E402
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
dl_times = []
orig_dl = nat.decode_layers


SYNC = os.environ.get("SYNC_BEFORE", "0") == "1"


def timed_dl(*a):
    if SYNC:  # GPU idle at the call: the pure host cost of the launches (no backpressure)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig_dl(*a)
    dl_times.append(time.perf_counter() - t0)
    return r


nat.decode_layers = timed_dl
import paper_2512_23049_b200.model as M  # noqa: E402
M.nat.decode_layers = timed_dl
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
eng.decode_parallel(calls, force_tokens=[f[:32] for f in forced[1]])
pr.disable()
torch.cuda.synchronize()
print(f"decode_layers host ms per call: median {1e3 * statistics.median(dl_times):.3f} "
      f"n={len(dl_times)}")
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
st.sort_stats("tottime").print_stats(25)
