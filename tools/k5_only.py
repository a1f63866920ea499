import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb
for wf in (1, 8):
    r = kb.k5_decode(wf)
    print(os.environ.get("CHOREO_ATTN_FLAGS", "3"), wf, r["us"], r["achieved"], r["frac"])
