import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb
for wf in (1, 8):
    for ppi in ("1", "2", "3", "4", "8"):
        os.environ["K5_PPI"] = ppi
        r = kb.k5_decode(wf, tc=True)
        print(f"tc wf={wf} ppi={ppi} items={r['items']} us={r['us']} comb={r['combine_us']} frac={r['frac']}", flush=True)
