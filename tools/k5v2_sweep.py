import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb
for wf in (1, 8):
    for ppi in ("auto", "1", "2", "4", "8", "16"):
        if ppi == "auto":
            os.environ.pop("K5_PPI", None)
        else:
            os.environ["K5_PPI"] = ppi
        r = kb.k5_decode(wf, v2=True)
        print(f"v2 wf={wf} ppi={r['pages_per_item']} items={r['items']} us={r['us']} comb={r['combine_us']} "
              f"GB/s={r['achieved']} frac={r['frac']}", flush=True)
