"""K5 configuration sweep at the C3 round-2 shape: precision flags x pages-per-item x
in-kernel combine, 1 and 8 workflows.  Prints kernel us (+ separate combine us)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402

for wf in (1, 8):
    for flags in ("3", "0"):
        os.environ["CHOREO_ATTN_FLAGS"] = flags
        for comb in ("1", "0"):
            os.environ["K5_FUSED_COMBINE"] = comb
            for ppi in ("auto", "1", "2", "4", "8"):
                if ppi == "auto":
                    os.environ.pop("K5_PPI", None)
                else:
                    os.environ["K5_PPI"] = ppi
                try:
                    r = kb.k5_decode(wf)
                    print(f"wf={wf} flags={flags} fused_comb={comb} ppi={r['pages_per_item']} "
                          f"items={r['items']} us={r['us']} comb_us={r['combine_us']} "
                          f"total={r['us'] + r['combine_us']:.2f} frac={r['frac']}", flush=True)
                except Exception as e:  # noqa: BLE001
                    print(f"wf={wf} flags={flags} comb={comb} ppi={ppi} failed: {e}", flush=True)
