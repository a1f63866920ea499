# K5 v2 unit schedule A/B: longest-first snake deal (K3 item_order) vs round-robin one-wave items
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "decode_v2 or assemble" 2>&1 | tail -2
for o in 1 0; do
  K5_ORDER=$o timeout 300 python -c "
import sys; sys.path.insert(0, 'tools')
import kernel_bench as kb, json
for wf in (1, 8):
    r = kb.k5_decode(wf); print('K5_ORDER=$o', wf, r['us'], r['frac'], r['items'], r['pages_per_item'])
"
done
for o in 1 0 1 0; do CHOREO_V2_LPT=$o timeout 300 python tools/step_timing.py --steps 200 2>&1 | tail -2; done
