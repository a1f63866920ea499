# K5 v2 change check: kernel + geometry + engine tests, microbench (1 / 8 workflows), in-situ step
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_geometry.py tests/test_gpu_engine.py -q -x 2>&1 | tail -2
timeout 300 python -c "
import sys; sys.path.insert(0, 'tools')
import kernel_bench as kb
for wf in (1, 8, 1, 8):
    r = kb.k5_decode(wf); print('K5', wf, r['us'], r['frac'], r['items'], r['pages_per_item'])
"
for i in 1 2; do timeout 300 python tools/step_timing.py --steps 200 2>&1 | tail -1; done
timeout 300 python tools/dv_trace_step.py 2>&1 | tail -18
