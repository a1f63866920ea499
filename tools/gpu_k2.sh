timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -k "rerotate" 2>&1 | tail -2
timeout -s KILL 300 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tools')
import kernel_bench as kb, json; print(json.dumps(kb.k2_rerotate()))"
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:rerotate -s 2 -c 1 -o gpurun_out/k2_full -f python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tools')
import kernel_bench as kb; kb.k2_rerotate()" > gpurun_out/k2_ncu.log 2>&1; echo ncu rc=$?
