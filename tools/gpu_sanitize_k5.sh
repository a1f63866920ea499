mkdir -p gpurun_out
timeout -s KILL 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_kernels.py tests/test_gpu_geometry.py -q -x -p no:cacheprovider -k "decode_v2 or k5v2" > gpurun_out/sanitize_racecheck_k5.log 2>&1
echo "rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_racecheck_k5.log | head -3; grep -m3 -A3 "Race reported" gpurun_out/sanitize_racecheck_k5.log
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_geometry.py -q -x -k "decode_v2 or k5v2" 2>&1 | tail -1
