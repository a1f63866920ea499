mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/chain_tests.log 2>&1; echo "chain rc=$?"; tail -30 gpurun_out/chain_tests.log
for c in 0 1; do CHOREO_CHAIN=$c timeout 300 python tools/step_timing.py --steps 64 2>&1 | tail -1; done
for c in 0 1; do CHOREO_CHAIN=$c timeout 300 python tools/header_timing.py 2>&1 | tail -2; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/pytest_gpu.log
