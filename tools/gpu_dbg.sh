timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_geometry.py -q -k "linear or k7 or gate_up" -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 300 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -3
timeout -s KILL 120 python tools/chain_bench.py --rows 72 --k7 --phases 2 2>&1 | tail -5
timeout -s KILL 120 python tools/header_timing.py 2>&1 | tail -2
