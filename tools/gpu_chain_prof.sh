mkdir -p gpurun_out
timeout 300 python tools/chain_bench.py --k7 2>&1 | tail -12
timeout 300 python tools/chain_bench.py --rows 72 2>&1 | tail -6
timeout 600 ncu --set full --import-source on --clock-control none -k regex:chain_sm100 -s 4 -c 1 -o gpurun_out/chain_full -f python tools/chain_bench.py --phases 15 --iters 2 > gpurun_out/chain_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/chain_ncu.log
