# round-2 ncu full captures: K7 (qkv shape), K5 v2 (8 workflows), K8 chain (8B layer)
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:linear_skinny -s 5 -c 1 \
  -o gpurun_out/r2_k7_qkv_full -f python tools/k7_only.py > gpurun_out/r2_k7_ncu.log 2>&1; echo k7 rc=$?
WF=8 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn_v2 -s 3 -c 1 \
  -o gpurun_out/r2_k5v2_8wf_full -f python tools/k5v2_one.py > gpurun_out/r2_k5_ncu.log 2>&1; echo k5 rc=$?
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:chain_sm100 -s 4 -c 1 \
  -o gpurun_out/r2_k8_chain_full -f python tools/chain_bench.py --phases 15 --iters 2 > gpurun_out/r2_k8_ncu.log 2>&1; echo k8 rc=$?
ls -la gpurun_out/*.ncu-rep
