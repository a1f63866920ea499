# compute-sanitizer racecheck / synccheck / memcheck over the mbarrier / TMA / tcgen05 kernels
mkdir -p gpurun_out
export CHOREO_PDL=1
for tool in racecheck synccheck memcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --target-processes all \
    python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider \
    -k "prefill_tcgen05 or decode_v2 or (linear_skinny and 4096-4096 and (8-True or 72-True)) or gate_up_silu or k7_pieces or rerotate" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Hazard|Error" gpurun_out/sanitize_$tool.log | head -5
done
timeout -s KILL 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_chain.py -q -x -p no:cacheprovider -k "8-True-1024" > gpurun_out/sanitize_chain_racecheck.log 2>&1
echo "chain racecheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_chain_racecheck.log | head -3
