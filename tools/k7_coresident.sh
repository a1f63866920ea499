# Decode-step time (C3 round 2, 8B) vs the K7 ring's shared memory: a ring small enough
# for two K7 CTAs per SM lets the next GEMM stream its weights under the current one.
mkdir -p gpurun_out
for cfg in "" "CHOREO_K7_SMEM_KB=112" "CHOREO_K7_SMEM_KB=100" "CHOREO_K7_SMEM_KB=100 CHOREO_K7_KSUB=1" "CHOREO_K7_SMEM_KB=80" "CHOREO_K7_SMEM_KB=80 CHOREO_K7_KSUB=1" ""; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/step_timing.py --steps 64 2>&1 | tail -1
done
