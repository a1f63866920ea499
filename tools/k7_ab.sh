# decode-step A/B of K7 ring sizes (CHOREO_K7_SMEM_KB caps the ring's shared memory)
for i in 1 2; do
for cfg in "X=0" "CHOREO_K7_SMEM_KB=148" "CHOREO_K7_SMEM_KB=130" "CHOREO_K7_SMEM_KB=112" "CHOREO_K7_SMEM_KB=96"; do
  echo -n "$cfg: "; env $cfg python tools/step_timing.py --steps 48 | tail -1 | grep -o "dev_step_ms=[0-9.]*"
done; done
