# repeat a pytest selection N times per config; print failures
N=${N:-10}
for cfg in "CHOREO_PDL=1" "CHOREO_PDL=0"; do
  fails=0
  for i in $(seq $N); do
    env $cfg timeout 120 python -m pytest tests/test_gpu_scheduler.py tests/test_gpu_engine.py -q -x -p no:randomly > /tmp/st.log 2>&1 || { fails=$((fails+1)); grep -E "^E |FAILED" /tmp/st.log | head -3; }
  done
  echo "$cfg fails=$fails/$N"
done
