for cfg in "1 1 1" "1 1 0" "0 0 0"; do set -- $cfg
CHOREO_NATIVE_STEP=$1 CHOREO_K7=$2 CHOREO_PDL=$3 timeout 600 python tools/step_timing.py --steps 96 2>&1 | tail -1
done
