# Profile bundle: decode-step launch list + ncu full captures of K5 v2 (decode) and K4 (prefill).
set -x
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches_decode.csv python tools/profile_decode.py --steps 2 > gpurun_out/prof_decode.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_decode.csv > gpurun_out/launches_decode.txt 2>&1
cat gpurun_out/launches_decode.txt | head -30
WF=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_v2 -s 3 -c 1 \
  -o gpurun_out/k5v2_full -f python tools/k5v2_one.py > gpurun_out/k5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_prefill -s 1 -c 1 \
  -o gpurun_out/k4_full -f python tools/k4_prof.py > gpurun_out/k4_ncu.log 2>&1
ls -la gpurun_out
