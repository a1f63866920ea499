# ncu full capture of K5 v2 at 8 workflows (longest-first unit deal) and at 1 workflow
mkdir -p gpurun_out
for wf in 8 1; do
WF=$wf timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn_v2 -s 3 -c 1 \
  -o gpurun_out/r2_k5v2_${wf}wf_lpt_full -f python tools/k5v2_one.py > gpurun_out/r2_k5_${wf}_ncu.log 2>&1; echo k5 $wf rc=$?
done
ls -la gpurun_out/*.ncu-rep
