set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_active.avg,sm__cycles_active.max --clock-control none -k regex:linear_skinny --csv --log-file gpurun_out/k7_launches.csv python tools/k7_only.py > gpurun_out/k7_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:linear_skinny -s 5 -c 1 -o gpurun_out/k7_full python tools/k7_only.py > gpurun_out/k7_n.log 2>&1
tail -3 gpurun_out/k7_n.log
