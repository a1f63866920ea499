mkdir -p gpurun_out
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_decode.csv python tools/profile_decode.py --steps 2 > gpurun_out/prof_decode.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_decode.csv > gpurun_out/launches_decode.txt 2>&1; head -12 gpurun_out/launches_decode.txt
PROFILE_HEADER=1 timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches_header.csv python tools/profile_decode.py --steps 1 > gpurun_out/prof_header.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_header.csv > gpurun_out/launches_header.txt 2>&1; head -16 gpurun_out/launches_header.txt
