# The torchrun (N > 1) path of bench.py, both arms, with 2 ranks sharing the one GPU (gloo).
set -x
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 1 --warmup 1 --no-cpu-baseline --no-c2 > gpurun_out/bench_2r.log 2>&1
echo "ours rc=$?"; grep '^{' gpurun_out/bench_2r.log | cut -c1-400; tail -3 gpurun_out/bench_2r.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_2r_ref.log 2>&1
echo "ref rc=$?"; grep '^{' gpurun_out/bench_2r_ref.log | cut -c1-300
