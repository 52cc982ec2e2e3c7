mkdir -p gpurun_out
# the torchrun launch of bench.py (2 ranks on one GPU here: exercises the sharded path, not its speed)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 2 --warmup 1 --config C2 --no-cpu-baseline > gpurun_out/bench_mp.log 2>&1; grep -v "OMP_NUM" gpurun_out/bench_mp.log | grep -B2 -A12 "Error\|error\|Traceback" | head -60; tail -2 gpurun_out/bench_mp.log
