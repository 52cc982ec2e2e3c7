mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json | cut -c1-400; tail -3 gpurun_out/bench.err
