# code-mode linkage: parity tests, bench, C4 trace
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -5 gpurun_out/pytest_gpu.txt
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace.txt 2>&1
grep -E "round (1|2|3|4|5|6|7|8|30) |ok" gpurun_out/trace.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json | cut -c1-900
