# Round re-entry check: GPU parity tests, smoke, bench line, C4 per-round linkage trace
mkdir -p gpurun_out
nvidia-smi -L; nproc; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/smoke.txt; tail -1 gpurun_out/bench.json
