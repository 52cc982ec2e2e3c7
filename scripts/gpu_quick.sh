# GPU parity tests + C4 per-round trace (fast iteration)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace.txt 2>&1
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace2.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; grep -E "round (1|2|3|30) |ok" gpurun_out/trace2.txt
