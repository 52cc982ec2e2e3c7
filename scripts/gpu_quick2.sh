# GPU parity tests with in-place rounds auto / forced / disabled + C4 trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
RAGB_INPLACE=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu_inplace.txt
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace.txt 2>&1
timeout 900 python scripts/cmp_inplace.py > gpurun_out/dbg3.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/pytest_gpu_inplace.txt; cat gpurun_out/dbg3.txt
grep -E "round|ok" gpurun_out/trace.txt | cut -c1-120
