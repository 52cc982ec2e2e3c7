# GPU parity tests + bench + C4 per-round linkage/host trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; grep -E "round (1|2|3|30) |ragb host|ok" gpurun_out/trace.txt
python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],d['e2e']['ms_per_step'])"
