set -x
nvidia-smi -L
nproc; free -g | head -2
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python bench.py --steps 3 --warmup 2 > gpurun_out/bench.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/smoke.txt; tail -5 gpurun_out/bench.txt
