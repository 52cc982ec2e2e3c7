# Full GPU suite (compute-sanitizer is not available on the GPU pool this round)
mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/pytest.log 2>&1; tail -4 gpurun_out/pytest.log
