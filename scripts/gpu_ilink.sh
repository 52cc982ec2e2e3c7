mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "intersection" --timeout 600 -p no:cacheprovider 2>&1 | tail -15
