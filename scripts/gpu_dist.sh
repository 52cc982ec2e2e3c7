mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sharded" --timeout 1200 -p no:cacheprovider 2>&1 | tail -25
