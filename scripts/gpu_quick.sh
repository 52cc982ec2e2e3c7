# Quick A/B loop for linkage kernels on one B200: the parity cases that reach
# the compaction kernels, then one traced C4 build (per-round times).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "full_size_paths or C2_full or round_strategy or code_mode or multiturn or intersection or variable or code_window or ragged or deterministic" 2>&1 | tail -25
timeout 300 python scripts/trace_build.py C4 "$@" 2> gpurun_out/trace.err | tail -1 | cut -c1-300
grep -o 'round [0-9]* M=[0-9]* .*merge=[0-9.]*ms' gpurun_out/trace.err | head -10
