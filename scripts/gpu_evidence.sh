# Round evidence on one B200: bench line, ncu launch list of one C4 build,
# ncu --set full of the top kernels (distance, round-1 compaction, the h = 1.0
# level cliques), the C5 K sweep.  Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json | cut -c1-300
bash scripts/gpu_launches.sh
bash scripts/prof_kernel.sh k_dist_tile prof_dist 0 100000 0
bash scripts/prof_kernel.sh k_merge_gather prof_gather 0 100000 0
bash scripts/prof_kernel.sh k_level_cliques prof_cliques 29 100000 0
timeout 600 python scripts/k_sweep.py > gpurun_out/ks.log 2>&1
tail -3 gpurun_out/ks.log
