mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dist_tile" -c 1 \
    -o gpurun_out/prof_dist -f python scripts/dbg2.py 100000 0 > gpurun_out/prof_dist.log 2>&1
tail -1 gpurun_out/prof_dist.log
