mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_dist" -c 1 \
    -o gpurun_out/prof_dist -f python scripts/dbg2.py 100000 8 > gpurun_out/prof_dist.log 2>&1
tail -2 gpurun_out/prof_dist.log
