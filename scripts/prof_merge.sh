mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_merge_compact|k_round_prep" -c 2 \
    -o gpurun_out/prof_merge -f python scripts/dbg2.py 40000 0 > gpurun_out/prof_merge.log 2>&1
tail -2 gpurun_out/prof_merge.log
