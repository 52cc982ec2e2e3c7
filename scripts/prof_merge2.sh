mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_merge_rows" -s 4 -c 1 \
    -o gpurun_out/prof_merge2 -f python scripts/dbg2.py 100000 0 > gpurun_out/prof_merge2.log 2>&1
tail -2 gpurun_out/prof_merge2.log
