# ncu capture of the round-1 and round-2 k_merge_rows launches at C4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_rows" --launch-count 2 \
    -o gpurun_out/prof_merge3 -f python scripts/dbg2.py 100000 0 > gpurun_out/prof_merge3.log 2>&1
tail -3 gpurun_out/prof_merge3.log
