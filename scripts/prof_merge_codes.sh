# ncu --set full of the first two compaction launches at C4 (code mode)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge" -c 2 \
    -o gpurun_out/prof_merge -f python scripts/dbg2.py 100000 0 > gpurun_out/prof_merge.log 2>&1
tail -2 gpurun_out/prof_merge.log
