# round profile (code mode): bench line, ncu launch list, ncu --set full of the distance + compaction kernels
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json | cut -c1-600
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python scripts/dbg2.py 100000 0 > gpurun_out/launches.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_dist_tile|k_merge_gather" \
    -o gpurun_out/prof_full -f python scripts/dbg2.py 100000 0 > gpurun_out/prof_full.log 2>&1
tail -2 gpurun_out/prof_full.log
