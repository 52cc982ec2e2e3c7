# bench + launch list + full ncu capture of the distance kernel (one GPU)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python scripts/dbg2.py 100000 0 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dist_tile" -c 1 \
    -o gpurun_out/prof_dist -f python scripts/dbg2.py 100000 8 > gpurun_out/prof_dist.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_rows|k_level_cliques|k_level_adj" -c 3 \
    -o gpurun_out/prof_link -f python scripts/dbg2.py 40000 0 > gpurun_out/prof_link.log 2>&1
ls -la gpurun_out
