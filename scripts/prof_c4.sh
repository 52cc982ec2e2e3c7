# ncu captures of the top kernels at C4 (one GPU).
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_dist_rows_nn|k_merge_compact" -c 2 \
    -o gpurun_out/prof_c4 -f python scripts/dbg2.py 100000 0 > gpurun_out/prof_c4.log 2>&1
tail -5 gpurun_out/prof_c4.log
