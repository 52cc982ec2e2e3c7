# per-launch durations at C4 (ncu, serialized): the launch list
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python scripts/dbg2.py 100000 0 > gpurun_out/launches.log 2>&1
tail -2 gpurun_out/launches.log
