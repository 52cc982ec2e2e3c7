# C4 per-round linkage trace only
mkdir -p gpurun_out
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace.txt 2>&1
RAGB_TRACE=1 timeout 600 python scripts/dbg2.py 100000 0 > gpurun_out/trace2.txt 2>&1
grep -E "round (1|2|3|29|30|31|35) |ok" gpurun_out/trace2.txt
