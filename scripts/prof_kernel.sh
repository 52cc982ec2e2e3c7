# usage: bash scripts/prof_kernel.sh <kernel regex> <out name> [skip] [dbg2 args...]
# one ncu --set full capture of one launch of the matching kernel in a C4-shaped build
mkdir -p gpurun_out
K=$1; OUT=$2; SKIP=${3:-0}; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c 1 \
    -o gpurun_out/$OUT -f python scripts/dbg2.py "$@" > gpurun_out/$OUT.log 2>&1
tail -3 gpurun_out/$OUT.log
