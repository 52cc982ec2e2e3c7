for i in 1 2 3 4; do
RAGB_BENCH_DEBUG=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/dbg_$i.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms']['total_ms'])"
grep step: gpurun_out/dbg_$i.err | tr '\n' ' '; echo
done
