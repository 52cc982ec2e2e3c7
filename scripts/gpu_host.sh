nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core|Socket|NUMA node\(s\)"
python scripts/save_c4_linkage.py
for t in 1 4 8 16; do echo "threads $t"; RAGB_HOST_THREADS=$t RAGB_TRACE=1 python scripts/host_bench.py 2>&1 | tail -8; done
