mkdir -p gpurun_out
for g in 0 1; do for ip in 0 1 2; do echo "gather=$g inplace=$ip"; RAGB_GATHER=$g RAGB_INPLACE=$ip timeout 120 python scripts/dbg_codes.py 1029; done; done > gpurun_out/dbg_codes.txt 2>&1
cat gpurun_out/dbg_codes.txt
bash scripts/gpu_codes.sh
