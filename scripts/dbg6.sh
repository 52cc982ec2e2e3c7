for i in 1 2 3 4 5 6 7 8; do timeout 120 python scripts/dbg2.py 100000 8 2>&1 | grep -E "ok|Error" | cut -c1-90; done
bash scripts/gpu_check.sh
