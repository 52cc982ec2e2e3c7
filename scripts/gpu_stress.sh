for i in 1 2 3 4 5 6 7 8 9 10; do timeout 120 python scripts/dbg2.py 100000 8 2>&1 | grep -E "ok|Error" | cut -c1-100; done
for i in 1 2 3 4; do timeout 300 python scripts/dbg2.py 100000 0 2>&1 | grep -E "ok|Error" | cut -c1-200; done
