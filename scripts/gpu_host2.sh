for t in 16 15 8 4; do echo "threads $t"; RAGB_HOST_THREADS=$t python scripts/host_in_build.py 2>&1 | tail -1; done
echo "passive"; OMP_WAIT_POLICY=passive python scripts/host_in_build.py 2>&1 | tail -1
echo "active"; OMP_WAIT_POLICY=active python scripts/host_in_build.py 2>&1 | tail -1
