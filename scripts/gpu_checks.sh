# GPU suite and the three benches against the bounds-checked build (make checks)
L=paper_2602_03609_b200/libstgp_b200_checks.so
O=profiles/r02/device_checks.log
mkdir -p gpurun_out
{
echo "# pytest -m gpu against the bounds-checked build (make checks; STGP_LIB=libstgp_b200_checks.so)"
date
STGP_LIB=$L timeout -s KILL 1800 python -m pytest tests -m gpu -q -rA 2>&1 | grep -v "^$"
echo "# benches (checked build): vecchia, vif, fitc"
STGP_LIB=$L timeout -s KILL 900 python bench.py --workload vecchia --steps 2 --warmup 3 2>/dev/null | tail -1 | cut -c1-400
STGP_LIB=$L timeout -s KILL 900 python bench.py --steps 2 --warmup 3 2>/dev/null | tail -1 | cut -c1-400
STGP_LIB=$L timeout -s KILL 900 python bench.py --workload fitc --steps 2 --warmup 3 2>/dev/null | tail -1 | cut -c1-400
} > gpurun_out/device_checks.log 2>&1
grep -E "passed|failed|error" gpurun_out/device_checks.log | tail -3
tail -3 gpurun_out/device_checks.log | cut -c1-200
