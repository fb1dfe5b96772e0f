# GEMV partials with all rows of a column in one pass: full GPU suite + A/B (VIF, FITC) + kernel times
export PATH=/usr/local/cuda/bin:$PATH
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif $lib', round(d['ms_per_step'],2), d['nll'], {k: round(v,2) for k,v in p.items() if k in ('g_nll','g_t_z')})"
  STGP_LIB=$lib timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('fitc $lib', round(d['ms_per_step'],1), d['nll'])"
done
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
STGP_LIB=$lib timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:gemv_n --metrics gpu__time_duration.sum --csv \
  python scripts/eval_launches.py vif 2>/dev/null | grep -E "gpu__time" | python -c "
import sys,csv
for row in csv.reader(sys.stdin): print('$lib'[-12:], row[4][:30], row[-1])"
done
