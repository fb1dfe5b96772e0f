# U and U-pair kernels with 4 pairs in flight per thread (bit-identical): tests + A/B
export PATH=/usr/local/cuda/bin:$PATH
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_lowrank.py tests/test_gpu_configs.py tests/test_gpu_switches.py 2>&1 | tail -2
for r in 1 2; do
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif $lib', round(d['ms_per_step'],2), d['nll'], d['grad'][:2], {k: round(v,2) for k,v in p.items() if k in ('U_cross_cov','g_upair_sigma')})"
done
done
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
STGP_LIB=$lib timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:"cross_cov|upair" --metrics gpu__time_duration.sum --csv \
  python scripts/eval_launches.py fitc 10000 110 2000 30 2>/dev/null | grep -E "gpu__time" | python -c "
import sys,csv
for row in csv.reader(sys.stdin): print('fitc', '$lib'[-12:], row[4][:30], row[-1])"
done
