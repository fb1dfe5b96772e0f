# FITC S product with the phi column factor applied by the slicer (no W diag(phi) pass)
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_ozaki.py tests/test_gpu_configs.py tests/test_gpu_lowrank.py tests/test_gpu_general_nu.py tests/test_gpu_predict.py tests/test_gpu_fit.py 2>&1 | tail -2
for r in 1 2; do
  timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc', round(d['ms_per_step'],1), d['nll'], d['grad'][:3], {k: round(v,2) for k,v in p.items()})"
done
