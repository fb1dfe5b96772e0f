# VIF build with branch-free closure covariances: tests + A/B (prev = correctly rounded everywhere)
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_lowrank.py tests/test_gpu_configs.py tests/test_gpu_tiles.py tests/test_gpu_predict.py tests/test_gpu_switches.py tests/test_gpu_fit.py tests/test_gpu_laplace.py tests/test_gpu_general_nu.py 2>&1 | tail -2
for r in 1 2; do
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif $lib', round(d['ms_per_step'],2), d['nll'], d['grad'][:3], {k: round(v,2) for k,v in p.items() if k in ('rows',)})"
done
done
