# cross-covariance rows emitted as digits: bit-identity test, parity, A/B timing (VIF cfg4, FITC cfg5)
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_ozaki.py tests/test_gpu_configs.py tests/test_gpu_lowrank.py tests/test_gpu_general_nu.py 2>&1 | tail -3
for r in 1 2; do
for cfg in "STGP_FUSED_CROSS=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), d['nll'], {k: round(v,2) for k,v in p.items() if k in ('W_trmm','U_cross_cov','g_omega_trmm')})"
done
done
for cfg in "STGP_FUSED_CROSS=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc [$cfg]', round(d['ms_per_step'],1), d['nll'], {k: round(v,2) for k,v in p.items() if k in ('W_trmm','U_cross_cov')})"
done
