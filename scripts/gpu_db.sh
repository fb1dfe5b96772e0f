# rows form with 32-row Y tiles and two TMEM accumulator sets (STGP_OZAKI_ROWS_BN=32): tests + A/B
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 600 python -m pytest -q -x -s tests/test_gpu_ozaki.py 2>&1 | grep -E "trmm ozaki|^ozaki|passed|failed" | tail -4
STGP_OZAKI_ROWS_BN=32 timeout -s KILL 600 python -m pytest -q -x -s tests/test_gpu_ozaki.py 2>&1 | grep -E "trmm ozaki|ozaki [0-9]|passed|failed|Error" | tail -6
STGP_OZAKI_ROWS_BN=32 timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_configs.py tests/test_gpu_lowrank.py tests/test_gpu_switches.py 2>&1 | tail -2
for r in 1 2; do
for cfg in "STGP_XX=0" "STGP_OZAKI_ROWS_BN=32"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), d['nll'], {k: round(v,2) for k,v in p.items() if k in ('W_trmm','g_omega_trmm','g_X_gemm')})"
done
done
