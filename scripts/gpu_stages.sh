# tcgen05 pipeline depth: 4 stages (default build) vs as many as fit (<= 6) -- paper_2602_03609_b200/libstgp_b200_st6.so
STGP_LIB=paper_2602_03609_b200/libstgp_b200_st6.so timeout -s KILL 900 python -m pytest -q -x -s tests/test_gpu_ozaki.py 2>&1 | grep -E "ozaki|passed|failed" | tail -5
for r in 1 2; do
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_st6.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif $lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in p.items() if k in ('W_trmm','g_omega_trmm','g_X_gemm','g_S_gemm','K_gemm_chol')})"
done
done
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_st6.so; do
  STGP_LIB=$lib timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc $lib', round(d['ms_per_step'],1), {k: round(v,2) for k,v in p.items() if k in ('W_trmm','f_KW_gemm','f_S_gemm','K_gemm_chol')})"
done
