# per-form cluster shapes of the tcgen05 kernel (CY): rows 2 vs 4, symmetric 2 vs 4
for r in 1 2; do
for cfg in "STGP_XX=0" "STGP_OZAKI_CLUSTER_ROWS=4" "STGP_OZAKI_CLUSTER_SYM=4"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), {k: round(v,2) for k,v in p.items() if k in ('W_trmm','g_omega_trmm','g_X_gemm','g_S_gemm','K_gemm_chol')})"
done
done
for cfg in "STGP_XX=0" "STGP_OZAKI_CLUSTER_ROWS=4" "STGP_OZAKI_CLUSTER_SYM=4"; do
  env $cfg timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc [$cfg]', round(d['ms_per_step'],1), {k: round(v,2) for k,v in p.items() if k in ('W_trmm','f_KW_gemm','f_S_gemm','K_gemm_chol','f_omega_trmm_upair')})"
done
