# VIF and FITC under the tcgen05 kernel's cluster shapes
for r in 1 2; do
for cfg in "STGP_XX=0" "STGP_OZAKI_CLUSTER_X=2" "STGP_OZAKI_CLUSTER=1 STGP_OZAKI_CLUSTER_X=2" "STGP_OZAKI_CLUSTER=4 STGP_OZAKI_CLUSTER_X=1"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), {k: p[k] for k in ('K_gemm_chol','g_S_gemm','g_X_gemm')}, round(d['roofline']['int8_tensor']['kernel_ms'],2))"
done
done
for cfg in "STGP_XX=0" "STGP_OZAKI_CLUSTER_X=2"; do
  env $cfg timeout -s KILL 900 python bench.py --workload fitc --steps 2 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc [$cfg]', round(d['ms_per_step'],1), {k: p[k] for k in ('f_KW_gemm','f_S_gemm','K_gemm_chol')})"
done
