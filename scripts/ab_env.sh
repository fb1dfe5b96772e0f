# A/B environment settings on the VIF bench: ab_env.sh "ENV1" "ENV2" ...  (each a space-separated list of VAR=VAL)
for r in 1 2; do
for cfg in "$@"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('[$cfg]', round(d['ms_per_step'],2), {k: p[k] for k in ('K_gemm_chol','g_S_gemm','g_X_gemm','vprime','g_ef') if k in p})"
done
done
