# rows-form epilogue (batched TMEM reads, early release, exact int->double): tests + A/B vs previous build
mkdir -p gpurun_out/epi
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x -s tests/test_gpu_ozaki.py 2>&1 | grep -E "trmm ozaki|ozaki [0-9]|passed|failed" | tail -5
timeout -s KILL 1200 python -m pytest -q -x tests/test_gpu_configs.py tests/test_gpu_lowrank.py 2>&1 | tail -2
for r in 1 2; do
  for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
    STGP_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif $lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in p.items() if k in ('W_trmm','g_omega_trmm','g_X_gemm','g_S_gemm','K_gemm_chol')})"
  done
done
