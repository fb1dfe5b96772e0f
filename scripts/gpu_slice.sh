# K = S S^T from one digit copy (no reversed slices); column-slicer block order A/B
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_ozaki.py tests/test_gpu_configs.py tests/test_gpu_lowrank.py tests/test_gpu_tiles.py 2>&1 | tail -2
for r in 1 2; do
for cfg in "STGP_XX=0" "STGP_OZ_SLICE_JFAST=1"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), {k: round(v,2) for k,v in p.items() if k in ('W_trmm','g_omega_trmm','g_X_gemm','g_S_gemm','K_gemm_chol')})"
done
done
export PATH=/usr/local/cuda/bin:$PATH
for cfg in "STGP_XX=0" "STGP_OZ_SLICE_JFAST=1"; do
env $cfg timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:slice_cols --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python scripts/eval_launches.py vif 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{print "'"$cfg"'", $(NF-2), $(NF-1), $NF}'
done
