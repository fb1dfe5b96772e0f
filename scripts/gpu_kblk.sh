# K-blocked column-form digit layout: tests + A/B (VIF cfg4, FITC cfg5) + slicer launch times
export PATH=/usr/local/cuda/bin:$PATH
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x -s tests/test_gpu_ozaki.py 2>&1 | grep -E "ozaki cols|passed|failed" | tail -3
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_configs.py tests/test_gpu_lowrank.py tests/test_gpu_tiles.py 2>&1 | tail -2
for r in 1 2; do
for cfg in "STGP_OZ_KBLK=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), d['nll'], {k: round(v,2) for k,v in p.items() if k in ('g_S_gemm','K_gemm_chol')})"
done
done
for cfg in "STGP_OZ_KBLK=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc [$cfg]', round(d['ms_per_step'],1), d['nll'], {k: round(v,2) for k,v in p.items() if k in ('f_S_gemm','K_gemm_chol')})"
done
for cfg in "STGP_OZ_KBLK=0" "STGP_XX=0"; do
env $cfg timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:"slice_cols|ozaki_tc_kernel<7, 1, 4>" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python scripts/eval_launches.py vif 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{print "'"$cfg"'", $5, $(NF-2), $NF}' | cut -c1-150
done
