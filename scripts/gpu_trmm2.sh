# triangle-cut Ozaki TRMM: unit tests, accuracy at cfg4 / cfg5 vs the all-DMMA path, A/B timing
mkdir -p gpurun_out/trmm2
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x -s tests/test_gpu_ozaki.py 2>&1 | grep -E "trmm|passed|failed|Error" | tail -8
P=scripts/ozaki_accuracy_probe.py
for k in vif fitc; do
  STGP_OZAKI=0 timeout -s KILL 600 python $P 10000 110 $k > gpurun_out/trmm2/acc_${k}_dmma.json
  timeout -s KILL 600 python $P 10000 110 $k > gpurun_out/trmm2/acc_${k}_s7.json
done
timeout -s KILL 1500 python -m pytest -q -x tests/test_gpu_configs.py tests/test_gpu_lowrank.py tests/test_gpu_tiles.py tests/test_gpu_predict.py tests/test_gpu_shards.py 2>&1 | tail -3
for r in 1 2; do
for cfg in "STGP_OZAKI_TRMM=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), {k: round(v,2) for k,v in p.items() if 'trmm' in k or k.startswith('W') or 'omega' in k})"
done
done
for cfg in "STGP_XX=0"; do
  env $cfg timeout -s KILL 900 python bench.py --workload fitc --steps 2 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('fitc [$cfg]', round(d['ms_per_step'],1), {k: round(v,2) for k,v in p.items()})"
done
