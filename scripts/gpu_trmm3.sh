# rotated item order for the triangle-cut TRMM; full GPU suite; benches
mkdir -p gpurun_out/trmm3
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 600 python -m pytest -q -x -s tests/test_gpu_ozaki.py -k trmm 2>&1 | grep -E "trmm ozaki|passed|failed" | tail -4
for r in 1 2; do
  timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/trmm3/bench_vif_$r.jsonl
  python -c "
import json; d=json.load(open('gpurun_out/trmm3/bench_vif_$r.jsonl')); p=d['roofline']['phase_ms']
print('vif', round(d['ms_per_step'],2), {k: round(v,2) for k,v in p.items() if 'trmm' in k or 'omega' in k})"
done
timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/trmm3/bench_fitc.jsonl
python -c "
import json; d=json.load(open('gpurun_out/trmm3/bench_fitc.jsonl')); p=d['roofline']['phase_ms']
print('fitc', round(d['ms_per_step'],1), {k: round(v,2) for k,v in p.items()})"
timeout -s KILL 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
