# U-pair gradient with the inducing point fixed per thread: tests + A/B
export PATH=/usr/local/cuda/bin:$PATH
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_lowrank.py tests/test_gpu_configs.py tests/test_gpu_many_times.py tests/test_gpu_shards.py tests/test_gpu_ozaki.py 2>&1 | tail -2
for r in 1 2; do
for cfg in "STGP_UPAIR_ZFIXED=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif [$cfg]', round(d['ms_per_step'],2), d['nll'], d['grad'][:3], {k: round(v,2) for k,v in p.items() if k in ('g_upair_sigma',)})"
done
done
for cfg in "STGP_UPAIR_ZFIXED=0" "STGP_XX=0"; do
env $cfg timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:upair --metrics gpu__time_duration.sum --csv \
  python scripts/eval_launches.py fitc 10000 110 2000 30 2>/dev/null | grep -E "gpu__time" | python -c "
import sys,csv
for row in csv.reader(sys.stdin): print('fitc $cfg', row[4][:40], row[-1])"
done
