make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 1500 python -m pytest -q -x tests -m gpu 2>&1 | tail -15
for r in 1 2; do
for cfg in "STGP_VGRAD_SPLIT=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 600 python bench.py --workload vecchia --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('vecchia [$cfg]', round(d['ms_per_step'],3), d['nll'], d['grad'][:3], round(d['roofline']['frac'],3))"
done
done
