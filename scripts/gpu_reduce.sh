# warp-parallel compensated reduction of the per-block partials: full GPU suite + Vecchia A/B
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_prev.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --workload vecchia --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('vecchia $lib', round(d['ms_per_step'],3), d['nll'], d['grad'][:3])"
done
done
