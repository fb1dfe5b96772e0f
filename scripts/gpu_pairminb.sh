# pair-gradient kernel occupancy: 6 (default), 7, 8 resident blocks per SM
for r in 1 2; do
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_mb7.so paper_2602_03609_b200/libstgp_b200_mb8.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --workload vecchia --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('vecchia $lib', round(d['ms_per_step'],3), d['nll'], d['grad'][:2])"
done
done
