# U-pair kernel occupancy: default (64 registers) vs 5 (48) and 6 (40) resident blocks per SM
for r in 1 2; do
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_up5.so paper_2602_03609_b200/libstgp_b200_up6.so; do
  STGP_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']
print('vif $lib', round(d['ms_per_step'],2), d['grad'][:2], {k: round(v,2) for k,v in p.items() if k in ('g_upair_sigma',)})"
done
done
