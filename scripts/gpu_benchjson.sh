# bench line after the roofline object moved to the tcgen05 kernel (VIF and FITC)
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bj_vif.jsonl 2> gpurun_out/bj_vif.err
timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 > gpurun_out/bj_fitc.jsonl 2> gpurun_out/bj_fitc.err
timeout -s KILL 600 python bench.py --workload vecchia --steps 10 --warmup 3 > gpurun_out/bj_vecchia.jsonl 2> gpurun_out/bj_vecchia.err
for w in vif fitc vecchia; do tail -1 gpurun_out/bj_$w.jsonl | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$w', round(d['value'],3), r['bound'], round(r['frac'],3), r.get('traffic'), r.get('kernel','')[:60], [k for k in r if isinstance(r[k], dict)])"; done
tail -3 gpurun_out/bj_vif.err
