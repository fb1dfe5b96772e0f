#!/bin/bash
# final check on the round's last code: GPU suite, smoke, cfg4 VIF bench; ncu --set full of the tcgen05 kernel on
# the V'F^T column-form product and on X = K^-1 V' (rows form)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/final_v15
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -1 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench_vif.jsonl 2> $O/bench_vif.err
tail -1 $O/bench_vif.jsonl | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('vif', round(d['value'],3), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],3), 'frac', round(r['frac'],3), d['clocks'])"
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:"ozaki_tc_kernel<7, 1, 4>" --launch-count 1 --set full \
  --clock-control none -o $O/tc_cols python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/ncu_summary.py $O/tc_cols.ncu-rep > $O/full_ozaki_tc_VFt_cols.txt 2>&1
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:"ozaki_tc_kernel<6, 1, 2>" --launch-count 1 --set full \
  --clock-control none -o $O/tc_rows python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/ncu_summary.py $O/tc_rows.ncu-rep > $O/full_ozaki_tc_X_rows.txt 2>&1
head -24 $O/full_ozaki_tc_VFt_cols.txt | grep -E "Duration|tensor|dram|Throughput"
head -24 $O/full_ozaki_tc_X_rows.txt | grep -E "Duration|tensor|dram|Throughput"
rm -f $O/*.ncu-rep
