#!/bin/bash
# round-2 closing evidence (v5): benches, the launch list of one cfg4 evaluation, full ncu captures
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/final_v5
mkdir -p $O
timeout -s KILL 900 python bench.py > $O/bench_vif.jsonl 2> $O/bench_vif.err
timeout -s KILL 600 python bench.py --workload vecchia > $O/bench_vecchia.jsonl 2> $O/bench_vecchia.err
timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 > $O/bench_fitc.jsonl 2> $O/bench_fitc.err
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_vif.csv python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/launch_table.py $O/launches_vif.csv > $O/launches_vif_summary.txt 2>&1
gzip -f $O/launches_vif.csv
for k in vecchia_rows_kernel vif_grad_stored_kernel slice_cols_kernel colmax_rows_kernel ozaki_tc_kernel; do
  timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:$k --launch-count 1 --set full --import-source on \
    --clock-control none -o /tmp/cap_$k python scripts/eval_launches.py vif > /dev/null 2>&1
  [ -f /tmp/cap_$k.ncu-rep ] && python tools/ncu_summary.py /tmp/cap_$k.ncu-rep > $O/full_$k.txt 2>&1
done
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:vecchia_rows_kernel --launch-skip 1 --launch-count 1 --set full \
  --import-source on --clock-control none -o /tmp/cap_vgrad python scripts/eval_launches.py vecchia > /dev/null 2>&1
[ -f /tmp/cap_vgrad.ncu-rep ] && python tools/ncu_summary.py /tmp/cap_vgrad.ncu-rep 1100000 > $O/full_vecchia_grad_rows.txt 2>&1
[ -f /tmp/cap_vgrad.ncu-rep ] && python tools/ncu_lines.py /tmp/cap_vgrad.ncu-rep 30 1100000 > $O/lines_vecchia_grad_rows.txt 2>&1
for f in $O/bench_*.jsonl; do echo "== $f"; tail -1 $f | cut -c1-400; done
cat $O/launches_vif_summary.txt | head -25
for f in $O/full_*.txt; do echo "== $f"; sed -n '3p;24p;25p;26p' $f; done
