#!/bin/bash
# launch list of one cfg4 evaluation after the triangular products moved to tcgen05; W-trmm tc kernel capture;
# full per-line table of the Vecchia gradient kernel
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/v9
mkdir -p $O
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_vif.csv python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/launch_table.py $O/launches_vif.csv > $O/launches_vif_summary.txt 2>&1
gzip -f $O/launches_vif.csv
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:ozaki_tc_kernel --launch-count 1 --set full --import-source on \
  --clock-control none -o $O/tc_W python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/ncu_summary.py $O/tc_W.ncu-rep > $O/full_ozaki_tc_W_trmm.txt 2>&1
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:vecchia_rows_kernel --launch-skip 1 --launch-count 1 --set full \
  --import-source on --clock-control none -o $O/vgrad python scripts/eval_launches.py vecchia > /dev/null 2>&1
python tools/ncu_summary.py $O/vgrad.ncu-rep 1100000 > $O/full_vecchia_grad_rows.txt 2>&1
python tools/ncu_lines.py $O/vgrad.ncu-rep 400 1100000 > $O/lines_vecchia_grad_rows.txt 2>&1
head -40 $O/launches_vif_summary.txt
sed -n 1,30p $O/full_ozaki_tc_W_trmm.txt
