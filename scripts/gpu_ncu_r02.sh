#!/bin/bash
# r02 evidence: launch list of one cfg4 VIF evaluation (real clocks) and full ncu captures of the top kernels
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/ncu_r02
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/ncu_r02/launches_vif.csv python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ncu_r02/launches_vif.csv > gpurun_out/ncu_r02/launches_vif_summary.txt 2>&1
gzip -f gpurun_out/ncu_r02/launches_vif.csv
for k in ozaki_tc_kernel vecchia_rows_kernel omega_prime tile_ga dgemm_kernel; do
  timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:$k --launch-count 1 --set full --import-source on \
    -o /tmp/cap_$k python scripts/eval_launches.py vif > /dev/null 2>&1
  if [ -f /tmp/cap_$k.ncu-rep ]; then
    python tools/ncu_summary.py /tmp/cap_$k.ncu-rep > gpurun_out/ncu_r02/full_$k.txt 2>&1
  fi
done
# the Vecchia half's gradient row kernel (cfg4 data, d_c, m = 30)
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:vecchia_rows_kernel --launch-count 1 --set full --import-source on \
  -o /tmp/cap_vgrad python scripts/eval_launches.py vecchia > /dev/null 2>&1
[ -f /tmp/cap_vgrad.ncu-rep ] && python tools/ncu_summary.py /tmp/cap_vgrad.ncu-rep > gpurun_out/ncu_r02/full_vecchia_grad_rows.txt 2>&1
cat gpurun_out/ncu_r02/launches_vif_summary.txt
for f in gpurun_out/ncu_r02/full_*.txt; do echo "== $f"; head -30 $f; done
