#!/bin/bash
# Full ncu captures of the engine's own kernels at cfg4, summarised on the box (the reports exceed
# gpurun's copy-back limit).  Ozaki cuBLASLt choices are replayed from a normal run.
set -u
rm -f /tmp/oztune.txt
STGP_OZAKI_TUNE_SAVE=/tmp/oztune.txt timeout 300 python scripts/vif_probe.py 10000 110 1000 30 dr 1 > /dev/null 2>&1
for k in ${KERNELS:-"vecchia_rows_kernel" "tile_ga" "tile_ef" "tile_vprime" "vif_grad_stored" "slice_cols" "combine_rows" "omega_prime" "i256x256" "knn_dr_kernel"}; do
  STGP_OZAKI_TUNE_LOAD=/tmp/oztune.txt timeout 600 ncu --set full --import-source on --kernel-name regex:"$k" \
    --launch-skip ${SKIP:-0} --launch-count 1 -o /tmp/cap_$k python scripts/vif_probe.py 10000 110 1000 30 dr 1 > /dev/null 2>&1
  if [ -f /tmp/cap_$k.ncu-rep ]; then
    python tools/ncu_summary.py /tmp/cap_$k.ncu-rep > gpurun_out/final_ncu_$k.txt 2>&1
    ncu -i /tmp/cap_$k.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active >> gpurun_out/final_ncu_raw.csv 2>/dev/null
  fi
done
