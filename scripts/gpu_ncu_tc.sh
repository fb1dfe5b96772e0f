# ncu --set full of the tcgen05 Ozaki kernel inside one VIF evaluation: launch 0 (W = L^-1 U, triangle-cut rows
# form) and launch 5 (K = S S^T, symmetric column form); summaries plus the memory-unit breakdown
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/nctc
for skip in 0 5; do
  timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:ozaki_tc_kernel --launch-skip $skip --launch-count 1 \
    --set full --import-source on --clock-control none -o gpurun_out/nctc/tc_$skip python scripts/eval_launches.py vif \
    > gpurun_out/nctc/tc_$skip.log 2>&1
  python tools/ncu_summary.py gpurun_out/nctc/tc_$skip.ncu-rep > gpurun_out/nctc/tc_$skip.txt 2>&1
  ncu -i gpurun_out/nctc/tc_$skip.ncu-rep --page raw --csv > gpurun_out/nctc/tc_${skip}_raw.csv 2>&1
  head -12 gpurun_out/nctc/tc_$skip.txt
done
