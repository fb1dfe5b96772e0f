# ncu --set full of the tcgen05 kernel inside one cfg4 VIF evaluation: launch 6 (X = K^-1 V', rows form, S = 6)
# and launch 10 (V'F^T, column form, CY = 4)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/nctc2; mkdir -p $O
for skip in 6 10; do
  timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:ozaki_tc_kernel --launch-skip $skip --launch-count 1 \
    --set full --clock-control none -o $O/tc_$skip python scripts/eval_launches.py vif > $O/tc_$skip.log 2>&1
  python tools/ncu_summary.py $O/tc_$skip.ncu-rep > $O/full_tc_$skip.txt 2>&1
  head -26 $O/full_tc_$skip.txt | grep -E "Duration|tensor|dram|kernel:"
done
rm -f $O/*.ncu-rep
