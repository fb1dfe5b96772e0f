# ncu full captures of the Ozaki slicing kernels (column form, S = 7) and colmax within one VIF evaluation
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for K in slice_cols_kernel colmax_kernel tile_ef_kernel; do
  timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:$K --launch-count 1 --set full --import-source on \
    --clock-control none -o gpurun_out/ncu_$K python scripts/eval_launches.py vif > gpurun_out/ncu_$K.log 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_$K.ncu-rep > gpurun_out/ncu_$K.txt 2>&1
  head -32 gpurun_out/ncu_$K.txt
done
