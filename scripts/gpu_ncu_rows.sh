# ncu full capture of the Vecchia gradient row kernel (cfg4 data, d_c m = 30) with source correlation
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout -s KILL 900 ncu --kernel-name vecchia_rows_kernel --launch-skip 2 --launch-count 1 --set full \
  --import-source on --clock-control none -o gpurun_out/rows_grad python bench.py --workload vecchia --steps 2 --warmup 3 \
  > gpurun_out/rows_grad_ncu.log 2>&1
ls -la gpurun_out/rows_grad.ncu-rep
ncu -i gpurun_out/rows_grad.ncu-rep --page source --csv --print-source cuda > gpurun_out/rows_grad_src_cuda.csv 2>&1
ncu -i gpurun_out/rows_grad.ncu-rep --page source --csv --print-source sass > gpurun_out/rows_grad_src_sass.csv 2>&1
python tools/ncu_summary.py gpurun_out/rows_grad.ncu-rep 1100000 > gpurun_out/rows_grad_summary.txt 2>&1
head -5 gpurun_out/rows_grad_src_cuda.csv | cut -c1-600
