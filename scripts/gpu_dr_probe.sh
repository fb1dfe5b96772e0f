# d_r search statistics at cfg4 and an ncu capture of knn_dr_kernel with per-line hot spots
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
STGP_DR_STATS=1 timeout -s KILL 300 python scripts/search_cold_probe.py > gpurun_out/dr_stats.log 2>&1
grep "d_r tiles\|lag \|search" gpurun_out/dr_stats.log | head -24
timeout -s KILL 1200 ncu --kernel-name regex:knn_dr_kernel --launch-skip 1 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/ncu_knn_dr python scripts/search_cold_probe.py > gpurun_out/ncu_knn_dr.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_knn_dr.ncu-rep > gpurun_out/ncu_knn_dr.txt 2>&1
head -40 gpurun_out/ncu_knn_dr.txt
