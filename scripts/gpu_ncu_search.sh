# ncu --set full of one launch of a search kernel ($1) in the cfg4 d_r search (search_cold_probe.py)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
K=$1
timeout -s KILL 900 ncu --kernel-name regex:$K --launch-skip 1 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/ncu_$K python scripts/search_cold_probe.py > gpurun_out/ncu_$K.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$K.ncu-rep > gpurun_out/ncu_$K.txt 2>&1
head -34 gpurun_out/ncu_$K.txt
python tools/ncu_lines.py gpurun_out/ncu_$K.ncu-rep 22 > gpurun_out/ncu_${K}_lines.txt 2>&1
head -23 gpurun_out/ncu_${K}_lines.txt
