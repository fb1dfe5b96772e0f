# ncu --set full of one launch of kernel $1 inside one VIF evaluation (eval_launches.py), summary + hot lines
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
K=$1; shift
timeout -s KILL 900 env "$@" ncu --profile-from-start off --kernel-name regex:$K --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/ncu_$K python scripts/eval_launches.py vif > gpurun_out/ncu_$K.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$K.ncu-rep > gpurun_out/ncu_$K.txt 2>&1
head -36 gpurun_out/ncu_$K.txt
python tools/ncu_lines.py gpurun_out/ncu_$K.ncu-rep 25 > gpurun_out/ncu_${K}_lines.txt 2>&1
head -26 gpurun_out/ncu_${K}_lines.txt
