set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
STGP_OZAKI_TC=0 timeout -s KILL 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shards.py -x -q -s -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r1_configs.log
timeout -s KILL 300 python -m pytest tests/test_gpu_ozaki.py -x -q -s -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r1_ozaki.log
cat gpurun_out/r1_configs.log gpurun_out/r1_ozaki.log
