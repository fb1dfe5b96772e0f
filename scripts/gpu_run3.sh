timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/r3_tests.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err
timeout -s KILL 600 python bench.py --workload fitc --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r3_fitc.json 2> gpurun_out/r3_fitc.err
STGP_OZAKI_MIN_M=100000 timeout -s KILL 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r3_bench_dmma.json 2> gpurun_out/r3_bench_dmma.err
cat gpurun_out/r3_tests.log
