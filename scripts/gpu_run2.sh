set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2_tests.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_tc.json 2> gpurun_out/r2_bench_tc.err
STGP_OZAKI_TC=0 timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_lt.json 2> gpurun_out/r2_bench_lt.err
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
cat gpurun_out/r2_tests.log
