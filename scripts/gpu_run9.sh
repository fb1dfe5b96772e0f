export PATH=/usr/local/cuda/bin:$PATH
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/r9_tests.log
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err
timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r9_fitc.json 2> gpurun_out/r9_fitc.err
timeout -s KILL 900 python bench.py --stations 1000 --days 100 --m_v 20 --m 200 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r9_cfg3.json 2> gpurun_out/r9_cfg3.err
timeout -s KILL 900 python bench.py --workload vecchia --stations 1000 --days 100 --m_v 20 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r9_cfg2.json 2> gpurun_out/r9_cfg2.err
cat gpurun_out/r9_tests.log
