export PATH=/usr/local/cuda/bin:$PATH
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/r7_tests.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r7_launches_vif.csv python scripts/eval_launches.py vif > gpurun_out/r7_vif.log 2>&1
python tools/launch_table.py gpurun_out/r7_launches_vif.csv > gpurun_out/r7_launches_vif.txt 2>&1
gzip -f gpurun_out/r7_launches_vif.csv
cat gpurun_out/r7_tests.log gpurun_out/r7_launches_vif.txt
