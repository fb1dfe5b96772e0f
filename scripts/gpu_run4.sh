export PATH=/usr/local/cuda/bin:$PATH
timeout -s KILL 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r4_launches_vif.csv python scripts/eval_launches.py vif > gpurun_out/r4_vif.log 2>&1
python tools/launch_table.py gpurun_out/r4_launches_vif.csv > gpurun_out/r4_launches_vif.txt 2>&1
gzip -f gpurun_out/r4_launches_vif.csv
cat gpurun_out/r4_launches_vif.txt
