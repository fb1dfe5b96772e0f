# two-pass Vecchia gradient: parity tests, A/B timing, capture of both passes
export PATH=/usr/local/cuda/bin:$PATH
make -C paper_2602_03609_b200/csrc -q || echo "stale build"
O=gpurun_out/vsplit; mkdir -p $O
timeout -s KILL 900 python -m pytest -q -x tests/test_gpu_vecchia.py tests/test_gpu_configs.py tests/test_gpu_fit.py tests/test_gpu_shards.py tests/test_gpu_many_times.py tests/test_gpu_wide_sets.py 2>&1 | tail -2
for r in 1 2; do
for cfg in "STGP_VGRAD_SPLIT=0" "STGP_XX=0"; do
  env $cfg timeout -s KILL 600 python bench.py --workload vecchia --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('vecchia [$cfg]', round(d['ms_per_step'],3), d['nll'], d['grad'][:3], round(d['roofline']['frac'],3))"
done
done
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_vecchia.csv python scripts/eval_launches.py vecchia > /dev/null 2>&1
python tools/launch_table.py $O/launches_vecchia.csv > $O/launches_vecchia_summary.txt 2>&1
head -8 $O/launches_vecchia_summary.txt
for k in vecchia_rows_kernel vecchia_pair_grad_kernel; do
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:$k --launch-count 1 --set full \
  --import-source on --clock-control none -o $O/$k python scripts/eval_launches.py vecchia > $O/$k.log 2>&1
python tools/ncu_summary.py $O/$k.ncu-rep 1100000 > $O/full_$k.txt 2>&1
python tools/ncu_lines.py $O/$k.ncu-rep 60 1100000 > $O/lines_$k.txt 2>&1
sed -n 1,30p $O/full_$k.txt
done
