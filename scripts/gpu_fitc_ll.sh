# FITC (cfg5) launch list of one evaluation; ncu of its rows-form int8 product (K^-1 W)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/fitc_ll; mkdir -p $O
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_fitc.csv python scripts/eval_launches.py fitc 10000 110 2000 30 > /dev/null 2>&1
python tools/launch_table.py $O/launches_fitc.csv > $O/launches_fitc_summary.txt 2>&1
gzip -f $O/launches_fitc.csv
head -25 $O/launches_fitc_summary.txt
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:"ozaki_tc_kernel<6" --launch-count 1 --set full \
  --clock-control none -o $O/tc6 python scripts/eval_launches.py fitc 10000 110 2000 30 > $O/tc6.log 2>&1
python tools/ncu_summary.py $O/tc6.ncu-rep > $O/full_tc6.txt 2>&1
ncu -i $O/tc6.ncu-rep --page raw --csv > $O/tc6_raw.csv 2>&1
head -30 $O/full_tc6.txt
