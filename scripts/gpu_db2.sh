export PATH=/usr/local/cuda/bin:$PATH
STGP_OZAKI_ROWS_BN=32 timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:ozaki_tc --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --csv \
  python scripts/eval_launches.py vif 2>/dev/null | grep -E "gpu__time|tensor" | python -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
for r in rows[:12]: print(r[4][:60], r[-3], r[-1])"
