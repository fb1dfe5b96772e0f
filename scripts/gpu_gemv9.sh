# FITC GEMV (M = 2144): 256-row passes (default) vs nine rows per thread in one pass (libstgp_b200_rb9.so)
export PATH=/usr/local/cuda/bin:$PATH
for lib in paper_2602_03609_b200/libstgp_b200.so paper_2602_03609_b200/libstgp_b200_rb9.so; do
STGP_LIB=$lib timeout -s KILL 900 ncu --clock-control none --profile-from-start off --kernel-name regex:gemv_n --metrics gpu__time_duration.sum --csv \
  python scripts/eval_launches.py fitc 10000 110 2000 30 2>/dev/null | grep -E "gpu__time" | python -c "
import sys,csv
for row in csv.reader(sys.stdin): print('$lib'[-12:], row[4][:34], row[-1])"
done
