export PATH=/usr/local/cuda/bin:$PATH
timeout -s KILL 600 ncu --profile-from-start off --kernel-name regex:dgemm_kernel --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r11_dgemm_list.csv python scripts/eval_launches.py vif > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r11_dgemm_list.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=[(float(r[vi].replace(',','')), int(r[ii]), r[ki][:40]) for r in rows[1:]]
d.sort(reverse=True)
print(d[:5])
open('gpurun_out/r11_big.txt','w').write(str(sorted(d[:2], key=lambda x: x[1])[0][1]))
PY
IDX=$(cat gpurun_out/r11_big.txt)
timeout -s KILL 900 ncu --profile-from-start off --kernel-name regex:dgemm_kernel --launch-skip $IDX --launch-count 1 --set full --import-source on -o /tmp/dg python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/ncu_summary.py /tmp/dg.ncu-rep > gpurun_out/r11_dgemm_ncu.txt 2>&1
head -60 gpurun_out/r11_dgemm_ncu.txt
