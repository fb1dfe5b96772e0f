#!/bin/bash
# closing evidence v16: GPU suite, smoke, the three benches, launch list of one cfg4 VIF evaluation,
# Vecchia gradient kernel capture (per-line table)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/final_v16
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -1 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench_vif.jsonl 2> $O/bench_vif.err
timeout -s KILL 600 python bench.py --workload vecchia > $O/bench_vecchia.jsonl 2> $O/bench_vecchia.err
timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 > $O/bench_fitc.jsonl 2> $O/bench_fitc.err
for w in vif vecchia fitc; do python - $O $w <<'PY'
import json, sys
O, w = sys.argv[1], sys.argv[2]
d = json.loads(open(f"{O}/bench_{w}.jsonl").read().strip().splitlines()[-1])
r = d["roofline"]
print(w, round(d["value"], 3), round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"], 3), "frac", round(r["frac"], 3),
      "int8", round(r.get("int8_tensor", r).get("frac", 0), 3), "step", round(r.get("step_fp64_equiv_frac", 0), 3), d["clocks"],
      {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items() if ("search" in k and "all" not in k) or k == "seeding_s"})
PY
done
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_vif.csv python scripts/eval_launches.py vif > /dev/null 2>&1
python tools/launch_table.py $O/launches_vif.csv > $O/launches_vif_summary.txt 2>&1
gzip -f $O/launches_vif.csv
head -16 $O/launches_vif_summary.txt
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_fitc.csv python scripts/eval_launches.py fitc 10000 110 2000 30 > /dev/null 2>&1
python tools/launch_table.py $O/launches_fitc.csv > $O/launches_fitc_summary.txt 2>&1
gzip -f $O/launches_fitc.csv
head -12 $O/launches_fitc_summary.txt
timeout -s KILL 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_vecchia.csv python scripts/eval_launches.py vecchia > /dev/null 2>&1
python tools/launch_table.py $O/launches_vecchia.csv > $O/launches_vecchia_summary.txt 2>&1
gzip -f $O/launches_vecchia.csv
head -6 $O/launches_vecchia_summary.txt
