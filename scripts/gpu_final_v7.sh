#!/bin/bash
# closing evidence v7: GPU suite, smoke, the three benches, ncu of the d_r search kernel
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/final_v7
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -1 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench_vif.jsonl 2> $O/bench_vif.err
timeout -s KILL 600 python bench.py --workload vecchia > $O/bench_vecchia.jsonl 2> $O/bench_vecchia.err
timeout -s KILL 900 python bench.py --workload fitc --steps 3 --warmup 3 > $O/bench_fitc.jsonl 2> $O/bench_fitc.err
STGP_DR_STATS=1 timeout -s KILL 300 python scripts/search_cold_probe.py 4 > $O/dr_stats.log 2>&1
timeout -s KILL 900 ncu --kernel-name regex:knn_dr_kernel --launch-skip 1 --launch-count 1 --set full --import-source on \
  --clock-control none -o /tmp/cap_knn_dr python scripts/search_cold_probe.py > /dev/null 2>&1
python tools/ncu_summary.py /tmp/cap_knn_dr.ncu-rep > $O/full_knn_dr_kernel.txt 2>&1
for w in vif vecchia fitc; do python - $O $w <<'PY'
import json, sys
O, w = sys.argv[1], sys.argv[2]
d = json.loads(open(f"{O}/bench_{w}.jsonl").read().strip().splitlines()[-1])
print(w, round(d["value"], 3), round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"], 3), "frac", round(d["roofline"]["frac"], 3),
      {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items() if ("search" in k and "all" not in k) or k == "seeding_s"})
PY
done
grep "phase " $O/dr_stats.log | tail -7
head -24 $O/full_knn_dr_kernel.txt | sed -n '3p;20,24p'
