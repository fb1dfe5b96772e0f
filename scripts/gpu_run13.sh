# full GPU suite, then both benches (search times are the check for the widened list code)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/r13_tests.log 2>&1
tail -3 gpurun_out/r13_tests.log
timeout -s KILL 600 python bench.py --workload vecchia --steps 10 --warmup 3 > gpurun_out/r13_bench_vecchia.jsonl 2> gpurun_out/r13_bench_vecchia.err
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r13_bench_vif.jsonl 2> gpurun_out/r13_bench_vif.err
python - <<'PY'
import json
for f in ("gpurun_out/r13_bench_vecchia.jsonl", "gpurun_out/r13_bench_vif.jsonl"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 3), round(d["ms_per_step"], 2), {k: d.get(k) for k in d if "search" in k or "seeding" in k})
    except Exception as e:
        print(f, "ERR", e)
PY
