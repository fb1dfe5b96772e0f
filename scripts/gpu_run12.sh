# general-nu parity + regression of the closed-form paths, then the Vecchia and VIF benches
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_general_nu.py tests/test_gpu_vecchia.py tests/test_gpu_selection.py -x -q > gpurun_out/r12_tests.log 2>&1
tail -5 gpurun_out/r12_tests.log
timeout -s KILL 600 python bench.py --workload vecchia --steps 10 --warmup 3 > gpurun_out/r12_bench_vecchia.jsonl 2> gpurun_out/r12_bench_vecchia.err
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r12_bench_vif.jsonl 2> gpurun_out/r12_bench_vif.err
python - <<'PY'
import json
for f in ("gpurun_out/r12_bench_vecchia.jsonl", "gpurun_out/r12_bench_vif.jsonl"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("search_s"), d.get("phase_ms", {}).get("rows"), {k: d.get(k) for k in ("dr_search_s", "dc_search_s", "search_warm_s")})
    except Exception as e:
        print(f, "ERR", e)
PY
