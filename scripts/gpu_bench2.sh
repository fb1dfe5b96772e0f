# Vecchia + VIF benches (short) and the row-kernel phase times
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
TAG=${1:-x}
timeout -s KILL 600 python bench.py --workload vecchia --steps 20 --warmup 3 > gpurun_out/${TAG}_vecchia.jsonl 2> gpurun_out/${TAG}_vecchia.err
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_vif.jsonl 2> gpurun_out/${TAG}_vif.err
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
for w in ("vecchia", "vif"):
    f = f"gpurun_out/{tag}_{w}.jsonl"
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(w, round(d["value"], 3), "ms", round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"], 3), "frac", round(r["frac"], 3), "phase", r.get("phase_ms"), "clk", d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "ERR", e)
PY
