import sys, time, statistics
sys.path.insert(0, ".")
import os
import paper_2602_03609_b200 as S
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t = x[perm], y[perm], t[perm]
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
ctx.fp64_peak_tflops()
res = {}
for mode in ("0", "1", "0", "1"):
    os.environ["STGP_DC_SPATIAL"] = mode
    ts = []
    for rep in range(6):
        t0 = time.perf_counter()
        nb = S.correlation_neighbors(ds, S.synth.THETA_T3, 30)
        ts.append(time.perf_counter() - t0)
    res.setdefault(mode, []).extend(ts[1:])
for m, v in res.items():
    print("spatial", m, "median", round(statistics.median(v), 4), "min", round(min(v), 4), [round(a, 3) for a in v])
