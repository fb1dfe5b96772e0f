"""Timing probe of the VIF pipeline phases at a given scale (GPU)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

stations, days, m, mv = (int(a) for a in sys.argv[1:5])
box = (4.6e6, 2.9e6) if stations >= 2000 else (1.0, 1.0)
theta = S.synth.THETA_T3 if stations >= 2000 else S.synth.THETA_SEC4
x, y, t, resp = S.synth.station_day(stations, days, box=box, theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ctx.profile(True)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
t0 = time.perf_counter(); ind = S.sts_kmeanspp(ds, m, 20260203); t1 = time.perf_counter()
print(f"n={len(x)} sts: M={ind.M} ({ind.m_s}x{ind.m_t}) {t1-t0:.3f}s", flush=True)
use_dc = len(sys.argv) > 5 and sys.argv[5] == "dc"
nb = (S.correlation_neighbors(ds, theta, mv) if use_dc else S.residual_neighbors(ds, theta, ind, mv))
t2 = time.perf_counter()
print(f"d_r search: {t2-t1:.3f}s whiten={ctx.profile_get('dr_whiten')} knn={ctx.profile_get('knn_dr')}", flush=True)
s = S.build_vif(ds, theta, ind, nb, S.OBSERVATION); t3 = time.perf_counter()
print(f"build_vif: {t3-t2:.3f}s", flush=True)
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
for rep in range(reps):
    t4 = time.perf_counter(); v, g = S.evaluate(s, theta); t5 = time.perf_counter()
    print(f"eval {rep}: {t5-t4:.3f}s nll={v:.6f} rows={ctx.profile_get('rows')} vifgrad={ctx.profile_get('rows_vifgrad')}", flush=True)
    if rep == 0:
        ctx.profile_reset()  # first evaluation allocates the work pool
prof = ctx.profile_all()
for k, (ms, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:16s} {ms / max(cnt, 1):9.2f} ms/call x{cnt}")
