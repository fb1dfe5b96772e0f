"""cfg5 probe (BASELINE.json): FITC with ~2000 sts inducing points on 1.1M station x day observations,
NLL + gradient evaluations, then 1-day-ahead predictive mean/variance at the 10k stations."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

stations = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
days = int(sys.argv[2]) if len(sys.argv) > 2 else 110
m = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(stations, days, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ctx.profile(True)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
t0 = time.perf_counter()
ind = S.sts_kmeanspp(ds, m, 20260203)
t1 = time.perf_counter()
print(f"n={len(x)} sts m={m}: M={ind.M} ({ind.m_s}x{ind.m_t}) {t1 - t0:.3f}s", flush=True)
s = S.build_fitc(ds, theta, ind)
t2 = time.perf_counter()
print(f"build_fitc {t2 - t1:.3f}s", flush=True)
for rep in range(3):
    t3 = time.perf_counter()
    v, g = S.evaluate(s, theta)
    t4 = time.perf_counter()
    print(f"eval {rep}: {t4 - t3:.3f}s nll={v:.6f}", flush=True)
    if rep == 0:
        ctx.profile_reset()
# 1-day-ahead prediction at every station
st_x, st_y = x[t == t.max()], y[t == t.max()]
targets = np.column_stack([st_x, st_y, np.full(len(st_x), t.max() + 1.0)])
t5 = time.perf_counter()
pr = S.predict(s, resp, None, None, targets)
t6 = time.perf_counter()
print(f"predict {len(targets)} targets: {t6 - t5:.3f}s mean|mu|={np.abs(pr.mu).mean():.4f} "
      f"var range=({pr.var.min():.4f}, {pr.var.max():.4f})", flush=True)
for k, (ms, cnt) in sorted(ctx.profile_all().items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:16s} {ms / max(cnt, 1):9.2f} ms/call x{cnt}")
