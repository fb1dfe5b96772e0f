import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2602_03609_b200 as S
theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
nb = S.correlation_neighbors(ds, theta, 30)
s = S.build_vecchia(ds, theta, nb, S.OBSERVATION)
last = t == t.max()
T = np.column_stack([x[last], y[last], np.full(int(last.sum()), t.max() + 1.0)])
for r in range(3):
    t0 = time.perf_counter(); pr = S.predict(s, resp, None, None, T, pred_m_v=30); print(f"vecchia predict {r}: {time.perf_counter()-t0:.3f}s", flush=True)
