"""VIF prediction at cfg4 scale: 1-day-ahead mean / variance at every station (a26)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ctx.profile(True)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
ind = S.sts_kmeanspp(ds, 1000, 20260203)
nb = S.residual_neighbors(ds, theta, ind, 30)
s = S.build_vif(ds, theta, ind, nb, S.OBSERVATION)
S.evaluate(s, theta)
last = t == t.max()
T = np.column_stack([x[last], y[last], np.full(int(last.sum()), t.max() + 1.0)])
for pm in (30,):
    for r in range(3):
        t0 = time.perf_counter()
        pr = S.predict(s, resp, None, None, T, pred_m_v=pm)
        dt = time.perf_counter() - t0
        print(f"pred_m_v={pm} rep {r}: {dt:.3f}s  var=({pr.var.min():.4f}, {pr.var.max():.4f})", flush=True)
for k, (ms, c) in sorted(ctx.profile_all().items(), key=lambda kv: -kv[1][0])[:8]:
    print(f"  {k:16s} {ms / max(c, 1):9.2f} ms x{c}")
