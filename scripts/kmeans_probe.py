"""Timing of joint kMeans++ seeding at the cfg4/cfg5 scale (n = 1.1M observations, k = 2000 centers in the
scaled (x / ss, y / ss, t / ts) space, joint_kmeanspp_inducing), certified parallel picks vs the
one-thread exact picks (STGP_KMEANS_CERTIFIED=0 in a second process); both give identical centers."""
import hashlib
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

x, y, t, _ = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t = x[perm], y[perm], t[perm]
tr, sr = S.effective_ranges(S.synth.THETA_T3)
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
S.joint_kmeanspp_inducing(ds, 50, sr, tr, 1)  # warm-up (module loads, pool)
ctx.profile(True)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
t0 = time.perf_counter()
ind = S.joint_kmeanspp_inducing(ds, k, sr, tr, 20260203)
dt = time.perf_counter() - t0
pts = ind.points
prof = {name: [round(ms, 3), cnt] for name, (ms, cnt) in ctx.profile_all().items()}
print(json.dumps({"n": len(x), "k": k, "joint_seeding_s": dt, "sha256": hashlib.sha256(pts.tobytes()).hexdigest()[:16],
                  "regions_ms_count": prof}))
