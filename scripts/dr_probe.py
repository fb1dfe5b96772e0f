import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2602_03609_b200 as S
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ctx.profile(True)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
ind = S.sts_kmeanspp(ds, 1000, 20260203)
for rep in range(3):
    t0 = time.perf_counter(); nb = S.residual_neighbors(ds, S.synth.THETA_T3, ind, 30); t1 = time.perf_counter()
    print(f"rep {rep}: d_r search wall {t1 - t0:.3f}s", flush=True)
    del nb
    t2 = time.perf_counter(); print(f"  release {t2 - t1:.3f}s", flush=True)
for k_, v_ in ctx.profile_all().items():
    print(f"  {k_:16s} {v_[0] / max(v_[1], 1):9.2f} ms/call x{v_[1]}")
