"""d_c search timing at cfg4: spatial-tile path (STGP_DC_SPATIAL=1) vs the default time-block kernel."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t = x[perm], y[perm], t[perm]
ctx = S.Context(0)
ctx.profile(True)
ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
ref = None
for legacy in ("0", "1", "0", "1"):
    os.environ["STGP_DC_SPATIAL"] = "0" if legacy == "1" else "1"
    ctx.profile_reset()
    t0 = time.perf_counter()
    nb = S.correlation_neighbors(ds, theta, 30)
    dt = time.perf_counter() - t0
    idx = nb.indices()
    same = ref is None or (idx == ref).all()
    ref = idx if ref is None else ref
    prof = {k: round(v[0], 2) for k, v in ctx.profile_all().items()}
    print(f"legacy={legacy}: wall {dt:.3f}s identical={same} {prof}", flush=True)
