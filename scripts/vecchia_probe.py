"""Vecchia NLL+grad at cfg4 (d_c neighbours, m = 30): per-call timing."""
import sys
import time

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ctx.profile(True)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
nb = S.correlation_neighbors(ds, theta, 30)
s = S.build_vecchia(ds, theta, nb, S.OBSERVATION)
for r in range(4):
    t0 = time.perf_counter()
    v, g = S.evaluate(s, theta)
    print(f"eval {r}: {time.perf_counter() - t0:.4f}s nll={v:.6f}", flush=True)
print(ctx.profile_all())
