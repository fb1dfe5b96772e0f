"""Cold and warm d_r search wall times at cfg4 (first call grows the device memory pool and loads modules)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t = x[perm], y[perm], t[perm]
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
ctx.fp64_peak_tflops()
ind = S.sts_kmeanspp(ds, 1000, 20260203)
ctx.profile(True)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    t0 = time.perf_counter()
    nb = S.residual_neighbors(ds, S.synth.THETA_T3, ind, 30)
    dt = time.perf_counter() - t0
    prof = {k: round(v[0], 1) for k, v in ctx.profile_all().items()}
    ctx.profile_reset()
    print(f"search {rep}: {dt:.3f} s  {prof}", flush=True)
