"""Cold vs warm d_r search at cfg4 (module loading, first allocations, clocks)."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
print("loading:", os.environ.get("CUDA_MODULE_LOADING", "default"))
t0 = time.perf_counter(); ctx.dmma_peak_tflops(); print(f"dmma peak {time.perf_counter() - t0:.3f}s", flush=True)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
ctx.profile(True)
ind = S.sts_kmeanspp(ds, 1000, 20260203)
for rep in range(int(os.environ.get("REPS", "3"))):
    ctx.profile_reset()
    t0 = time.perf_counter(); nb = S.residual_neighbors(ds, theta, ind, 30); dt = time.perf_counter() - t0
    prof = {k: round(v[0], 1) for k, v in ctx.profile_all().items()}
    print(f"search {rep}: {dt:.3f}s {prof}", flush=True)
    del nb
