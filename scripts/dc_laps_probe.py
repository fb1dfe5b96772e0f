"""Host-side phase laps of the spatial d_c search (M = 0) at cfg4 (STGP_DR_HOSTLAPS=1)."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ["STGP_DC_SPATIAL"] = "1"
import paper_2602_03609_b200 as S  # noqa: E402

x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t = x[perm], y[perm], t[perm]
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
ctx.fp64_peak_tflops()
for rep in range(4):
    t0 = time.perf_counter()
    nb = S.correlation_neighbors(ds, S.synth.THETA_T3, 30)
    print(f"search {rep}: {time.perf_counter() - t0:.4f} s", file=sys.stderr, flush=True)
