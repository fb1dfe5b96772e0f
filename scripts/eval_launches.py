"""One VIF (or FITC / Vecchia) evaluation at a BASELINE configuration between cudaProfilerStart/Stop, for an
ncu launch list of exactly one evaluation:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file out.csv \
        python scripts/eval_launches.py [vif|fitc|vecchia] [stations days m m_v]
"""
import ctypes
import sys

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "vif"
stations, days, m, mv = (int(a) for a in (sys.argv[2:6] if len(sys.argv) > 5 else (10000, 110, 1000, 30)))
box = (4.6e6, 2.9e6) if stations >= 2000 else (1.0, 1.0)
theta = S.synth.THETA_T3 if stations >= 2000 else S.synth.THETA_SEC4
x, y, t, resp = S.synth.station_day(stations, days, box=box, theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
if kind == "vecchia":
    s = S.build_vecchia(ds, theta, S.correlation_neighbors(ds, theta, mv), S.OBSERVATION)
else:
    ind = S.sts_kmeanspp(ds, m, 20260203)
    s = (S.build_fitc(ds, theta, ind) if kind == "fitc"
         else S.build_vif(ds, theta, ind, S.residual_neighbors(ds, theta, ind, mv), S.OBSERVATION))
S.evaluate(s, theta)
S.evaluate(s, theta)
cudart = ctypes.CDLL("libcudart.so.12")
ctx.synchronize()
cudart.cudaProfilerStart()
v, g = S.evaluate(s, theta)
ctx.synchronize()
cudart.cudaProfilerStop()
print("nll", v, "launches", ctx.kernel_launches())
