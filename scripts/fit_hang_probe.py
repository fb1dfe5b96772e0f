"""Where does the cfg3 VIF fit stall at its second refresh? (timing of each selection step at theta_2)"""
import sys
import time

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

th2 = (0.005139336675910685, 1.3400172752771755, 0.07243396810989822, 26.491407042620768, 0.8177841134789464, 1.5,
       0.5221141790727776, 0.5712035695098758)
x, y, t, resp = S.synth.station_day(1000, 100, theta=S.synth.THETA_SEC4, seed=20260203)
ds = S.order_observations(x, y, t, resp, seed=20260203)
ctx = ds.ctx
ctx.profile(True)
t0 = time.perf_counter(); ind = S.sts_kmeanspp(ds, 200, 20260203); print("sts", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter(); nbc = S.correlation_neighbors(ds, th2, 20); print("dc search", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter(); nb = S.residual_neighbors(ds, th2, ind, 20); print("dr search", time.perf_counter() - t0, flush=True)
print({k: v for k, v in ctx.profile_all().items()}, flush=True)
t0 = time.perf_counter(); s = S.build_vif(ds, th2, ind, nb, S.OBSERVATION); print("build", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter(); v, g = S.evaluate(s, th2); print("eval", time.perf_counter() - t0, v, flush=True)
