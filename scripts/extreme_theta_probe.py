"""Robustness: evaluate Vecchia/VIF at extreme finite parameters (must return or raise, never hang)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

x, y, t, resp = S.synth.station_day(200, 10, theta=S.synth.THETA_SEC4, seed=3)
ds = S.order_observations(x, y, t, resp, seed=3)
th0 = S.synth.THETA_SEC4
ind = S.sts_kmeanspp(ds, 30, 1)
nb = S.residual_neighbors(ds, th0, ind, 10)
nbc = S.correlation_neighbors(ds, th0, 10)
for th in [(4e186, 1e297, 1e300, 6.6e-119, 1.0, 1.5, 1.0, 2e260), (1e-300, 1e300, 1e-300, 1e300, 1e-6, 1.5, 0.0, 0.0),
           (1.0, 1.0, 1e300, 1e300, 1.0, 1.5, 1.0, 1e300), (0.0, 1e-300, 1.0, 1.0, 0.5, 1.5, 0.5, 0.5)]:
    for kind in ("vecchia", "vif"):
        t0 = time.perf_counter()
        try:
            s = S.build_vecchia(ds, th0, nbc, S.OBSERVATION) if kind == "vecchia" else S.build_vif(ds, th0, ind, nb, S.OBSERVATION)
            v, g = S.evaluate(s, th)
            r = f"ok {v}"
        except Exception as e:  # noqa: BLE001
            r = f"{type(e).__name__}: {str(e)[:80]}"
        print(kind, th, f"{time.perf_counter() - t0:.3f}s", r, flush=True)
