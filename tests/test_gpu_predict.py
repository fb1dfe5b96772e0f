"""GPU parity for predictions and GLS (test_approximations.cpp:321-455) against the oracle."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _theta(s2):
    return (s2,) + SEC4[1:]


def _targets(np_, seed, tmax):
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.random(np_), rng.random(np_), 1 + (tmax - 1) * rng.random(np_)])


def test_predict_exactness_limits(S):
    # test_approximations.cpp:321-368: full conditioning / all points vs dense kriging
    n = 80
    x, y, t, yv, _ = O.test_dataset(1, n, 21, n_times=6)
    th = _theta(0.05)
    T = _targets(12, 5, 9)
    mu_ref, var_ref = O.dense_predict(x, y, t, th, yv, T)
    ds = S.SpaceTimeDataset(x, y, t)
    full = S.NeighborSets.from_sets(ds, O.full_conditioning(n))
    pv = S.predict(S.build_vecchia(ds, th, full, S.OBSERVATION), yv, None, None, T, pred_m_v=n)
    assert np.allclose(pv.mu, mu_ref, rtol=1e-6, atol=1e-9) and np.allclose(pv.var, var_ref, rtol=1e-6)
    P = np.column_stack([x, y, t])
    pf = S.predict(S.build_fitc(ds, th, S.InducingSet.from_points(P)), yv, None, None, T)
    assert np.allclose(pf.mu, mu_ref, rtol=1e-5, atol=1e-8) and np.allclose(pf.var, var_ref, rtol=1e-5, atol=1e-5)
    vif = S.build_vif(ds, th, S.InducingSet.from_points(P[[3, 30, 60]]), full, S.OBSERVATION)
    pw = S.predict(vif, yv, None, None, T, pred_m_v=n)
    assert np.allclose(pw.mu, mu_ref, rtol=1e-6, atol=1e-9) and np.allclose(pw.var, var_ref, rtol=1e-6)


@pytest.mark.parametrize("m", [10, 31])
def test_vecchia_predict_parity(S, m):
    x, y, t, yv, X = O.test_dataset(1, 1500, 25, n_times=8, p=1)
    beta = np.array([0.5])
    th = _theta(0.1)
    T = _targets(60, 7, 10)
    Xp = np.random.default_rng(1).normal(size=(60, 1))
    nbr = O.dc_neighbors(x, y, t, th, 10)
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_vecchia(ds, th, S.NeighborSets.from_sets(ds, nbr), S.OBSERVATION)
    pr = S.predict(s, yv, X, beta, T, Xp, pred_m_v=m)
    mu, var = O.OracleModel("vecchia", x, y, t, th, nbr=nbr).predict(yv, T, m, X, beta, Xp)
    assert np.allclose(pr.mu, mu, rtol=1e-9, atol=1e-12) and np.allclose(pr.var, var, rtol=1e-9, atol=1e-12)


def test_euclid_predict(S):
    # Vecchia with Euclidean neighbour sets predicts with the scaled Euclidean target metric
    x, y, t, yv, _ = O.test_dataset(1, 800, 27, n_times=8)
    th = _theta(0.1)
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.euclidean_neighbors(ds, 10, 0.2, 3.0)
    s = S.build_vecchia(ds, th, nb, S.OBSERVATION)
    T = _targets(30, 3, 9)
    pr = S.predict(s, yv, None, None, T, pred_m_v=10)
    # reference semantics restated here: nearest 10 by ((dx/ss)^2 + (dy/ss)^2) + (dt/ts)^2
    for p in range(30):
        d = ((T[p, 0] - x) / 0.2) ** 2 + ((T[p, 1] - y) / 0.2) ** 2 + ((T[p, 2] - t) / 3.0) ** 2
        N = np.sort(np.lexsort((np.arange(len(x)), d))[:10])
        C = np.array([[O.kernel_eval(th, np.hypot(x[a] - x[b], y[a] - y[b]), abs(t[a] - t[b])) for b in N] for a in N])
        C += th[0] * np.eye(10)
        c = np.array([O.kernel_eval(th, np.hypot(T[p, 0] - x[a], T[p, 1] - y[a]), abs(T[p, 2] - t[a])) for a in N])
        A = np.linalg.solve(C, c)
        assert pr.mu[p] == pytest.approx(A @ yv[N], rel=1e-8, abs=1e-10)
        assert pr.var[p] == pytest.approx(max(th[1] + th[0] - A @ c, 0.0), rel=1e-8, abs=1e-10)


def test_fitc_predict_parity(S):
    x, y, t, yv, _ = O.test_dataset(1, 1200, 29, n_times=8)
    th = _theta(0.2)
    Z = np.column_stack([np.random.default_rng(2).random(30), np.random.default_rng(3).random(30),
                         1 + 7 * np.random.default_rng(4).random(30)])
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_fitc(ds, th, S.InducingSet.from_points(Z))
    T = _targets(50, 9, 10)
    pr = S.predict(s, yv, None, None, T)
    mu, var = O.OracleModel("fitc", x, y, t, th, Z=Z).predict(yv, T, 0)
    assert np.allclose(pr.mu, mu, rtol=1e-8, atol=1e-11) and np.allclose(pr.var, var, rtol=1e-8, atol=1e-11)


def test_vif_predict_parity(S):
    x, y, t, yv, _ = O.test_dataset(1, 1000, 31, n_times=8)
    th = _theta(0.1)
    Z = np.column_stack([x, y, t])[::37]
    nbr = O.dr_neighbors(x, y, t, th, Z, 10)
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_vif(ds, th, S.InducingSet.from_points(Z), S.NeighborSets.from_sets(ds, nbr, S.api.METRIC_DR),
                    S.OBSERVATION)
    T = _targets(40, 11, 10)
    pr = S.predict(s, yv, None, None, T, pred_m_v=10)
    mu, var = O.OracleModel("vif", x, y, t, th, nbr=nbr, Z=Z).predict(yv, T, 10)
    assert np.allclose(pr.mu, mu, rtol=1e-8, atol=1e-10) and np.allclose(pr.var, var, rtol=1e-8, atol=1e-10)
    assert (pr.var >= 0).all() and (pr.var <= th[1] + th[0] + 1e-8).all()


def test_prediction_limit_cases(S):
    # test_approximations.cpp:370-396
    x, y, t, yv, _ = O.test_dataset(1, 50, 23, n_times=8)
    th = _theta(1e-12)
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.correlation_neighbors(ds, th, 10)
    pr = S.predict(S.build_vecchia(ds, th, nb, S.OBSERVATION), yv, None, None, [[x[20], y[20], t[20]]], pred_m_v=10)
    assert pr.mu[0] == pytest.approx(yv[20], rel=1e-5) and pr.var[0] < 1e-8
    th2 = _theta(0.25)
    pr = S.predict(S.build_vecchia(ds, th2, nb, S.OBSERVATION), yv, None, None, [[300.0, 300.0, 500.0]], pred_m_v=10)
    assert abs(pr.mu[0]) < 1e-10 and pr.var[0] == pytest.approx(1.25, rel=1e-10)


@pytest.mark.parametrize("kind", ["vecchia", "fitc", "vif"])
def test_gls_parity(S, kind):
    # test_approximations.cpp:444-455 plus differential parity for FITC / VIF
    n = 600
    x, y, t, yv, X = O.test_dataset(1, n, 29, n_times=6, p=2)
    th = _theta(0.15)
    ds = S.SpaceTimeDataset(x, y, t)
    Z = np.column_stack([x, y, t])[::29]
    if kind == "vecchia":
        nbr = O.dc_neighbors(x, y, t, th, 12)
        s = S.build_vecchia(ds, th, S.NeighborSets.from_sets(ds, nbr), S.OBSERVATION)
        om = O.OracleModel("vecchia", x, y, t, th, nbr=nbr)
    elif kind == "fitc":
        s = S.build_fitc(ds, th, S.InducingSet.from_points(Z))
        om = O.OracleModel("fitc", x, y, t, th, Z=Z)
    else:
        nbr = O.dr_neighbors(x, y, t, th, Z, 12)
        s = S.build_vif(ds, th, S.InducingSet.from_points(Z), S.NeighborSets.from_sets(ds, nbr), S.OBSERVATION)
        om = O.OracleModel("vif", x, y, t, th, nbr=nbr, Z=Z)
    b = S.gls_beta(s, yv, X)
    assert np.allclose(b, om.gls_beta(yv, X), rtol=1e-9, atol=1e-12)


def test_vif_predict_station_day_pruned_search(S):
    # time-sorted station x day data: the d_r target search visits time blocks nearest first and
    # prunes blocks and pairs with the |w| bounds; results must equal the oracle's exhaustive search
    x, y, t, yv = S.synth.station_day(150, 6, seed=17)
    perm = O.order_observations(t, 17)
    x, y, t, yv = x[perm], y[perm], t[perm], yv[perm]
    th = S.synth.THETA_SEC4
    Z, _, _ = O.sts_kmeanspp(x, y, t, 60, 17)
    nbr = O.dr_neighbors(x, y, t, th, Z, 10)
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_vif(ds, th, S.InducingSet.from_points(Z), S.NeighborSets.from_sets(ds, nbr, S.api.METRIC_DR),
                    S.OBSERVATION)
    last = t == t.max()
    T = np.vstack([np.column_stack([x[last], y[last], np.full(int(last.sum()), t.max() + 1.0)]),
                   np.column_stack([x[:20] + 0.01, y[:20], t[:20] + 0.5])])
    pr = S.predict(s, yv, None, None, T, pred_m_v=10)
    mu, var = O.OracleModel("vif", x, y, t, th, nbr=nbr, Z=Z).predict(yv, T, 10)
    assert np.allclose(pr.mu, mu, rtol=1e-8, atol=1e-10) and np.allclose(pr.var, var, rtol=1e-8, atol=1e-10)
