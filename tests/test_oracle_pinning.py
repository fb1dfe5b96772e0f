"""Pin the CPU oracle against the reference's own known-answer tests.

The reference cannot be compiled here (Eigen3 and vendor/ are absent), so the
oracle is pinned by re-running the reference suite's assertions on it, with the
reference's datasets regenerated from the same std::mt19937_64 streams.
Each test cites the reference test it restates (proj/tests/...).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)  # test_covariance.cpp:14-17
T3 = (1.539, 6.193, 0.090, 3.37e-6, 0.831, 1.5, 0.999, 1.667)


def _params_with(**kw):
    names = ("sigma2", "sigma1_2", "a", "c", "alpha", "nu", "beta", "delta")
    d = dict(zip(names, SEC4))
    d.update(kw)
    return tuple(d[k] for k in names)


# --- covariance (test_covariance.cpp) ---------------------------------------

def test_frozen_kernel_value():
    # test_covariance.cpp:51-60
    assert O.kernel_eval(SEC4, 0.0, 0.0) == pytest.approx(1.0, rel=1e-15)
    v = O.kernel_eval(SEC4, 0.1, 1.0)
    assert v == pytest.approx(0.35267529426257880, rel=1e-12)


def test_separable_limit():
    # test_covariance.cpp:62-77 (beta = 0 factorizes)
    th = (0.0, 1.3, 0.5, 20.0, 0.4, 1.5, 0.0, 0.2)
    rng = np.random.default_rng(7)
    for _ in range(50):
        h, u = rng.random() * 0.5, rng.random() * 10
        temporal = (0.5 * u ** (2 * 0.4) + 1.0) ** (-0.2)
        x = 20.0 * h
        spatial = (1 + x) * math.exp(-x) if x > 0 else 1.0
        assert O.kernel_eval(th, h, u) == pytest.approx(1.3 * temporal * spatial, rel=1e-13)



def test_kernel_vs_high_precision():
    # test_covariance.cpp:79-93 long-double oracle; here a decimal re-evaluation
    from decimal import Decimal, getcontext
    getcontext().prec = 40

    def dexp(x):
        return Decimal(x).exp()

    def dpow(b, e):
        return (Decimal(b).ln() * Decimal(e)).exp()

    rng = np.random.default_rng(11)
    for _ in range(200):
        nu = [0.5, 1.5, 2.5][rng.integers(3)]
        th = (0.001 + rng.random(), 0.2 + 2 * rng.random(), 0.05 + 2 * rng.random(), 0.5 + 30 * rng.random(),
              0.05 + 0.9 * rng.random(), nu, rng.random(), 2 * rng.random())
        h, u = 2 * rng.random(), 5 * rng.random()
        s2, s1, a, c, alpha, nu, beta, delta = th
        T = Decimal(a) * dpow(u, 2 * alpha) + 1 if u > 0 else Decimal(1)
        x = Decimal(c) * Decimal(h) / (dpow(T, beta / 2) if T != 1 else Decimal(1))
        if x == 0:
            M = Decimal(1)
        elif nu == 0.5:
            M = dexp(-x)
        elif nu == 1.5:
            M = (1 + x) * dexp(-x)
        else:
            M = (1 + x + x * x / 3) * dexp(-x)
        ref = float(Decimal(s1) * (dpow(T, -(delta + beta)) if T != 1 else 1) * M)
        assert O.kernel_eval(th, h, u) == pytest.approx(ref, rel=1e-12, abs=1e-300)


def test_gradient_fd():
    # test_covariance.cpp:129-161
    rng = np.random.default_rng(23)
    for k in range(100):
        th = [0.001 + rng.random(), 0.2 + 2 * rng.random(), 0.05 + 2 * rng.random(), 0.5 + 30 * rng.random(),
              0.05 + 0.9 * rng.random(), [0.5, 1.5, 2.5][k % 3], rng.random(), 2 * rng.random()]
        h = math.hypot(rng.random() - rng.random(), rng.random() - rng.random())
        u = abs(3 * rng.random() - 3 * rng.random())
        g = O.kernel_grad(th, h, u)
        for q, field in enumerate([1, 2, 3, 4, 6, 7]):
            base = th[field]
            step = 1e-6 * max(abs(base), 1e-2)
            hi = list(th); hi[field] = base + step
            lo = list(th); lo[field] = base - step
            fd = (O.kernel_eval(hi, h, u) - O.kernel_eval(lo, h, u)) / (2 * step)
            scale = max(abs(fd), abs(g[q]), 1e-8)
            assert abs(g[q] - fd) / scale < 1e-5


def test_temporal_components_vanish_at_zero_lag():
    g = O.kernel_grad(SEC4, math.hypot(0.4, 0.2), 0.0)
    assert g[1] == 0.0 and g[3] == 0.0 and g[4] == 0.0 and g[5] == 0.0


def test_general_nu_rejects_gradient():
    th = _params_with(nu=1.0)
    with pytest.raises(O.OracleError) as e:
        O.kernel_grad(th, 0.1, 1.0)
    assert e.value.kind == "NumericError"


def test_dc_metric_properties():
    # test_covariance.cpp:170-185
    p = (0.1, 0.9, 3.0)
    assert O.dc_pair(SEC4, p, p) == 0.0
    far = (0.1 + 50.0 / 20.0, 0.9, 3.0)
    assert O.dc_pair(SEC4, p, far) == pytest.approx(1.0, rel=1e-12)


def test_effective_ranges():
    # test_covariance.cpp:223-249
    tr, sr = O.effective_ranges((0.0, 6.193, 0.090, 3.37e-6, 0.831, 1.5, 0.999, 1.667))
    assert tr == pytest.approx(6.6086, rel=1e-3)
    assert sr / 1000 == pytest.approx(1408.0, rel=5.0 / 1408.0)
    tr, sr = O.effective_ranges((0.0, 0.9, 1.0, 50.0, 0.6, 1.0, 0.9, 0.1))
    assert abs(tr - 11.63) < 0.01 and abs(sr - 0.08) < 0.001
    tr, sr = O.effective_ranges((0.0, 18.286, 0.230, 1.08e-6, 0.860, 0.5, 0.265, 2.353))
    assert abs(tr - 3.7) < 0.05 and abs(sr / 1000 - 2774.0) < 5.0
    tr, _ = O.effective_ranges((0.0, 1.0, 1.0, 1.0, 0.5, 1.5, 0.0, 0.0))
    assert math.isinf(tr)


def test_config_validation():
    with pytest.raises(O.OracleError) as e:
        O.kernel_grad((0.0, -1.0, 1, 1, 0.5, 1.5, 0.5, 0.5), 0.1, 1.0)
    assert e.value.kind == "ConfigError"


# --- neighbours (test_neighbors.cpp) -----------------------------------------

def _brute(metric, i, m):
    cand = sorted((metric(i, j), j) for j in range(i))
    return sorted(j for _, j in cand[: min(m, i)])


def test_knn_edge_behavior():
    # test_neighbors.cpp:81-94: the first rows take all predecessors
    x, y, t, _, _ = O.test_dataset(0, 40, 13)
    nb = O.dc_neighbors(x, y, t, SEC4, 10)
    assert (nb[0] == -1).all()
    for i in range(1, 6):
        assert list(nb[i, :i]) == list(range(i))


def test_dc_knn_equals_brute_force():
    # test_neighbors.cpp:96-109 (n = 1000, m = 30, seed 17): pruned scan == brute force
    x, y, t, _, _ = O.test_dataset(0, 1000, 17)
    pruned = O.dc_neighbors(x, y, t, SEC4, 30)
    O.set_prune(False)
    try:
        plain = O.dc_neighbors(x, y, t, SEC4, 30)
    finally:
        O.set_prune(True)
    assert (pruned == plain).all()
    metric = lambda i, j: O.dc_pair(SEC4, (x[i], y[i], t[i]), (x[j], y[j], t[j]))
    for i in [1, 2, 29, 30, 31, 100, 517, 999]:
        got = [v for v in pruned[i] if v >= 0]
        assert got == _brute(metric, i, 30)


def test_dr_knn_brute_force_and_degenerate():
    # test_neighbors.cpp:111-131 and 222-238
    x, y, t, _, _ = O.test_dataset(0, 300, 19)
    rng = np.random.default_rng(5)
    Z = np.column_stack([rng.random(25), rng.random(25), 1 + 9 * rng.random(25)])
    nb, d = O.dr_neighbors(x, y, t, SEC4, Z, 20, with_dist=True)
    for i in range(300):
        k = min(20, i)
        assert (nb[i, :k] >= 0).all() and (nb[i, k:] == -1).all()
        assert (np.diff(nb[i, :k]) > 0).all()
        assert (np.diff(d[i, :k]) >= 0).all()
    # degenerate: a data point on an inducing location sits at distance 1
    pts = np.array([[0.5, 0.5, 1.0], [0.2, 0.8, 1.0], [0.9, 0.1, 2.0]])
    nb, d, W, resid = O.dr_neighbors(pts[:, 0], pts[:, 1], pts[:, 2], SEC4, pts[:1], 2, with_dist=True, with_w=True)
    assert resid[0] <= 1e-7 and resid[1] > 1e-7
    assert d[1, 0] == 1.0  # d(1, 0) with 0 degenerate
    assert d[2, 0] < 1.0 and d[2, 1] == 1.0


def test_dr_empty_inducing_equals_dc():
    x, y, t, _, _ = O.test_dataset(0, 200, 3)
    a = O.dc_neighbors(x, y, t, SEC4, 8)
    b = O.dr_neighbors(x, y, t, SEC4, np.zeros((0, 3)), 8)
    assert (a == b).all()


def test_euclidean_neighbors():
    # test_neighbors.cpp:148-196
    n = 30
    nb = O.euclid_neighbors(np.arange(n, dtype=float), np.zeros(n), np.ones(n), 5, 1.0, 1.0)
    for i in range(6, n):
        assert list(nb[i]) == list(range(i - 5, i))
    x, y, t, _, _ = O.test_dataset(0, 400, 31)
    ss, ts = 0.3, 2.5
    nb = O.euclid_neighbors(x, y, t, 12, ss, ts)

    def metric(i, j):
        dx, dy, dt = (x[i] - x[j]) / ss, (y[i] - y[j]) / ss, (t[i] - t[j]) / ts
        return dx * dx + dy * dy + dt * dt
    for i in range(0, 400, 7):
        assert [v for v in nb[i] if v >= 0] == _brute(metric, i, 12)
    with pytest.raises(O.OracleError):
        O.euclid_neighbors(x, y, t, 5, 0.0, 1.0)


# --- inducing (test_inducing.cpp) ---------------------------------------------

def test_kmeanspp_cases():
    pts = np.array([[0, 0], [1, 0], [0, 1], [1, 1]], dtype=float)
    c = O.kmeanspp(pts, 4, 7)
    assert sorted(map(tuple, c)) == sorted(map(tuple, pts))
    c = O.kmeanspp(np.array([[1.0], [2], [3], [4], [10]]), 1, 3)
    assert c[0, 0] == pytest.approx(4.0)
    with pytest.raises(O.OracleError) as e:
        O.kmeanspp(np.array([[1.0], [1], [2], [2]]), 3, 1)
    assert e.value.kind == "DataError"


def test_kmeanspp_two_clusters_and_determinism():
    rng = np.random.default_rng(11)
    pts = np.vstack([rng.normal(0, 0.05, (20, 2)), 10 + rng.normal(0, 0.05, (20, 2))])
    for seed in range(1, 6):
        c = O.kmeanspp(pts, 2, seed)
        d0 = min(np.linalg.norm(c[0]), np.linalg.norm(c[1]))
        d1 = min(np.linalg.norm(c[0] - 10), np.linalg.norm(c[1] - 10))
        assert d0 < 0.1 and d1 < 0.1
    assert (O.kmeanspp(pts, 5, 99) == O.kmeanspp(pts, 5, 99)).all()


def test_sts_counts():
    # test_inducing.cpp:101-127
    x, y, t, _, _ = O.test_dataset(2, 500, 5, n_times=20)
    Z, ms, mt = O.sts_kmeanspp(x, y, t, 500, 1)
    assert (ms, mt, len(Z)) == (112, 4, 448)
    x, y, t, _, _ = O.test_dataset(2, 30, 7, n_times=5)
    Z, ms, mt = O.sts_kmeanspp(x, y, t, 1, 2)
    assert (ms, mt, len(Z)) == (1, 1, 1)
    x, y, t, _, _ = O.test_dataset(2, 40, 9, n_times=1)
    Z, ms, mt = O.sts_kmeanspp(x, y, t, 12, 3)
    assert mt == 1 and len(Z) == ms and (Z[:, 2] == 1.0).all()


def test_sts_product_grid():
    x, y, t, _, _ = O.test_dataset(2, 80, 15, n_times=12)
    Z, ms, mt = O.sts_kmeanspp(x, y, t, 60, 4)
    assert len(Z) == ms * mt
    assert len({tuple(r) for r in Z}) == len(Z)
    assert abs(len(Z) - 60) <= 30
    Z2, _, _ = O.sts_kmeanspp(x, y, t, 60, 4)
    assert (Z == Z2).all()


def test_joint_kmeanspp():
    x, y, t, _, _ = O.test_dataset(2, 60, 23, n_times=6)
    Z = O.joint_kmeanspp(x, y, t, 25, 0.5, 2.0, 5)
    assert len(Z) == 25
    with pytest.raises(O.OracleError):
        O.joint_kmeanspp(x, y, t, 25, 0.0, 2.0, 5)


# --- approximations (test_approximations.cpp) ----------------------------------

def _theta(sigma2):
    return _params_with(sigma2=sigma2)


def test_exactness_limits_vs_dense():
    # test_approximations.cpp:97-142
    n = 60
    x, y, t, yv, X = O.test_dataset(1, n, 7, n_times=6, p=2)
    th = _theta(0.05)
    beta = np.array([0.4, -0.9])
    ref = O.dense_nll(x, y, t, th, yv, X, beta)
    full = O.full_conditioning(n)
    v = O.OracleModel("vecchia", x, y, t, th, nbr=full).nll(yv, X, beta)
    assert v == pytest.approx(ref, rel=1e-8)
    allpts = np.column_stack([x, y, t])
    f = O.OracleModel("fitc", x, y, t, th, Z=allpts).nll(yv, X, beta)
    assert f == pytest.approx(ref, rel=1e-6)
    small = allpts[[0, 10, 20]]
    w = O.OracleModel("vif", x, y, t, th, nbr=full, Z=small).nll(yv, X, beta)
    assert w == pytest.approx(ref, rel=1e-8)
    one = O.OracleModel("vecchia", [0.5], [0.5], [1.0], th, nbr=np.full((1, 1), -1))
    assert one.nll([0.0]) == pytest.approx(0.5 * math.log(2 * math.pi) + 0.5 * math.log(1.05), rel=1e-12)


def test_fitc_structural_properties():
    # test_approximations.cpp:144-170
    x, y, t, yv, _ = O.test_dataset(1, 80, 9, n_times=8)
    th = _theta(0.3)
    Z = np.column_stack([x, y, t])[[6 * j for j in range(12)]]
    d = O.OracleModel("fitc", x, y, t, th, Z=Z).fitc_diag()
    assert (d >= 0).all()
    far = O.OracleModel("fitc", x[:30], y[:30], t[:30], _theta(0.5), Z=[[500.0, 500.0, 900.0]]).fitc_diag()
    assert np.allclose(far, 1.0, rtol=1e-10)


def test_vif_empty_equals_vecchia():
    # test_approximations.cpp:172-188
    x, y, t, yv, _ = O.test_dataset(1, 70, 13, n_times=8)
    th = _theta(0.1)
    nb = O.dc_neighbors(x, y, t, th, 8)
    for pol in ("latent", "observation"):
        Dv, Av = O.OracleModel("vif", x, y, t, th, nbr=nb, policy=pol).rows()
        Dw, Aw = O.OracleModel("vecchia", x, y, t, th, nbr=nb, policy=pol).rows()
        assert (Dv == Dw).all() and (Av == Aw).all()
    a = O.OracleModel("vif", x, y, t, th, nbr=nb).nll(yv)
    b = O.OracleModel("vecchia", x, y, t, th, nbr=nb).nll(yv)
    assert a == pytest.approx(b, rel=1e-14)


def _fd_check(make, th, yv, X, beta, tol=2e-4):
    g = make(th).nll_grad(yv, X, beta)
    for k in range(7):
        base = th[k if k < 5 else k + 1]
        h = 1e-6 * max(abs(base), 1e-2)
        idx = k if k < 5 else k + 1
        hi = list(th); hi[idx] = base + h
        lo = list(th); lo[idx] = base - h
        fd = (make(tuple(hi)).nll(yv, X, beta) - make(tuple(lo)).nll(yv, X, beta)) / (2 * h)
        scale = max(abs(fd), abs(g[k]), 1e-6)
        assert abs(g[k] - fd) / scale < tol, (k, g[k], fd)


def _rand_theta(rng, lo_s2):
    return (lo_s2 + 0.3 * rng.random(), 0.5 + rng.random(), 0.3 + rng.random(), 5 + 20 * rng.random(),
            0.2 + 0.6 * rng.random(), 1.5, rng.random(), rng.random())


def test_gradients_match_fd():
    # test_approximations.cpp:213-305
    n = 60
    x, y, t, yv, X = O.test_dataset(1, n, 17, n_times=6, p=1)
    beta = np.array([0.7])
    rng = np.random.default_rng(3)
    nb = O.dc_neighbors(x, y, t, SEC4, 6)
    for _ in range(2):
        th = _rand_theta(rng, 0.02)
        _fd_check(lambda th_: O.OracleModel("vecchia", x, y, t, th_, nbr=nb), th, yv, X, beta)
    allpts = np.column_stack([x, y, t])
    Zf = allpts[[5 * j for j in range(10)]]
    for _ in range(2):
        th = _rand_theta(rng, 0.05)
        _fd_check(lambda th_: O.OracleModel("fitc", x, y, t, th_, Z=Zf), th, yv, X, beta)
    Zv = allpts[[7 * j for j in range(8)]]
    nbr = O.dr_neighbors(x, y, t, SEC4, Zv, 6)
    for _ in range(2):
        th = _rand_theta(rng, 0.05)
        _fd_check(lambda th_: O.OracleModel("vif", x, y, t, th_, nbr=nbr, Z=Zv), th, yv, X, beta)


def test_nugget_gradient_limit():
    # test_approximations.cpp:307-319
    x, y, t, yv, _ = O.test_dataset(1, 80, 19, n_times=8)
    th = _theta(400.0)
    nb = O.dc_neighbors(x, y, t, th, 5)
    g = O.OracleModel("vecchia", x, y, t, th, nbr=nb).nll_grad(yv)
    expect = 80 / (2 * 400.0) - (yv @ yv) / (2 * 400.0 ** 2)
    assert g[0] == pytest.approx(expect, rel=5e-3)


def test_predictions_vs_kriging():
    # test_approximations.cpp:321-368
    n = 80
    x, y, t, yv, _ = O.test_dataset(1, n, 21, n_times=6)
    th = _theta(0.05)
    rng = np.random.default_rng(5)
    T = np.column_stack([rng.random(12), rng.random(12), 1 + 8 * rng.random(12)])
    mu_ref, var_ref = O.dense_predict(x, y, t, th, yv, T)
    full = O.full_conditioning(n)
    mu, var = O.OracleModel("vecchia", x, y, t, th, nbr=full).predict(yv, T, n)
    assert np.allclose(mu, mu_ref, rtol=1e-6, atol=1e-9) and np.allclose(var, var_ref, rtol=1e-6)
    allpts = np.column_stack([x, y, t])
    mu, var = O.OracleModel("fitc", x, y, t, th, Z=allpts).predict(yv, T, 0)
    assert np.allclose(mu, mu_ref, rtol=1e-5, atol=1e-8) and np.allclose(var, var_ref, rtol=1e-5, atol=1e-5)
    mu, var = O.OracleModel("vif", x, y, t, th, nbr=full, Z=allpts[[3, 30, 60]]).predict(yv, T, n)
    assert np.allclose(mu, mu_ref, rtol=1e-6, atol=1e-9) and np.allclose(var, var_ref, rtol=1e-6)


def test_prediction_limit_cases_and_bounds():
    # test_approximations.cpp:370-428
    x, y, t, yv, _ = O.test_dataset(1, 50, 23, n_times=8)
    th = _theta(1e-12)
    nb = O.dc_neighbors(x, y, t, th, 10)
    m = O.OracleModel("vecchia", x, y, t, th, nbr=nb)
    mu, var = m.predict(yv, [[x[20], y[20], t[20]]], 10)
    assert mu[0] == pytest.approx(yv[20], rel=1e-5) and var[0] < 1e-8
    th2 = _theta(0.25)
    mu, var = O.OracleModel("vecchia", x, y, t, th2, nbr=nb).predict(yv, [[300.0, 300.0, 500.0]], 10)
    assert abs(mu[0]) < 1e-10 and var[0] == pytest.approx(1.25, rel=1e-10)
    x, y, t, yv, _ = O.test_dataset(1, 150, 25, n_times=8)
    th = _theta(0.1)
    rng = np.random.default_rng(7)
    T = np.column_stack([rng.random(40), rng.random(40), 9 * rng.random(40) + 1])
    nb = O.dc_neighbors(x, y, t, th, 10)
    _, var = O.OracleModel("vecchia", x, y, t, th, nbr=nb).predict(yv, T, 10)
    assert (var >= 0).all() and (var <= 1.1 + 1e-8).all()
    Z = np.column_stack([x, y, t])[[11 * j for j in range(10)]]
    rn = O.dr_neighbors(x, y, t, th, Z, 10)
    _, var = O.OracleModel("vif", x, y, t, th, nbr=rn, Z=Z).predict(yv, T, 10)
    assert (var >= 0).all() and (var <= 1.1 + 1e-8).all()


def test_gls_vs_dense():
    # test_approximations.cpp:444-455 (dense GLS via numpy on the dense Gram)
    n = 60
    x, y, t, yv, X = O.test_dataset(1, n, 29, n_times=6, p=2)
    th = _theta(0.15)
    b = O.OracleModel("vecchia", x, y, t, th, nbr=O.full_conditioning(n)).gls_beta(yv, X)
    G = np.array([[O.kernel_eval(th, math.hypot(x[i] - x[j], y[i] - y[j]), abs(t[i] - t[j])) for j in range(n)]
                  for i in range(n)]) + 0.15 * np.eye(n)
    SX = np.linalg.solve(G, X)
    ref = np.linalg.solve(X.T @ SX, SX.T @ yv)
    assert np.abs(b - ref).max() < 1e-8


def test_singular_latent_block_raises():
    # test_approximations.cpp:65-75
    th = _theta(0.0)
    m = O.OracleModel("vecchia", [0.1, 0.1], [0.2, 0.2], [1.0, 1.0], th, nbr=np.array([[-1], [0]]), policy="latent")
    with pytest.raises(O.OracleError) as e:
        m.rows()
    assert e.value.kind == "NumericError"


def test_ordering_properties():
    # dataset.cpp:81-114: stable time sort, shuffles only inside equal-t blocks
    rng = np.random.default_rng(1)
    t = rng.integers(1, 6, 300).astype(float)
    perm = O.order_observations(t, 42)
    assert sorted(perm) == list(range(300))
    assert (np.diff(t[perm]) >= 0).all()
    assert (O.order_observations(t, 42) == perm).all()
    assert not (O.order_observations(t, 43) == perm).all()


@pytest.mark.parametrize("kind", ["fitc", "vif"])
def test_blas_mode_matches_sequential(kind):
    """The oracle's BLAS timing mode (dense n x M^2 contractions on OpenBLAS) equals the sequential
    restatement up to rounding: NLL 1e-12 relative, gradient 1e-12 of the per-component scale."""
    if O.openblas_path() is None:
        pytest.skip("no scipy OpenBLAS in this image")
    x, y, t, yv, _ = O.test_dataset(1, 1200, 5, n_times=6)
    th = (0.05, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
    nb = O.dc_neighbors(x, y, t, th, 12) if kind == "vif" else None
    Z = np.column_stack([x, y, t])[::17]
    res = []
    try:
        for mode in (False, True):
            O.set_blas(mode, 4)
            om = O.OracleModel(kind, x, y, t, th, nbr=nb, Z=Z)
            res.append((om.nll(yv),) + om.nll_grad_scale(yv))
    finally:
        O.set_blas(False)
    (v0, g0, sc), (v1, g1, _) = res
    assert v1 == pytest.approx(v0, rel=1e-12)
    assert (np.abs(g1 - g0) <= 1e-12 * sc).all()


# ---- latent policy / Laplace / ZC-PTN (restating test_laplace.cpp and the latent-policy limits) ----
LATENT = (0.0, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)  # test_laplace.cpp:14-16


def _tiny(n, seed=404):
    rng = np.random.default_rng(seed)
    x, y = rng.random(n), rng.random(n)
    t = 1.0 + np.arange(n) % 3
    perm = O.order_observations(t, 1)
    return x[perm], y[perm], t[perm]


def test_normal_tail_helpers():  # test_laplace.cpp:44-53
    assert O.normal_tail(0.0)[1] == pytest.approx(math.log(0.5), rel=1e-12)
    assert O.normal_tail(1.96)[0] == pytest.approx(0.9750021, rel=1e-6)
    assert O.normal_tail(-7.999999)[1] == pytest.approx(O.normal_tail(-8.000001)[1], rel=1e-6)
    assert O.normal_tail(-7.999999)[2] == pytest.approx(O.normal_tail(-8.000001)[2], rel=1e-6)
    assert math.isfinite(O.normal_tail(-40.0)[1])
    assert O.normal_tail(-40.0)[2] == pytest.approx(40.0, rel=1e-2)


def test_zcptn_branches_and_derivatives():  # test_laplace.cpp:55-142
    assert O.zcptn(0.0, 0.0, 1.0, 1.0)[0] == pytest.approx(math.log(0.5), rel=1e-12)
    assert O.zcptn(1.0, 1.0, 1.0, 1.0)[0] == pytest.approx(-0.5 * math.log(2 * math.pi), rel=1e-12)
    with pytest.raises(O.OracleError):
        O.zcptn(-0.5, 0.0, 1.0, 1.0)
    d1 = O.zcptn(0.0, 0.0, 2.0, 1.0)[1]
    assert d1 == pytest.approx(-2.0 * math.exp(-0.5 * math.log(2 * math.pi)) / 2.0, rel=1e-12)
    assert O.zcptn(2.3, 0.4, 1.7, 1.0)[2] == pytest.approx(-1.0 / 1.7 ** 2, rel=1e-12)
    rng = np.random.default_rng(31)
    for _ in range(200):
        sig, lam = 0.3 + 2.0 * rng.random(), 0.4 + 2.0 * rng.random()
        yy = 0.0 if rng.random() < 0.3 else 3.0 * rng.random()
        mu = -2.0 + 4.0 * rng.random()
        _, d1, d2 = O.zcptn(yy, mu, sig, lam)
        h1, h2 = 1e-6, 2e-4
        fd1 = (O.zcptn(yy, mu + h1, sig, lam)[0] - O.zcptn(yy, mu - h1, sig, lam)[0]) / (2 * h1)
        fd2 = (O.zcptn(yy, mu + h2, sig, lam)[0] - 2 * O.zcptn(yy, mu, sig, lam)[0]
               + O.zcptn(yy, mu - h2, sig, lam)[0]) / h2 ** 2
        assert d1 == pytest.approx(fd1, rel=1e-6, abs=1e-8)
        assert d2 == pytest.approx(fd2, rel=1e-5, abs=1e-6)
        assert d2 <= 0.0


def test_latent_gaussian_nll_full_conditioning_is_exact():
    """Latent-policy Vecchia at full conditioning through the Laplace algebra equals the dense GP
    (approximations.cpp:320-334 with w = 1 / sigma^2)."""
    x, y, t = _tiny(40)
    yv = np.sin(7 * x) + y
    th = (0.3,) + LATENT[1:]
    om = O.OracleModel("vecchia", x, y, t, th, nbr=O.full_conditioning(len(x)), policy="latent")
    assert om.nll(yv) == pytest.approx(O.dense_nll(x, y, t, th, yv), rel=1e-10)


@pytest.mark.parametrize("kind", ["vecchia", "fitc", "vif"])
def test_laplace_exact_in_gaussian_case(kind):
    """test_laplace.cpp:144-192: lambda = 1 and strictly positive data make the ZC-PTN model Gaussian with
    noise sigma^2, so the Laplace marginal equals the Gaussian marginal."""
    x, y, t = _tiny(8)
    yv = np.array([3.1, 2.4, 4.0, 2.9, 3.3, 2.2, 3.8, 2.6])
    sig = 0.9
    th_obs = (sig * sig,) + LATENT[1:]
    full = O.full_conditioning(len(x))
    P = np.column_stack([x, y, t])
    if kind == "vecchia":
        om = O.OracleModel("vecchia", x, y, t, LATENT, nbr=full, policy="latent")
        ref = O.dense_nll(x, y, t, th_obs, yv)
    elif kind == "fitc":
        Z = P[[0, 3, 6]]
        om = O.OracleModel("fitc", x, y, t, LATENT, Z=Z)
        ref = O.OracleModel("fitc", x, y, t, th_obs, Z=Z).nll(yv)
    else:
        Z = P[[1, 4]]
        om = O.OracleModel("vif", x, y, t, LATENT, nbr=full, Z=Z, policy="latent")
        ref = O.dense_nll(x, y, t, th_obs, yv)
    v, st = O.laplace_marginal(om, yv, sig, 1.0)
    assert v == pytest.approx(ref, rel=1e-8)
