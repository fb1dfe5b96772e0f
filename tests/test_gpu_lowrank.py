"""GPU parity for the low-rank structures (FITC, VIF) against the oracle.

Restates test_approximations.cpp:97-188 (exactness limits, FITC properties,
VIF(empty) == Vecchia) and adds differential NLL/gradient parity at 1e-8.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _close(a, b, rtol):
    b = np.asarray(b)
    return np.allclose(a, b, rtol=rtol, atol=rtol * np.abs(b).max())


def _rand_inducing(n_ind, seed, tmax):
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.random(n_ind), rng.random(n_ind), 1 + (tmax - 1) * rng.random(n_ind)])


@pytest.mark.parametrize("m", [6, 20])
def test_vif_nll_grad_parity(S, m):
    x, y, t, yv, X = O.test_dataset(1, 2000, 41, n_times=10, p=1)
    beta = np.array([0.3])
    th = (0.05, 1.2, 0.6, 15.0, 0.5, 1.5, 0.5, 0.3)
    Z = _rand_inducing(24, 3, 10)
    nbr = O.dr_neighbors(x, y, t, th, Z, m)
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.NeighborSets.from_sets(ds, nbr, S.api.METRIC_DR)
    ind = S.InducingSet.from_points(Z)
    s = S.build_vif(ds, th, ind, nb, S.OBSERVATION)
    om = O.OracleModel("vif", x, y, t, th, nbr=nbr, Z=Z)
    Dr, Ar = om.rows()
    assert np.allclose(s.D, Dr, rtol=1e-10)
    v = S.nll(s, yv, X, beta)
    assert v == pytest.approx(om.nll(yv, X, beta), rel=1e-8)
    g = S.nll_grad(s, yv, X, beta)
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert O.grad_close(g, gr, sc), (g, gr, sc)
    v2, g2 = S.evaluate(s, th, yv, X, beta)
    assert v2 == pytest.approx(v, rel=1e-12) and _close(g2, g, 1e-11)


def test_vif_integral_inducing_times_snap(S):
    # inducing times on (and within 1e-9 of) integer days exercise the lag-table snap rule
    x, y, t, yv, _ = O.test_dataset(1, 800, 43, n_times=8)
    th = SEC4
    Z = _rand_inducing(12, 5, 8)
    Z[:6, 2] = np.round(Z[:6, 2])
    Z[6:9, 2] = np.round(Z[6:9, 2]) + 3e-10
    nbr = O.dr_neighbors(x, y, t, th, Z, 8)
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_vif(ds, th, S.InducingSet.from_points(Z), S.NeighborSets.from_sets(ds, nbr), S.OBSERVATION)
    om = O.OracleModel("vif", x, y, t, th, nbr=nbr, Z=Z)
    assert S.nll(s, yv) == pytest.approx(om.nll(yv), rel=1e-8)
    gr, sc = om.nll_grad_scale(yv)
    assert O.grad_close(S.nll_grad(s, yv), gr, sc)


def test_vif_empty_equals_vecchia(S):
    # test_approximations.cpp:172-188: bit-identical B and D
    x, y, t, yv, _ = O.test_dataset(1, 70, 13, n_times=8)
    th = (0.1,) + SEC4[1:]
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.correlation_neighbors(ds, th, 8)
    empty = S.InducingSet.from_points(np.zeros((0, 3)))
    for pol in (S.LATENT, S.OBSERVATION):
        v = S.build_vif(ds, th, empty, nb, pol)
        w = S.build_vecchia(ds, th, nb, pol)
        assert (v.D == w.D).all() and (v.A == w.A).all()
    vo = S.build_vif(ds, th, empty, nb, S.OBSERVATION)
    wo = S.build_vecchia(ds, th, nb, S.OBSERVATION)
    assert S.nll(vo, yv) == pytest.approx(S.nll(wo, yv), rel=1e-14)


def test_exactness_limits(S):
    # test_approximations.cpp:97-142 (VIF full residual conditioning 1e-8, FITC all points 1e-6)
    n = 60
    x, y, t, yv, X = O.test_dataset(1, n, 7, n_times=6, p=2)
    th = (0.05,) + SEC4[1:]
    beta = np.array([0.4, -0.9])
    ref = O.dense_nll(x, y, t, th, yv, X, beta)
    ds = S.SpaceTimeDataset(x, y, t)
    full = S.NeighborSets.from_sets(ds, O.full_conditioning(n))
    P = np.column_stack([x, y, t])
    s = S.build_vif(ds, th, S.InducingSet.from_points(P[[0, 10, 20]]), full, S.OBSERVATION)
    assert S.nll(s, yv, X, beta) == pytest.approx(ref, rel=1e-8)
    f = S.build_fitc(ds, th, S.InducingSet.from_points(P))
    assert S.nll(f, yv, X, beta) == pytest.approx(ref, rel=1e-6)


def test_fitc_nll_grad_parity(S):
    x, y, t, yv, X = O.test_dataset(1, 1500, 47, n_times=8, p=1)
    beta = np.array([-0.2])
    th = (0.2, 1.1, 0.8, 12.0, 0.6, 1.5, 0.3, 0.5)
    Z = _rand_inducing(40, 9, 8)
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_fitc(ds, th, S.InducingSet.from_points(Z))
    om = O.OracleModel("fitc", x, y, t, th, Z=Z)
    assert np.allclose(s.fitc_diag, om.fitc_diag(), rtol=1e-9, atol=1e-12)
    assert S.nll(s, yv, X, beta) == pytest.approx(om.nll(yv, X, beta), rel=1e-8)
    g = S.nll_grad(s, yv, X, beta)
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert O.grad_close(g, gr, sc), (g, gr, sc)


def test_fitc_structural(S):
    # test_approximations.cpp:144-170
    x, y, t, yv, _ = O.test_dataset(1, 30, 11, n_times=8)
    ds = S.SpaceTimeDataset(x, y, t)
    s = S.build_fitc(ds, (0.5,) + SEC4[1:], S.InducingSet.from_points([[500.0, 500.0, 900.0]]))
    assert np.allclose(s.fitc_diag, 1.0, rtol=1e-10)
    P = np.column_stack([x, y, t])
    f = S.build_fitc(ds, (0.3,) + SEC4[1:], S.InducingSet.from_points(P[::3]))
    assert (f.fitc_diag >= 0).all()
