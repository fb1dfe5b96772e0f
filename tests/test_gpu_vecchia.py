"""GPU parity: device exp / kernel / d_c + euclid search / Vecchia NLL+grad vs the oracle.

Mirrors the reference tests: test_covariance.cpp (kernel), test_neighbors.cpp
(searches == brute force, edge cases), test_approximations.cpp (Vecchia
exactness limits, gradients).  Bit-exact for integer/index work and the
kernel values; 1e-8 relative for the likelihood and gradient (north_star).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
T3 = (1.539, 6.193, 0.090, 3.37e-6, 0.831, 1.5, 0.999, 1.667)
RTOL = 1e-8


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _ds(S, x, y, t, yv=None, X=None):
    return S.SpaceTimeDataset(x, y, t, yv, X)


def test_exp_kat(S):
    # the device exp port must equal host glibc exp bit-for-bit
    rng = np.random.default_rng(1)
    xs = np.concatenate([-rng.random(4_000_000) * 50, -rng.random(1_000_000) * 745, -rng.random(500_000) * 1e-3,
                         rng.uniform(-1, 1, 500_000), -rng.uniform(700, 760, 200_000), rng.uniform(-1e-17, 1e-17, 1000),
                         [0.0, -0.0, -745.2, -708.4, 709.0, -1e-300]])
    dev = S.api.debug_exp(xs)
    host = O.exp_array(xs)
    mism = np.flatnonzero(dev.view(np.uint64) != host.view(np.uint64))
    assert len(mism) == 0, (len(mism), xs[mism[:5]])


def test_kernel_bit_exact(S):
    rng = np.random.default_rng(2)
    for th in (SEC4, T3, (0.1, 2.0, 1.3, 7.0, 0.7, 0.5, 0.9, 1.2), (0.1, 0.7, 0.2, 3.0, 0.3, 2.5, 0.1, 0.0)):
        scale = 1e6 if th[3] < 1e-3 else 1.0
        h = rng.random(2000) * scale * (0.1 if th[3] > 1 else 1.0)
        u = rng.integers(0, 30, 2000).astype(float)
        u[::7] = rng.random(len(u[::7])) * 10  # non-integral lags
        h[0] = 0.0
        cov, g = S.api.debug_kernel(th, h, u)
        ref = np.array([O.kernel_eval(th, a, b) for a, b in zip(h, u)])
        assert (cov.view(np.uint64) == ref.view(np.uint64)).all()
        gref = np.array([O.kernel_grad(th, a, b) for a, b in zip(h, u)])
        assert np.allclose(g, gref, rtol=1e-13, atol=1e-300)
    # frozen value of test_covariance.cpp:58-59
    cov, _ = S.api.debug_kernel(SEC4, [0.1], [1.0])
    assert cov[0] == pytest.approx(0.35267529426257880, rel=1e-12)


def _check_dc(S, x, y, t, th, m):
    ds = _ds(S, x, y, t)
    nb = S.correlation_neighbors(ds, th, m)
    idx, dist = nb.indices(), nb.distances()
    ref, rdist = O.dc_neighbors(x, y, t, th, m, with_dist=True)
    assert (idx == ref).all(), np.argwhere(idx != ref)[:5]
    ok = ~np.isnan(rdist)
    assert (dist[ok].view(np.uint64) == rdist[ok].view(np.uint64)).all()


def test_dc_search_reference_datasets(S):
    # test_neighbors.cpp:96-109 (n = 1000, m = 30, seed 17) and edge rows
    x, y, t, _, _ = O.test_dataset(0, 1000, 17)
    _check_dc(S, x, y, t, SEC4, 30)
    x, y, t, _, _ = O.test_dataset(0, 40, 13)
    ds = _ds(S, x, y, t)
    idx = S.correlation_neighbors(ds, SEC4, 10).indices()
    assert (idx[0] == -1).all()
    for i in range(1, 6):
        assert list(idx[i, :i]) == list(range(i)) and (idx[i, i:] == -1).all()


def test_dc_search_station_day(S):
    x, y, t, _ = S.synth.station_day(300, 12, theta=SEC4, seed=5)
    perm = O.order_observations(t, 5)
    x, y, t = x[perm], y[perm], t[perm]
    _check_dc(S, x, y, t, SEC4, 20)
    x, y, t, _ = S.synth.station_day(400, 9, box=(4.6e6, 2.9e6), theta=T3, seed=6)
    perm = O.order_observations(t, 6)
    _check_dc(S, x[perm], y[perm], t[perm], T3, 30)


def test_dc_search_unsorted_times(S):
    rng = np.random.default_rng(3)
    n = 500
    x, y, t = rng.random(n), rng.random(n), rng.integers(1, 6, n).astype(float)
    _check_dc(S, x, y, t, SEC4, 12)  # not time ordered: plain brute force path


def test_euclid_search(S):
    x, y, t, _, _ = O.test_dataset(0, 400, 31)
    ds = _ds(S, x, y, t)
    for ss, ts, m in ((0.3, 2.5, 12), (1.0, 1e12, 8), (0.05, 0.5, 10)):
        idx = S.euclidean_neighbors(ds, m, ss, ts).indices()
        assert (idx == O.euclid_neighbors(x, y, t, m, ss, ts)).all()
    n = 30
    ds = _ds(S, np.arange(n, dtype=float), np.zeros(n), np.ones(n))
    idx = S.euclidean_neighbors(ds, 5, 1.0, 1.0).indices()
    for i in range(6, n):
        assert list(idx[i]) == list(range(i - 5, i))
    with pytest.raises(S.ConfigError):
        S.euclidean_neighbors(ds, 5, 0.0, 1.0)


def _vecchia_pair(S, x, y, t, yv, th, nbr, X=None, beta=None):
    ds = _ds(S, x, y, t)
    nb = S.NeighborSets.from_sets(ds, nbr)
    s = S.build_vecchia(ds, th, nb, S.OBSERVATION)
    om = O.OracleModel("vecchia", x, y, t, th, nbr=nbr)
    return ds, nb, s, om


@pytest.mark.parametrize("m", [6, 20, 31])
def test_vecchia_nll_grad_parity(S, m):
    x, y, t, yv, X = O.test_dataset(1, 3000, 7, n_times=12, p=2)
    beta = np.array([0.3, -0.5])
    nbr = O.dc_neighbors(x, y, t, SEC4, m)
    ds, nb, s, om = _vecchia_pair(S, x, y, t, yv, SEC4, nbr)
    Dr, Ar = om.rows()
    assert np.allclose(s.D, Dr, rtol=1e-11, atol=0)
    assert np.allclose(s.A, Ar, rtol=1e-9, atol=1e-12)
    v = S.nll(s, yv, X, beta)
    assert v == pytest.approx(om.nll(yv, X, beta), rel=RTOL)
    g = S.nll_grad(s, yv, X, beta)
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert O.grad_close(g, gr, sc, RTOL), (g, gr, sc)
    v2, g2 = S.nll_and_grad(s, yv, X, beta)
    assert v2 == pytest.approx(v, rel=1e-12) and np.allclose(g2, g, rtol=1e-12, atol=1e-12 * np.abs(g).max())


def test_vecchia_eval_rebuild(S):
    x, y, t, yv, _ = O.test_dataset(1, 2000, 11, n_times=10)
    nbr = O.dc_neighbors(x, y, t, SEC4, 15)
    ds, nb, s, _ = _vecchia_pair(S, x, y, t, yv, SEC4, nbr)
    th2 = (0.05, 1.3, 0.7, 15.0, 0.5, 1.5, 0.6, 0.4)
    v, g = S.evaluate(s, th2, yv)
    om = O.OracleModel("vecchia", x, y, t, th2, nbr=nbr)
    assert v == pytest.approx(om.nll(yv), rel=RTOL)
    gr, sc = om.nll_grad_scale(yv)
    assert O.grad_close(g, gr, sc, RTOL), (g, gr, sc)
    assert np.allclose(s.D, om.rows()[0], rtol=1e-11)


def test_vecchia_full_conditioning_exactness(S):
    # test_approximations.cpp:97-116: full conditioning == dense likelihood (1e-8)
    n = 60
    x, y, t, yv, X = O.test_dataset(1, n, 7, n_times=6, p=2)
    th = (0.05,) + SEC4[1:]
    beta = np.array([0.4, -0.9])
    full = O.full_conditioning(n)
    ds, nb, s, om = _vecchia_pair(S, x, y, t, yv, th, full)
    ref = O.dense_nll(x, y, t, th, yv, X, beta)
    assert S.nll(s, yv, X, beta) == pytest.approx(ref, rel=1e-8)
    g = S.nll_grad(s, yv, X, beta)
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert O.grad_close(g, gr, sc), (g, gr, sc)


def test_vecchia_univariate_and_errors(S):
    th = SEC4
    ds = _ds(S, [0.5], [0.5], [1.0])
    nb = S.NeighborSets.from_sets(ds, np.full((1, 1), -1))
    s = S.build_vecchia(ds, th, nb, S.OBSERVATION)
    expect = 0.5 * math.log(2 * math.pi) + 0.5 * math.log(1.0 + 0.01)
    assert S.nll(s, [0.0]) == pytest.approx(expect, rel=1e-12)
    # two identical points, no nugget, latent: singular block (test_approximations.cpp:65-75)
    ds2 = _ds(S, [0.1, 0.1], [0.2, 0.2], [1.0, 1.0])
    nb2 = S.NeighborSets.from_sets(ds2, np.array([[-1], [0]]))
    with pytest.raises(S.NumericError):
        S.build_vecchia(ds2, (0.0,) + th[1:], nb2, S.LATENT)
    with pytest.raises(S.ConfigError):
        S.build_vecchia(ds2, (0.0, -1.0) + th[2:], nb2, S.LATENT)
    s_lat = S.build_vecchia(ds, th, nb, S.LATENT)
    with pytest.raises(S.NumericError):
        S.nll_grad(s_lat, [0.0])


def test_vecchia_noise_limit(S):
    # test_approximations.cpp:307-319
    x, y, t, yv, _ = O.test_dataset(1, 80, 19, n_times=8)
    th = (400.0,) + SEC4[1:]
    nbr = O.dc_neighbors(x, y, t, th, 5)
    ds, nb, s, _ = _vecchia_pair(S, x, y, t, yv, th, nbr)
    g = S.nll_grad(s, yv)
    expect = 80 / (2 * 400.0) - (yv @ yv) / (2 * 400.0 ** 2)
    assert g[0] == pytest.approx(expect, rel=5e-3)
