"""Neighbour sets wider than a warp (m_v > 32), against the oracle.

The reference's searches and structures take any m_v (neighbors.cpp:150-226, approximations.cpp:
42-111).  Here the searches keep lists of up to 4 slots per lane (m_v <= 128, search.cuh topl_*;
the d_r tile kernel's per-query lists grow to 32 LR shared-memory slots), and rows with k > 31
neighbours run the serial row kernel in every mode, including the VIF gradient's per-row pass.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
TH = (0.05, 1.2, 0.6, 15.0, 0.5, 1.5, 0.5, 0.3)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _bits(a, b):
    return (np.asarray(a).view(np.uint64) == np.asarray(b).view(np.uint64)).all()


@pytest.mark.parametrize("m", [33, 64, 65, 128])
def test_dc_search_wide(S, m):
    x, y, t, _, _ = O.test_dataset(0, 1500, 17)
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.correlation_neighbors(ds, SEC4, m)
    ref, rdist = O.dc_neighbors(x, y, t, SEC4, m, with_dist=True)
    assert (nb.indices() == ref).all(), np.argwhere(nb.indices() != ref)[:5]
    ok = ~np.isnan(rdist)
    assert _bits(nb.distances()[ok], rdist[ok])
    # the first rows hold every predecessor, ascending
    idx = nb.indices()
    for i in (1, 20, m):
        assert list(idx[i, :i]) == list(range(i)) and (idx[i, i:] == -1).all()


@pytest.mark.parametrize("m", [40, 100])
def test_euclid_search_wide(S, m):
    x, y, t, _, _ = O.test_dataset(0, 900, 31)
    ds = S.SpaceTimeDataset(x, y, t)
    idx = S.euclidean_neighbors(ds, m, 0.3, 2.5).indices()
    assert (idx == O.euclid_neighbors(x, y, t, m, 0.3, 2.5)).all()


@pytest.mark.parametrize("m", [45, 100])
def test_dr_search_wide(S, m):
    x, y, t, _, _ = O.test_dataset(0, 1200, 19)
    rng = np.random.default_rng(5)
    Z = np.column_stack([rng.random(25), rng.random(25), 1 + 9 * rng.random(25)])
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.residual_neighbors(ds, SEC4, S.InducingSet.from_points(Z), m)
    ref, rdist = O.dr_neighbors(x, y, t, SEC4, Z, m, with_dist=True)
    assert (nb.indices() == ref).all(), np.argwhere(nb.indices() != ref)[:5]
    ok = ~np.isnan(rdist)
    assert _bits(nb.distances()[ok], rdist[ok])


def test_search_limit(S):
    x, y, t, _, _ = O.test_dataset(0, 300, 3)
    ds = S.SpaceTimeDataset(x, y, t)
    with pytest.raises(S.ConfigError):
        S.correlation_neighbors(ds, SEC4, 129)


def test_vecchia_wide_nll_grad(S):
    x, y, t, yv, X = O.test_dataset(1, 1200, 7, n_times=10, p=1)
    beta = np.array([0.3])
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.correlation_neighbors(ds, TH, 40)
    nbr = O.dc_neighbors(x, y, t, TH, 40)
    assert (nb.indices() == nbr).all()
    s = S.build_vecchia(ds, TH, nb, S.OBSERVATION)
    om = O.OracleModel("vecchia", x, y, t, TH, nbr=nbr)
    assert S.nll(s, yv, X, beta) == pytest.approx(om.nll(yv, X, beta), rel=1e-8)
    g = S.nll_grad(s, yv, X, beta)
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert O.grad_close(g, gr, sc), (g, gr, sc)


def test_vif_wide_nll_grad(S):
    # VIF with m_v = 40: serial rows in build and in the gradient's per-row pass
    x, y, t, yv, X = O.test_dataset(1, 900, 41, n_times=8, p=1)
    beta = np.array([0.3])
    rng = np.random.default_rng(3)
    Z = np.column_stack([rng.random(24), rng.random(24), 1 + 7 * rng.random(24)])
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.InducingSet.from_points(Z)
    nb = S.residual_neighbors(ds, TH, ind, 40)
    nbr = O.dr_neighbors(x, y, t, TH, Z, 40)
    assert (nb.indices() == nbr).all()
    s = S.build_vif(ds, TH, ind, nb, S.OBSERVATION)
    om = O.OracleModel("vif", x, y, t, TH, nbr=nbr, Z=Z)
    assert S.nll(s, yv, X, beta) == pytest.approx(om.nll(yv, X, beta), rel=1e-8)
    g = S.nll_grad(s, yv, X, beta)
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert O.grad_close(g, gr, sc), (g, gr, sc)
    v2, g2 = S.evaluate(s, TH, yv, X, beta)
    assert v2 == pytest.approx(om.nll(yv, X, beta), rel=1e-8)
    assert O.grad_close(g2, gr, sc)
