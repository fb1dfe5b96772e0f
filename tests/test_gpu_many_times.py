"""More than 4096 distinct times (hourly or irregular data): the lag tables switch to live factors
(csrc/rows.cuh LagTable): the structure's integer-lag table when all times are integral (bit-identical
to the table mode), CUDA pow/log otherwise.  Against the oracle, which evaluates any lag
(covariance.cpp:138-149)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TH = (0.05, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _data(n, integral, seed=3):
    rng = np.random.default_rng(seed)
    x, y = rng.random(n), rng.random(n)
    t = np.arange(n, dtype=np.float64) if integral else np.sort(rng.random(n) * 0.37 * n)
    perm = O.order_observations(t, seed)
    r = np.sin(6 * x[perm]) + 0.3 * rng.standard_normal(n)
    return x[perm], y[perm], t[perm], r


def _check(g, sc, gref):
    assert (np.abs(g - gref) <= 1e-8 * sc).all(), (np.abs(g - gref) / sc).max()


@pytest.mark.parametrize("integral", [False, True])
def test_vecchia_many_times(S, integral):
    x, y, t, r = _data(5000, integral)
    assert len(np.unique(t)) > 4096
    ctx = S.Context(0)
    ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
    nb = S.correlation_neighbors(ds, TH, 12)
    ref = O.dc_neighbors(x, y, t, TH, 12)
    assert (nb.indices() == ref).mean() > 0.9999  # live pow may break exact near-ties only
    s = S.build_vecchia(ds, TH, S.NeighborSets.from_sets(ds, ref), S.OBSERVATION)
    v, g = S.nll_and_grad(s, r)
    om = O.OracleModel("vecchia", x, y, t, TH, nbr=ref)
    assert v == pytest.approx(om.nll(r), rel=1e-8)
    gr, sc = om.nll_grad_scale(r)
    _check(g, sc, gr)


@pytest.mark.parametrize("integral", [True, False])
def test_vif_and_fitc_many_times(S, integral):
    x, y, t, r = _data(4500, integral, seed=5)
    Z = np.column_stack([x, y, t])[::97].copy()
    Z[:, 2] += 0.5  # inducing times off the data grid: live factors for data-inducing lags
    ctx = S.Context(0)
    ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
    ind = S.InducingSet.from_points(Z, ctx=ctx)
    nbr = O.dr_neighbors(x, y, t, TH, Z, 10)
    s = S.build_vif(ds, TH, ind, S.NeighborSets.from_sets(ds, nbr, S.METRIC_DR), S.OBSERVATION)
    v, g = S.nll_and_grad(s, r)
    om = O.OracleModel("vif", x, y, t, TH, nbr=nbr, Z=Z)
    gr, sc = om.nll_grad_scale(r)
    assert v == pytest.approx(om.nll(r), rel=1e-8)
    _check(g, sc, gr)
    f = S.build_fitc(ds, TH, ind)
    v, g = S.nll_and_grad(f, r)
    of = O.OracleModel("fitc", x, y, t, TH, Z=Z)
    gr, sc = of.nll_grad_scale(r)
    assert v == pytest.approx(of.nll(r), rel=1e-8)
    _check(g, sc, gr)
