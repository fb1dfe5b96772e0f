"""GPU parity for the selection path: kMeans++ / sts / joint seeding and the
residual-correlation (d_r) neighbour search, bit-exact against the oracle
(test_inducing.cpp, test_neighbors.cpp:111-131, 222-238)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _bits(a, b):
    return (np.asarray(a).view(np.uint64) == np.asarray(b).view(np.uint64)).all()


@pytest.mark.parametrize("n,d,k,seed", [(500, 2, 20, 1), (300, 1, 7, 2), (400, 3, 25, 3), (4, 2, 4, 7), (5, 1, 1, 3)])
def test_kmeanspp_bit_exact(S, n, d, k, seed):
    rng = np.random.default_rng(seed)
    P = rng.random((n, d)) if n > 5 else (np.array([[0, 0], [1, 0], [0, 1], [1, 1]], float) if d == 2 else
                                           np.array([[1.0], [2], [3], [4], [10]]))
    c = S.kmeanspp(P, k, seed)
    assert _bits(c, O.kmeanspp(P, k, seed))


def test_kmeanspp_errors(S):
    with pytest.raises(S.DataError):
        S.kmeanspp(np.array([[1.0], [1], [2], [2]]), 3, 1)
    with pytest.raises(S.ConfigError):
        S.kmeanspp(np.array([[1.0], [2]]), 0, 1)


def test_sts_counts_and_bits(S):
    # test_inducing.cpp:101-110: 500 locations x 20 times, m = 500 -> 112 x 4
    x, y, t, _, _ = O.test_dataset(2, 500, 5, n_times=20)
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.sts_kmeanspp(ds, 500, 1)
    assert (ind.m_s, ind.m_t, ind.M) == (112, 4, 448)
    Z, ms, mt = O.sts_kmeanspp(x, y, t, 500, 1)
    assert _bits(ind.points, Z)


def test_sts_cfg3_shape(S):
    x, y, t, _ = S.synth.station_day(1000, 100, seed=11)
    perm = O.order_observations(t, 11)
    x, y, t = x[perm], y[perm], t[perm]
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.sts_kmeanspp(ds, 200, 20260203)
    assert (ind.m_s, ind.m_t) == (45, 4)
    Z, _, _ = O.sts_kmeanspp(x, y, t, 200, 20260203)
    assert _bits(ind.points, Z)


def test_joint_kmeanspp_bits(S):
    x, y, t, _, _ = O.test_dataset(2, 60, 23, n_times=6)
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.joint_kmeanspp_inducing(ds, 25, 0.5, 2.0, 5)
    assert ind.M == 25
    assert _bits(ind.points, O.joint_kmeanspp(x, y, t, 25, 0.5, 2.0, 5))
    with pytest.raises(S.ConfigError):
        S.joint_kmeanspp_inducing(ds, 25, 0.0, 2.0, 5)


def test_joint_kmeanspp_large_certified(S):
    """Certified parallel picks and cluster-sorted Lloyd sums (csrc/kmeans.cu) at n = 2e5, k = 300: bit-equal
    to the oracle's sequential kmeanspp (inducing.cpp:32-115)."""
    rng = np.random.default_rng(3)
    n = 200000
    x, y, t = rng.random(n), rng.random(n), np.repeat(np.arange(100.0), n // 100)
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.joint_kmeanspp_inducing(ds, 300, 0.2, 5.0, 7)
    assert _bits(ind.points, O.joint_kmeanspp(x, y, t, 300, 0.2, 5.0, 7))


def _check_dr(S, x, y, t, th, Z, m):
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.residual_neighbors(ds, th, S.InducingSet.from_points(Z), m)
    idx, dist = nb.indices(), nb.distances()
    ref, rdist = O.dr_neighbors(x, y, t, th, Z, m, with_dist=True)
    assert (idx == ref).all(), np.argwhere(idx != ref)[:5]
    ok = ~np.isnan(rdist)
    assert _bits(dist[ok], rdist[ok])


def test_dr_reference_case(S):
    # test_neighbors.cpp:111-131: n = 600, m = 20, 25 random inducing points
    x, y, t, _, _ = O.test_dataset(0, 600, 19)
    rng = np.random.default_rng(5)
    Z = np.column_stack([rng.random(25), rng.random(25), 1 + 9 * rng.random(25)])
    _check_dr(S, x, y, t, SEC4, Z, 20)


def test_dr_station_day_sts(S):
    x, y, t, _ = S.synth.station_day(200, 15, seed=4)
    perm = O.order_observations(t, 4)
    x, y, t = x[perm], y[perm], t[perm]
    Z, _, _ = O.sts_kmeanspp(x, y, t, 100, 9)
    _check_dr(S, x, y, t, SEC4, Z, 30)
    _check_dr(S, x, y, t, SEC4, Z[:70], 7)


def test_dr_degenerate(S):
    # test_neighbors.cpp:222-238
    pts = np.array([[0.5, 0.5, 1.0], [0.2, 0.8, 1.0], [0.9, 0.1, 2.0]])
    ds = S.SpaceTimeDataset(pts[:, 0], pts[:, 1], pts[:, 2])
    nb = S.residual_neighbors(ds, SEC4, S.InducingSet.from_points(pts[:1]), 2)
    d = nb.distances()
    assert d[1, 0] == 1.0 and d[2, 1] == 1.0 and d[2, 0] < 1.0
    _check_dr(S, pts[:, 0], pts[:, 1], pts[:, 2], SEC4, pts[:1], 2)


def test_dr_empty_inducing_equals_dc(S):
    x, y, t, _, _ = O.test_dataset(0, 300, 3)
    ds = S.SpaceTimeDataset(x, y, t)
    a = S.correlation_neighbors(ds, SEC4, 8).indices()
    b = S.residual_neighbors(ds, SEC4, S.InducingSet.from_points(np.zeros((0, 3))), 8).indices()
    assert (a == b).all()


@pytest.mark.parametrize("spatial", ["0", "1"])
def test_dc_both_search_kernels(S, monkeypatch, spatial):
    # the d_c search runs on the time-block kernel or on the spatial-tile kernel (the default where
    # equal-time blocks average >= 4096 rows, e.g. cfg4); both must return the oracle's sets and
    # distances bit for bit, here on the cfg4 geometry with 4500 rows per day
    monkeypatch.setenv("STGP_DC_SPATIAL", spatial)
    x, y, t, _ = S.synth.station_day(4500, 3, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=33)
    perm = O.order_observations(t, 33)
    x, y, t = x[perm], y[perm], t[perm]
    ds = S.SpaceTimeDataset(x, y, t)
    nb = S.correlation_neighbors(ds, S.synth.THETA_T3, 30)
    ref, rdist = O.dc_neighbors(x, y, t, S.synth.THETA_T3, 30, with_dist=True)
    assert (nb.indices() == ref).all(), np.argwhere(nb.indices() != ref)[:5]
    ok = ~np.isnan(rdist)
    assert _bits(nb.distances()[ok], rdist[ok])


def test_dr_spatial_pruning_geometry(S):
    # cfg4 geometry (Table 3 theta, 4600 x 2900 km box): spatial tiles, box-distance and
    # block-norm pruning and the early time stop are all active; exactness against the oracle
    x, y, t, _ = S.synth.station_day(2000, 8, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=21)
    perm = O.order_observations(t, 21)
    x, y, t = x[perm], y[perm], t[perm]
    Z, _, _ = O.sts_kmeanspp(x, y, t, 200, 21)
    _check_dr(S, x, y, t, S.synth.THETA_T3, Z, 30)


def test_dr_unsorted_rows_brute_force(S):
    # rows not time sorted: one index-order bucket, no pruning
    x, y, t, _ = S.synth.station_day(60, 8, seed=5)
    rng = np.random.default_rng(3)
    perm = rng.permutation(len(x))
    x, y, t = x[perm], y[perm], t[perm]
    Z, _, _ = O.sts_kmeanspp(x, y, t, 40, 2)
    _check_dr(S, x, y, t, SEC4, Z, 12)


def test_dr_low_rank_dominant(S):
    # many inducing points per datum: |w|^2 / r is large, the half-precision filter's bound is at
    # its loosest; the sets must still equal the oracle's
    x, y, t, _ = S.synth.station_day(120, 6, seed=8)
    perm = O.order_observations(t, 8)
    x, y, t = x[perm], y[perm], t[perm]
    Z, _, _ = O.sts_kmeanspp(x, y, t, 300, 3)
    _check_dr(S, x, y, t, SEC4, Z, 16)


def test_dr_filter_on_off_identical(S, monkeypatch):
    x, y, t, _ = S.synth.station_day(1500, 6, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=31)
    perm = O.order_observations(t, 31)
    x, y, t = x[perm], y[perm], t[perm]
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.sts_kmeanspp(ds, 300, 31)
    a = S.residual_neighbors(ds, S.synth.THETA_T3, ind, 30)
    monkeypatch.setenv("STGP_DR_FILTER", "0")
    b = S.residual_neighbors(ds, S.synth.THETA_T3, ind, 30)
    assert (a.indices() == b.indices()).all()
    assert _bits(a.distances(), b.distances())


def test_dc_spatial_path_identical(S, monkeypatch):
    # the spatial-tile search with no inducing points is the exact d_c search
    x, y, t, _ = S.synth.station_day(1200, 5, box=(4.6e6, 2.9e6), theta=S.synth.THETA_T3, seed=12)
    perm = O.order_observations(t, 12)
    x, y, t = x[perm], y[perm], t[perm]
    ds = S.SpaceTimeDataset(x, y, t)
    a = S.correlation_neighbors(ds, S.synth.THETA_T3, 30)
    monkeypatch.setenv("STGP_DC_SPATIAL", "1")
    b = S.correlation_neighbors(ds, S.synth.THETA_T3, 30)
    assert (a.indices() == b.indices()).all()
    assert _bits(a.distances(), b.distances())


def test_sts_signed_zero_and_duplicates(S):
    # distinct locations / times follow std::set: -0.0 == +0.0 (first occurrence kept), duplicates merged
    rng = np.random.default_rng(4)
    x = rng.random(400)
    y = rng.random(400)
    x[::7] = 0.0
    x[3::7] = -0.0
    y[5::11] = -0.0
    t = np.repeat(np.arange(1.0, 9.0), 50)
    t[::13] = -0.0 + 0.0
    ds = S.SpaceTimeDataset(x, y, t)
    ind = S.sts_kmeanspp(ds, 40, 9)
    Z, ms, mt = O.sts_kmeanspp(x, y, t, 40, 9)
    assert (ind.m_s, ind.m_t) == (ms, mt)
    assert _bits(ind.points, Z)
