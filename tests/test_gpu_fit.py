"""Fit driver (csrc/fit.cu) against the oracle restatement of
estimation.cpp:423-619 (oracle.fit_gaussian): identical selection refreshes (the searches are
bit-exact), objective values within 1e-8, so the L-BFGS trajectories agree iterate by iterate."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _data(S, st, days, seed, p=0):
    th = S.synth.THETA_SEC4
    x, y, t, resp = S.synth.station_day(st, days, theta=th, seed=seed)
    X = None
    if p:
        rng = np.random.default_rng(seed)
        X = np.column_stack([np.ones(len(x))] + [rng.standard_normal(len(x)) for _ in range(p - 1)])
        resp = resp + X @ np.linspace(0.5, -0.3, p)
    return x, y, t, resp, X


@pytest.mark.parametrize("method,m_v,m,p", [("vecchia-corr", 8, 0, 0), ("vecchia-euclid", 6, 0, 2),
                                            ("vif", 6, 20, 0), ("fitc-sts", 0, 24, 0)])
def test_fit_matches_oracle(S, method, m_v, m, p):
    x, y, t, resp, X = _data(S, 60, 8, 7, p)
    init = (0.05, 0.8, 0.4, 12.0, 0.5, 1.5, 0.4, 0.3)
    cfg = S.FitConfig(method=method, m_v=max(m_v, 1), m=max(m, 1), max_iterations=6, seed=11)
    fm = S.fit(x, y, t, resp, X, config=cfg, init=init)
    ds = fm.data
    Xo = None if X is None else ds.X
    th, beta, f, conv, trace = O.fit_gaussian(ds.x, ds.y, ds.t, ds.resp, Xo, method, max(m_v, 1), max(m, 1), 11, 1.5,
                                               init, max_iterations=6)
    assert len(fm.trace) == len(trace)
    for a, b in zip(fm.trace, trace):
        assert a[0] == b[0] and a[3] == b[3]
        assert a[1] == pytest.approx(b[1], rel=1e-8)
    assert np.allclose(fm.theta.as_tuple(), th, rtol=1e-6)
    assert fm.final_nll == pytest.approx(f, rel=1e-8)
    if p:
        assert np.allclose(fm.beta, beta, rtol=1e-6, atol=1e-9)


def test_default_init(S):
    x, y, t, resp, _ = _data(S, 80, 6, 3)
    cfg = S.FitConfig(method="vecchia-corr", seed=5)
    ds = S.order_observations(x, y, t, resp, seed=5)
    th = S.default_init(ds, cfg)
    var = np.var(ds.resp, ddof=1)
    assert th.sigma2 == pytest.approx(0.5 * var, rel=1e-12) and th.sigma1_2 == pytest.approx(0.5 * var, rel=1e-12)
    assert (th.alpha, th.beta, th.delta, th.nu) == (0.8, 0.5, 0.5, 1.5)
    assert 1e-8 <= th.a <= 1e12 and 1e-8 <= th.c <= 1e12


def test_fit_converges_small(S):
    x, y, t, resp, _ = _data(S, 40, 6, 9)
    fm = S.fit(x, y, t, resp, config=S.FitConfig(method="vecchia-corr", m_v=6, max_iterations=60, seed=1))
    f0 = fm.trace[0][1]
    assert fm.final_nll < f0 and np.isfinite(fm.final_nll)
    refreshed = {r[0] for r in fm.trace if r[3]}
    assert {1, 2, 4} <= refreshed  # power-of-two selection refreshes (neighbors.cpp:331-334)
