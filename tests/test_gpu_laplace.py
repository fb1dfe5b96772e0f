"""Latent-policy likelihoods on the device (csrc/laplace.cu) against the oracle:
the Gaussian latent-policy NLL through the Laplace algebra (approximations.cpp:320-334) and the ZC-PTN
Laplace marginal with its Newton state (laplace.cpp:115-203), for Vecchia, FITC and VIF.  Tolerances:
values 1e-8 relative, mode / w / grad_at_mode 1e-6 of their scale (Newton stops at a 1e-6 gradient gap)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TH = (0.25, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
LATENT = (0.0, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _data(S, stations=120, days=8, seed=5):
    x, y, t, resp = S.synth.station_day(stations, days, seed=seed)
    perm = O.order_observations(t, seed)
    return x[perm], y[perm], t[perm], resp[perm]


def _structures(S, kind, x, y, t, th, m_v=10):
    ctx = S.Context(0)
    ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
    Z = np.column_stack([x, y, t])[::41]
    nbr = None
    if kind == "vecchia":
        nbr = O.dc_neighbors(x, y, t, th, m_v)
        s = S.build_vecchia(ds, th, S.NeighborSets.from_sets(ds, nbr), S.LATENT)
    elif kind == "vif":
        nbr = O.dr_neighbors(x, y, t, th, Z, m_v)
        s = S.build_vif(ds, th, S.InducingSet.from_points(Z, ctx=ctx), S.NeighborSets.from_sets(ds, nbr, S.METRIC_DR),
                        S.LATENT)
    else:
        s = S.build_fitc(ds, th, S.InducingSet.from_points(Z, ctx=ctx))
    om = O.OracleModel(kind, x, y, t, th, nbr=nbr, Z=None if kind == "vecchia" else Z, policy="latent")
    return s, om, (ctx, ds)


@pytest.mark.parametrize("kind", ["vecchia", "vif"])
def test_latent_gaussian_nll(S, kind):
    x, y, t, resp = _data(S)
    s, om, keep = _structures(S, kind, x, y, t, TH)
    v = S.nll(s, resp)
    assert v == pytest.approx(om.nll(resp), rel=1e-8)


def test_latent_nll_full_conditioning_equals_dense(S):
    # approximations.cpp:97-142 limit through the latent path
    x, y, t, resp = _data(S, 30, 6)
    ctx = S.Context(0)
    ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
    s = S.build_vecchia(ds, TH, S.NeighborSets.from_sets(ds, O.full_conditioning(len(x))), S.LATENT)
    assert S.nll(s, resp) == pytest.approx(O.dense_nll(x, y, t, TH, resp), rel=1e-9)


@pytest.mark.parametrize("kind", ["vecchia", "fitc", "vif"])
def test_laplace_marginal_zcptn(S, kind):
    x, y, t, resp = _data(S)
    rng = np.random.default_rng(11)
    amounts = np.where(rng.random(len(x)) < 0.45, 0.0, rng.gamma(1.5, 1.2, len(x)))  # censored amounts
    s, om, keep = _structures(S, kind, x, y, t, LATENT)
    lik = S.LikelihoodParams(0.8, 1.6)
    v, st = S.laplace_marginal(s, amounts, lik=lik)
    vr, str_ = O.laplace_marginal(om, amounts, 0.8, 1.6)
    assert v == pytest.approx(vr, rel=1e-8)
    for key, dev in (("mode", st.mode), ("grad_at_mode", st.grad_at_mode), ("w", st.w)):
        ref = str_[key]
        assert np.abs(dev - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max()), key
    # warm start from the mode converges at once to the same value
    v2, st2 = S.laplace_marginal(s, amounts, lik=lik, warm_start=st.mode)
    assert v2 == pytest.approx(v, rel=1e-8) and st2.iterations <= 2


@pytest.mark.parametrize("kind", ["vecchia", "fitc", "vif"])
def test_laplace_exact_gaussian_case_device(S, kind):
    """test_laplace.cpp:144-192 on the device: all-positive data, lambda = 1 -> the Gaussian marginal."""
    x, y, t, _ = _data(S, 40, 5)
    amounts = 2.0 + np.cos(5 * x) + y
    sig = 0.9
    th_obs = (sig * sig,) + LATENT[1:]
    ctx = S.Context(0)
    ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
    full = O.full_conditioning(len(x))
    P = np.column_stack([x, y, t])
    if kind == "vecchia":
        s = S.build_vecchia(ds, LATENT, S.NeighborSets.from_sets(ds, full), S.LATENT)
        ref = O.dense_nll(x, y, t, th_obs, amounts)
    elif kind == "fitc":
        Z = P[::13]
        s = S.build_fitc(ds, LATENT, S.InducingSet.from_points(Z, ctx=ctx))
        ref = O.OracleModel("fitc", x, y, t, th_obs, Z=Z).nll(amounts)
    else:
        Z = P[::17]
        s = S.build_vif(ds, LATENT, S.InducingSet.from_points(Z, ctx=ctx), S.NeighborSets.from_sets(ds, full),
                        S.LATENT)
        ref = O.dense_nll(x, y, t, th_obs, amounts)
    v, _ = S.laplace_marginal(s, amounts, lik=S.LikelihoodParams(sig, 1.0))
    assert v == pytest.approx(ref, rel=1e-8)


def test_laplace_rejects_bad_inputs(S):
    x, y, t, resp = _data(S, 30, 4)
    s, _, keep = _structures(S, "fitc", x, y, t, LATENT)
    with pytest.raises(S.DataError):
        S.laplace_marginal(s, resp - 10.0, lik=S.LikelihoodParams(1.0, 1.0))
    with pytest.raises(S.ConfigError):
        S.laplace_marginal(s, np.abs(resp), lik=S.LikelihoodParams(-1.0, 1.0))
    ctx = S.Context(0)
    ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
    so = S.build_vecchia(ds, TH, S.NeighborSets.from_sets(ds, O.dc_neighbors(x, y, t, TH, 5)), S.OBSERVATION)
    with pytest.raises(S.NumericError):  # LaplaceAlgebra: requires a latent-policy structure
        S.laplace_marginal(so, np.abs(resp), lik=S.LikelihoodParams(1.0, 1.0))


@pytest.mark.parametrize("kind", ["vecchia", "fitc", "vif"])
def test_zcptn_predict(S, kind):
    """zcptn_predict (laplace.cpp:205-259): latent moments 1e-8, P(rain) and the Monte Carlo amounts from
    the same RNG streams (draws differ from the oracle's only through the moments)."""
    x, y, t, resp = _data(S)
    rng = np.random.default_rng(13)
    amounts = np.where(rng.random(len(x)) < 0.4, 0.0, rng.gamma(1.5, 1.0, len(x)))
    s, om, keep = _structures(S, kind, x, y, t, LATENT)
    lik = S.LikelihoodParams(0.7, 1.4)
    last = t == t.max()
    T = np.column_stack([x[last][:25], y[last][:25], np.full(min(25, int(last.sum())), t.max() + 1.0)])
    # the same Laplace state on both sides (each Newton stops at its own 1e-6 gradient gap, which would
    # otherwise enter mu = k . a at that level)
    _, str_ = O.laplace_marginal(om, amounts, 0.7, 1.4)
    st = S.LaplaceState(str_["mode"], str_["grad_at_mode"], str_["w"], 0.0, True, str_["iterations"])
    pr = S.zcptn_predict(st, s, T, lik=lik, pred_m_v=8, n_samples=64, seed=9)
    ref = O.zcptn_predict(om, str_, T, 0.7, 1.4, 8, 64, 9)
    s1 = LATENT[1]
    assert np.allclose(pr.mu_latent, ref["mu_latent"], rtol=1e-8, atol=1e-8 * np.sqrt(s1))
    # the variance is k_pp - k'Wk + (Wk)'(Sigma^-1 + W)^-1 (Wk): 1e-8 of the magnitude it cancels from
    verr = np.abs(pr.var_latent - ref["var_latent"])
    assert (verr <= 1e-8 * ref["var_scale"]).all(), (verr / ref["var_scale"]).max()
    tol = 1e-8 * np.maximum(ref["var_scale"], 1.0)  # P(rain), draws: through mu and var
    assert (np.abs(pr.p_rain - ref["p_rain"]) <= tol).all()
    assert (np.abs(pr.samples - ref["samples"]) <= 10 * tol[:, None] * (1 + np.abs(ref["samples"]))).all()
    assert (np.abs(pr.amount_mean - ref["amount_mean"]) <= 10 * tol * (1 + np.abs(ref["amount_mean"]))).all()
