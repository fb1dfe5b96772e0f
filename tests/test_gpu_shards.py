"""Sharded (multi-rank) evaluation emulated with two contexts on one GPU.

Each rank owns a contiguous row range (stgp_ctx_set_shard) and exchanges its
partial sums through a host all-reduce hook; the kernels of the two ranks never
wait on each other on the device.  The sharded NLL and gradient must equal the
single-context values."""
import threading

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEC4 = (0.05, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def _run(S, world, build, x, y, t, yv, X=None, beta=None):
    out = [None] * world
    err = [None] * world
    hub = S.api.HostAllreduce(world) if world > 1 else None

    def work(rank):
        try:
            ctx = S.Context(0)
            if world > 1:
                ctx.set_shard(rank, world)
                ctx.set_host_allreduce(hub.for_rank(rank))
            ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
            s = build(S, ds, ctx)
            out[rank] = S.nll_and_grad(s, yv, X, beta)
        except Exception as e:  # noqa: BLE001
            err[rank] = e
            if hub:
                hub.barrier.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    # the first rank's own failure, not the aborted all-reduce it caused on the other ranks
    real = [e for e in err if e is not None and "all-reduce callback failed" not in str(e)]
    for e in real + [e for e in err if e is not None]:
        raise e
    return out


@pytest.mark.parametrize("kind", ["vecchia", "vif", "fitc"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single(S, kind, world):
    x, y, t, yv, X = O.test_dataset(1, 1800, 53, n_times=9, p=1)
    beta = np.array([0.2])
    Z = np.column_stack([x, y, t])[::61]
    nbr = O.dr_neighbors(x, y, t, SEC4, Z, 12) if kind == "vif" else O.dc_neighbors(x, y, t, SEC4, 12)

    def build(S, ds, ctx):
        nb = S.NeighborSets.from_sets(ds, nbr)
        ind = S.InducingSet.from_points(Z, ctx=ctx)
        if kind == "vecchia":
            return S.build_vecchia(ds, SEC4, nb, S.OBSERVATION)
        if kind == "vif":
            return S.build_vif(ds, SEC4, ind, nb, S.OBSERVATION)
        return S.build_fitc(ds, SEC4, ind)

    (v1, g1), = _run(S, 1, build, x, y, t, yv, X, beta)
    res = _run(S, world, build, x, y, t, yv, X, beta)
    for v, g in res:
        assert v == pytest.approx(v1, rel=1e-11)
        assert np.allclose(g, g1, rtol=1e-10, atol=1e-10 * np.abs(g1).max())
    # every rank holds identical bits
    assert all(r[0] == res[0][0] and (r[1] == res[0][1]).all() for r in res)


@pytest.mark.parametrize("metric", ["dr", "dc", "euclid"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_equals_single(S, metric, world):
    # queries shard by rows / time buckets, rows are gathered: every rank holds the full sets, bit-equal
    x, y, t, _ = S.synth.station_day(150, 8, seed=6)
    perm = O.order_observations(t, 6)
    x, y, t = x[perm], y[perm], t[perm]
    Z, _, _ = O.sts_kmeanspp(x, y, t, 60, 6)

    def search(S, ctx):
        ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
        if metric == "dr":
            nb = S.residual_neighbors(ds, SEC4, S.InducingSet.from_points(Z, ctx=ctx), 10)
        elif metric == "dc":
            nb = S.correlation_neighbors(ds, SEC4, 10)
        else:
            nb = S.euclidean_neighbors(ds, 10, 0.5, 2.0)
        return nb.indices(), nb.distances()

    def run(world):
        out, err = [None] * world, [None] * world
        hub = S.api.HostAllreduce(world) if world > 1 else None

        def work(rank):
            try:
                ctx = S.Context(0)
                if world > 1:
                    ctx.set_shard(rank, world)
                    ctx.set_host_allreduce(hub.for_rank(rank))
                out[rank] = search(S, ctx)
            except Exception as e:  # noqa: BLE001
                err[rank] = e
                if hub:
                    hub.barrier.abort()

        th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for h in th:
            h.start()
        for h in th:
            h.join()
        real = [e for e in err if e is not None and "all-reduce callback failed" not in str(e)]
        for e in real + [e for e in err if e is not None]:
            raise e
        return out

    (i1, d1), = run(1)
    for ir, dr in run(world):
        assert (ir == i1).all()
        ok = ~np.isnan(d1)
        assert (np.isnan(dr) == ~ok).all() and (dr[ok].view(np.int64) == d1[ok].view(np.int64)).all()


def test_sharded_failure_raises_on_every_rank(S):
    """A non-PD conditioning block on one shard only: every rank raises NumericError together (no rank is
    left waiting in the next collective, so the fit's step halving works sharded, estimation.cpp:575-579)."""
    x, y, t, _ = S.synth.station_day(60, 6, seed=11)
    perm = O.order_observations(t, 11)
    x, y, t = x[perm].copy(), y[perm].copy(), t[perm].copy()
    n = len(x)
    # row i in the second shard duplicates an earlier same-day row j and conditions on j alone: with the
    # latent policy (no nugget) and sigma1^2 = 1 its conditional variance is exactly 1 - 1*1 = 0
    # -> "non-positive conditional variance" (approximations.cpp:107-110)
    i = 3 * n // 4
    j = int(np.nonzero(t[:i] == t[i])[0][0])
    x[i], y[i] = x[j], y[j]
    nbr = O.dc_neighbors(x, y, t, SEC4, 1)
    assert nbr[i][0] == j
    world = 2
    err = [None] * world
    hub = S.api.HostAllreduce(world, timeout=60.0)

    def work(rank):
        try:
            ctx = S.Context(0)
            ctx.set_shard(rank, world)
            ctx.set_host_allreduce(hub.for_rank(rank))
            ds = S.SpaceTimeDataset(x, y, t, ctx=ctx)
            nb = S.NeighborSets.from_sets(ds, nbr)
            S.build_vecchia(ds, SEC4, nb, S.LATENT)
        except Exception as e:  # noqa: BLE001
            err[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    assert all(isinstance(e, S.NumericError) for e in err), err
    assert "another shard" in str(err[0]) and "another shard" not in str(err[1])
