"""Dataset CSV and neighbour-audit formats (csrc/csvio.cu), restating test_dataset.cpp:146-189 and
checking the bytes the reference's streams produce (precision 17 = "%.17g")."""
import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


def test_csv_round_trip_with_stations_and_covariates(S, tmp_path):
    p = tmp_path / "test_dataset_io.csv"
    p.write_text("# provenance line\nx,y,t,value,station_id,elev,slope\n"
                 "0.5,0.25,1,2.5,alpha,120.0,0.1\n0.75,0.5,2,3.5,bravo,80.0,0.2\n")
    d = S.read_dataset_csv(str(p))
    assert len(d.x) == 2 and d.X.shape == (2, 2)
    assert d.stations[0] == "alpha" and d.X[1, 0] == 80.0 and d.value[1] == 3.5
    assert d.covariate_names == ["elev", "slope"]
    out = tmp_path / "test_dataset_io_out.csv"
    S.write_dataset_csv(str(out), d.x, d.y, d.t, d.value, d.X, d.stations, "hash=abc")
    assert out.read_text() == ("# hash=abc\nx,y,t,value,station_id,x0,x1\n"
                               "0.5,0.25,1,2.5,alpha,120,0.10000000000000001\n"
                               "0.75,0.5,2,3.5,bravo,80,0.20000000000000001\n")
    back = S.read_dataset_csv(str(out))
    assert len(back.x) == 2 and back.X[0, 1] == 0.1


def test_csv_whitespace_trailing_comma_and_bytes(S, tmp_path):
    rng = np.random.default_rng(4)
    x, y, t, v = rng.random(20), rng.random(20) * 1e-7, np.arange(20.0), rng.standard_normal(20) * 1e12
    out = tmp_path / "w.csv"
    S.write_dataset_csv(str(out), x, y, t, v)
    lines = ["x,y,t,value"] + [",".join("%.17g" % c for c in row) for row in zip(x, y, t, v)]
    assert out.read_text() == "\n".join(lines) + "\n"
    back = S.read_dataset_csv(str(out))
    assert (back.x == x).all() and (back.y == y).all() and (back.value == v).all()  # %.17g round-trips exactly
    p = tmp_path / "ws.csv"
    p.write_text("x , y,t,value\n 0.5\t, 0.25 ,1,2.5\r\n")
    d = S.read_dataset_csv(str(p))
    assert d.x[0] == 0.5 and d.y[0] == 0.25
    p.write_text("x,y,t,value\n0.5,0.25,1,\n")  # trailing comma: an empty last field
    with pytest.raises(S.DataError):
        S.read_dataset_csv(str(p))


@pytest.mark.parametrize("body", ["x,y,t,value\n0.5,,1,2.5\n", "x,y,value\n0.5,0.5,1\n", "x,y,t,value\n0.5,0.1,1,nope\n",
                                  "x,y,t,value\n0.5,0.1,1,inf\n", "x,y,t,value\n", "x,y,t,value,station_id\n1,2,3,4,\n",
                                  "x,y,t,value\n1,2,3\n", "# only a comment\n"])
def test_csv_rejects_missing_and_malformed(S, tmp_path, body):
    p = tmp_path / "bad.csv"
    p.write_text(body)
    with pytest.raises(S.DataError):
        S.read_dataset_csv(str(p))


def test_csv_missing_file(S, tmp_path):
    with pytest.raises(S.DataError):
        S.read_dataset_csv(str(tmp_path / "nope.csv"))


@pytest.mark.gpu
@pytest.mark.parametrize("metric", ["dc", "euclidean"])
def test_neighbor_audit_bytes(S, tmp_path, metric):
    from oracle import oracle as O
    th = S.synth.THETA_SEC4
    x, y, t, resp = S.synth.station_day(60, 6, theta=th, seed=2)
    ds = S.order_observations(x, y, t, resp, seed=2)
    if metric == "dc":
        nb = S.correlation_neighbors(ds, th, 8)
        idx, dist = O.dc_neighbors(ds.x, ds.y, ds.t, th, 8, with_dist=True)
    else:
        tr, sr = S.effective_ranges(th)
        nb = S.euclidean_neighbors(ds, 8, sr, tr)
        idx = O.euclid_neighbors(ds.x, ds.y, ds.t, 8, sr, tr)
    out = tmp_path / "audit.csv"
    S.write_neighbor_debug_csv(str(out), nb, ds, "seed=2")
    lines = ["# seed=2", "i,rank,neighbor_index,distance"]
    for i in range(len(ds.x)):
        rows = []
        for a, j in enumerate(idx[i]):
            if j < 0:
                continue
            if metric == "dc":
                d = dist[i, a]
            else:  # cli.cpp:549-563
                dx, dy, dt = (ds.x[i] - ds.x[j]) / sr, (ds.y[i] - ds.y[j]) / sr, (ds.t[i] - ds.t[j]) / tr
                d = float(np.sqrt(dx * dx + dy * dy + dt * dt))
            rows.append((d, int(j)))
        for r, (d, j) in enumerate(sorted(rows)):
            lines.append(f"{i},{r},{j},{'%.17g' % d}")
    assert out.read_text() == "\n".join(lines) + "\n"
