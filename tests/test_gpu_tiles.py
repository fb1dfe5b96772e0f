"""Tile-staged gathers (csrc/tiles.cu) against the per-row gathers and the oracle.

V', Ga and E/F are formed over tiles of space-time neighbours whose union of closure columns is
staged in shared memory (STGP_TILES=1, the default).  STGP_TILES=0 runs the per-row gathers
(lowrank.cu vprime_kernel / ef_kernel and the DMMA Ga pass of the rows kernel).  Both must give
the oracle's NLL and gradient (1e-8) and agree with each other far tighter; m_v = 30 exercises the
31-slot closure of the cfg4 headline.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_2602_03609_b200 as S
th = S.synth.THETA_SEC4
x, y, t, resp = S.synth.station_day(%(st)d, %(days)d, theta=th, seed=11)
perm = S.order_observations_perm(t, 11)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ds = S.SpaceTimeDataset(x, y, t, resp)
ind = S.sts_kmeanspp(ds, %(m)d, 5)
nb = S.residual_neighbors(ds, th, ind, %(mv)d)
s = S.build_vif(ds, th, ind, nb, S.OBSERVATION)
v, g = S.nll_and_grad(s, resp)
np.savez(%(out)r, x=x, y=y, t=t, resp=resp, Z=ind.points, nbr=nb.indices())
print(json.dumps({"nll": v, "grad": list(map(float, g))}))
"""


def _run(tmp_path, tiles, st, days, m, mv, **extra_env):
    out = str(tmp_path / f"case_{tiles}_{len(extra_env)}.npz")
    env = dict(os.environ, STGP_TILES=str(tiles), **extra_env)
    code = _SCRIPT % dict(root=ROOT, st=st, days=days, m=m, mv=mv, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1]), np.load(out)


@pytest.mark.parametrize("st,days,m,mv", [(400, 12, 60, 30), (300, 9, 40, 17)])
def test_tiles_match_row_gathers_and_oracle(tmp_path, st, days, m, mv):
    a, case = _run(tmp_path, 1, st, days, m, mv)
    b, _ = _run(tmp_path, 0, st, days, m, mv)
    ga, gb = np.array(a["grad"]), np.array(b["grad"])
    assert a["nll"] == pytest.approx(b["nll"], rel=1e-12)
    assert np.allclose(ga, gb, rtol=1e-10, atol=1e-10 * np.abs(gb).max())
    th = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
    om = O.OracleModel("vif", case["x"], case["y"], case["t"], th, nbr=case["nbr"], Z=case["Z"])
    vr, (gr, sc) = om.nll(case["resp"]), om.nll_grad_scale(case["resp"])
    assert a["nll"] == pytest.approx(vr, rel=1e-8)
    assert O.grad_close(ga, gr, sc), (ga, gr, sc)


def test_ozaki_products_inside_vif_match_oracle(tmp_path):
    # the int8 Ozaki products run only from M >= 512 by default; force them at test size
    a, case = _run(tmp_path, 1, 300, 9, 40, 17, STGP_OZAKI_MIN_M="0")
    b, _ = _run(tmp_path, 1, 300, 9, 40, 17, STGP_OZAKI="0")
    ga, gb = np.array(a["grad"]), np.array(b["grad"])
    assert a["nll"] == pytest.approx(b["nll"], rel=1e-11)
    assert np.allclose(ga, gb, rtol=1e-9, atol=1e-9 * np.abs(gb).max())
    th = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
    om = O.OracleModel("vif", case["x"], case["y"], case["t"], th, nbr=case["nbr"], Z=case["Z"])
    vr, (gr, sc) = om.nll(case["resp"]), om.nll_grad_scale(case["resp"])
    assert a["nll"] == pytest.approx(vr, rel=1e-8)
    assert O.grad_close(ga, gr, sc), (ga, gr, sc)
