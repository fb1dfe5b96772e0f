"""The engine's A/B switches against their defaults, each in its own process (the
switches are read once): the alternative paths must agree with the defaults and the oracle.

* STGP_VGRAD_SPLIT=0: the Vecchia gradient as one fused row kernel instead of the factor and pair passes;
* STGP_OZAKI_TRMM=0: W = L_m^-1 U and omega = L_m^-T omega' on the DMMA TRMM instead of the int8 kernel;
* STGP_FITC_SYM_S=0: FITC's W diag(phi) W^T on all tiles instead of one triangle, mirrored.
The int8 paths are forced at test size with STGP_OZAKI_MIN_M=0.
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
from oracle import oracle as O
x, y, t, yv, X = O.test_dataset(1, 1600, 61, n_times=8, p=1)
rng = np.random.default_rng(5)
Z = np.column_stack([rng.random(44), rng.random(44), 1 + 7 * rng.random(44)])
th = (0.2, 1.1, 0.8, 12.0, 0.6, 1.5, 0.3, 0.5)
beta = np.array([-0.2])
ds = S.SpaceTimeDataset(x, y, t)
ind = S.InducingSet.from_points(Z)
out = {}
s = S.build_vecchia(ds, th, S.NeighborSets.from_sets(ds, O.dc_neighbors(x, y, t, th, 25)), S.OBSERVATION)
v, g = S.nll_and_grad(s, yv, X, beta)
out["vecchia"] = [float(v)] + list(map(float, g))
s = S.build_vif(ds, th, ind, S.NeighborSets.from_sets(ds, O.dr_neighbors(x, y, t, th, Z, 12)), S.OBSERVATION)
v, g = S.nll_and_grad(s, yv, X, beta)
out["vif"] = [float(v)] + list(map(float, g))
s = S.build_fitc(ds, th, ind)
v, g = S.nll_and_grad(s, yv, X, beta)
out["fitc"] = [float(v)] + list(map(float, g))
print(json.dumps(out))
"""


def _run(**env):
    e = dict(os.environ, STGP_OZAKI_MIN_M="0", **env)
    r = subprocess.run([sys.executable, "-c", _SCRIPT % dict(root=ROOT)], env=e, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return {k: np.array(v) for k, v in json.loads(r.stdout.strip().splitlines()[-1]).items()}


@pytest.fixture(scope="module")
def default():
    return _run()


@pytest.fixture(scope="module")
def oracle_results():
    x, y, t, yv, X = O.test_dataset(1, 1600, 61, n_times=8, p=1)
    rng = np.random.default_rng(5)
    Z = np.column_stack([rng.random(44), rng.random(44), 1 + 7 * rng.random(44)])
    th = (0.2, 1.1, 0.8, 12.0, 0.6, 1.5, 0.3, 0.5)
    beta = np.array([-0.2])
    res = {}
    for kind, kw in (("vecchia", dict(nbr=O.dc_neighbors(x, y, t, th, 25))),
                     ("vif", dict(nbr=O.dr_neighbors(x, y, t, th, Z, 12), Z=Z)), ("fitc", dict(Z=Z))):
        om = O.OracleModel(kind, x, y, t, th, **kw)
        gr, sc = om.nll_grad_scale(yv, X, beta)
        res[kind] = (om.nll(yv, X, beta), gr, sc)
    return res


def _check(res, ref, kind):
    nll, gr, sc = ref[kind]
    assert res[kind][0] == pytest.approx(nll, rel=1e-8)
    assert O.grad_close(res[kind][1:], gr, sc), (kind, res[kind][1:], gr)


def test_defaults_match_oracle(default, oracle_results):
    for kind in ("vecchia", "vif", "fitc"):
        _check(default, oracle_results, kind)


@pytest.mark.parametrize("switch", ["STGP_VGRAD_SPLIT", "STGP_OZAKI_TRMM", "STGP_FITC_SYM_S"])
def test_switch_off_matches(default, oracle_results, switch):
    alt = _run(**{switch: "0"})
    for kind in ("vecchia", "vif", "fitc"):
        _check(alt, oracle_results, kind)
        # the alternative and the default path agree far inside the parity tolerance
        sc = oracle_results[kind][2]
        assert alt[kind][0] == pytest.approx(default[kind][0], rel=1e-11)
        assert O.grad_close(alt[kind][1:], default[kind][1:], sc, rtol=1e-10), (switch, kind, alt[kind] - default[kind])
    if switch == "STGP_VGRAD_SPLIT":  # the NLL comes from the same factor arithmetic
        assert alt["vecchia"][0] == default["vecchia"][0]
