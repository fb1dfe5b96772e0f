"""cfg4 VIF NLL+grad with the FP64 GEMMs on DMMA (STGP_OZAKI=0) vs the int8 Ozaki path at
S slices (STGP_OZAKI_S): prints the relative deviations (run once per setting)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

st, days = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "vif"
theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(st, days, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ds = S.SpaceTimeDataset(x, y, t, resp)
if kind == "fitc":
    ind = S.sts_kmeanspp(ds, 2000, 20260203)
    s = S.build_fitc(ds, theta, ind)
else:
    ind = S.sts_kmeanspp(ds, 1000, 20260203)
    nb = S.residual_neighbors(ds, theta, ind, 30)
    s = S.build_vif(ds, theta, ind, nb, S.OBSERVATION)
v, g = S.nll_and_grad(s, resp)
print(json.dumps({"kind": kind, "oz": os.environ.get("STGP_OZAKI", "1"), "S": os.environ.get("STGP_OZAKI_S", "6/7"),
                  "nll": v, "grad": [float(a) for a in g]}))
