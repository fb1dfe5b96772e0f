"""Generate the golden parity fixtures of the BASELINE.json configurations from the CPU oracle.

TEST INFRASTRUCTURE ONLY.  The oracle (oracle/stgp_oracle.cpp, the reference algorithm restated) is too
slow to run at these sizes inside the GPU test step, so its outputs are computed once here and committed;
the GPU tests (tests/test_gpu_configs.py) regenerate the same inputs (checked by a SHA-256 of the input
arrays) and compare the CUDA path with these values.

    python tests/golden/make_golden.py [case ...]      (cases: cfg2 cfg3 cfg4g cfg4s cfg5s; default all)

Searches and kMeans++ always run the sequential-order restatement (their outputs are defined bit for bit).
At M ~ 900-1900 the NLL / gradient / prediction of cfg4g and cfg5s take the oracle's BLAS mode for the
dense n x M^2 contractions (oracle.set_blas; it agrees with the sequential restatement to ~1e-14, see
tests/test_oracle_pinning.py::test_blas_mode_matches_sequential), which the tolerances dwarf.

Each case is one compressed .npz next to this script.  Full neighbour sets are stored as the SHA-256 of
their n x m_v int32 array (ascending, -1 padded) plus 2000 sampled rows for diagnosis.
"""
from __future__ import annotations

import hashlib
import importlib.util
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

_spec = importlib.util.spec_from_file_location("_synth", os.path.join(ROOT, "paper_2602_03609_b200", "synth.py"))
synth = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synth)

SEED = 20260203
BOX4 = (4.6e6, 2.9e6)

# name: (stations, days, box, theta, selection, m_v, m)
CASES = {
    # cfg2: n = 1e5 Vecchia, d_c m = 20, theta of PAPER.md section 4
    "cfg2": dict(stations=1000, days=100, box=(1.0, 1.0), theta=synth.THETA_SEC4, kind="vecchia", m_v=20),
    # cfg3: n = 1e5 VIF, sts m = 200 (M = 45 x 4 = 180), d_r m = 20
    "cfg3": dict(stations=1000, days=100, box=(1.0, 1.0), theta=synth.THETA_SEC4, kind="vif", m_v=20, m=200),
    # cfg4 geometry at n = 2e4: 1000 stations x 20 days in the cfg4 box, theta T3, m = 1000 -> M = 224 x 4 = 896
    # (>= 512: the default int8 Ozaki products are what is compared)
    "cfg4g": dict(stations=1000, days=20, box=BOX4, theta=synth.THETA_T3, kind="vif", m_v=30, m=1000,
                  blas=True),
    # cfg4 itself: sts (M = 906) and the d_r sets of 2000 sampled query rows against all their predecessors
    "cfg4s": dict(stations=10000, days=110, box=BOX4, theta=synth.THETA_T3, kind="dr-sample", m_v=30, m=1000,
                  rows=2000),
    # cfg5 shape at reduced n: FITC with sts m = 2000 on 2000 stations x 10 days (M = 632 x 3 = 1896), NLL,
    # gradient and the 1-day-ahead predictive mean / variance at every station
    "cfg5s": dict(stations=2000, days=10, box=BOX4, theta=synth.THETA_T3, kind="fitc", m=2000,
                  blas=True),
}


def inputs(c):
    x, y, t, r = synth.station_day(c["stations"], c["days"], box=c["box"], theta=c["theta"], seed=SEED)
    perm = O.order_observations(t, SEED)
    return x[perm], y[perm], t[perm], r[perm]


def input_sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def sets_sha(nbr) -> str:
    return hashlib.sha256(np.ascontiguousarray(nbr, dtype=np.int32).tobytes()).hexdigest()


def pack_sets(nbr):
    """full sets -> SHA-256 plus sampled rows"""
    rows = sampled_rows(len(nbr), min(2000, len(nbr) - 1))
    return {"nbr_sha": sets_sha(nbr), "nbr_rows": rows, "nbr_sample": np.ascontiguousarray(nbr[rows], dtype=np.int32)}


def sampled_rows(n, k, seed=SEED):
    rng = np.random.default_rng(seed ^ 0x5A)
    return np.sort(rng.choice(np.arange(1, n), size=k, replace=False)).astype(np.int32)


def make(name):
    c = CASES[name]
    O.set_blas(False)
    th = c["theta"]
    x, y, t, r = inputs(c)
    out = {"input_sha": input_sha(x, y, t, r), "theta": np.array(th)}
    t0 = time.time()
    if c["kind"] == "vecchia":
        nbr = O.dc_neighbors(x, y, t, th, c["m_v"])
        om = O.OracleModel("vecchia", x, y, t, th, nbr=nbr)
        out.update(**pack_sets(nbr), nll=om.nll(r))
        out["grad"], out["scale"] = om.nll_grad_scale(r)
    elif c["kind"] == "vif":
        Z, ms, mt = O.sts_kmeanspp(x, y, t, c["m"], SEED)
        nbr = O.dr_neighbors_rows(x, y, t, th, Z, c["m_v"])
        O.set_blas(bool(c.get("blas")), os.cpu_count() or 1)
        om = O.OracleModel("vif", x, y, t, th, nbr=nbr, Z=Z)
        out.update(Z=Z, ms=ms, mt=mt, **pack_sets(nbr), nll=om.nll(r))
        out["grad"], out["scale"] = om.nll_grad_scale(r)
    elif c["kind"] == "dr-sample":
        Z, ms, mt = O.sts_kmeanspp(x, y, t, c["m"], SEED)
        rows = sampled_rows(len(x), c["rows"])
        # m_v + 1 in (distance, index) order: the first m_v are the set, the gap to the next is the tie margin
        idx, dist = O.dr_neighbors_rows(x, y, t, th, Z, c["m_v"] + 1, rows=rows, with_dist=True, by_dist=True)
        m = c["m_v"]
        sets = np.sort(np.where(idx[:, :m] >= 0, idx[:, :m], np.iinfo(np.int32).max), axis=1)
        sets = np.where(sets == np.iinfo(np.int32).max, -1, sets).astype(np.int32)
        out.update(Z=Z, ms=ms, mt=mt, rows=rows, sets=sets, dist=dist[:, :m],
                   gap=dist[:, m] - dist[:, m - 1])
    elif c["kind"] == "fitc":
        Z, ms, mt = O.sts_kmeanspp(x, y, t, c["m"], SEED)
        O.set_blas(bool(c.get("blas")), os.cpu_count() or 1)
        om = O.OracleModel("fitc", x, y, t, th, Z=Z)
        out.update(Z=Z, ms=ms, mt=mt, nll=om.nll(r))
        out["grad"], out["scale"] = om.nll_grad_scale(r)
        last = t == t.max()
        targets = np.column_stack([x[last], y[last], np.full(int(last.sum()), t.max() + 1.0)])
        mu, var = om.predict(r, targets, 0)
        out.update(targets=targets, mu=mu, var=var)
    out["oracle_s"] = time.time() - t0
    out["dense"] = "openblas" if c.get("blas") else "sequential"
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {time.time() - t0:.1f} s -> {os.path.getsize(path) / 1e6:.2f} MB", flush=True)


if __name__ == "__main__":
    O.set_threads(os.cpu_count() or 1)
    for name in (sys.argv[1:] or list(CASES)):
        make(name)
