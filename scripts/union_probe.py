"""Locality probe (GPU): for tiles of R rows processed together, how many distinct W columns does
the union of their closures (neighbours + the row itself) touch?  This bounds the L2 traffic of a
tile-staged gather (union columns read once per tile) against the per-row gathers (m_v + 1 columns
per row).  Tiles: consecutive rows of (day, Morton(x, y)) order."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2602_03609_b200 as S  # noqa: E402

stations, days, m, mv = (int(a) for a in sys.argv[1:5])
theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(stations, days, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
ind = S.sts_kmeanspp(ds, m, 20260203)
nb = S.residual_neighbors(ds, theta, ind, mv)
N = nb.indices()
n = len(x)
lag = (np.arange(n)[:, None] - N)
tn = np.where(N >= 0, t[np.maximum(N, 0)], np.nan)
print("neighbour day lag histogram:", {int(d): int(c) for d, c in zip(*np.unique((t[:, None] - tn)[N >= 0], return_counts=True)) if c > n // 1000})


def spread(v):
    v = v.astype(np.uint64) & np.uint64(0xffff)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00ff00ff)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0f0f0f0f)
    v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
    return v


qx = ((x - x.min()) / (x.max() - x.min()) * 65535).astype(np.uint64)
qy = ((y - y.min()) / (y.max() - y.min()) * 65535).astype(np.uint64)
mort = spread(qx) | (spread(qy) << np.uint64(1))
order = np.lexsort((mort, t))
cl = np.concatenate([N, np.arange(n)[:, None]], axis=1)[order]
for R in (8, 16, 32, 64, 128):
    nt = n // R
    sizes = []
    for b in range(0, nt, max(1, nt // 4000)):
        blk = cl[b * R:(b + 1) * R].ravel()
        sizes.append(len(np.unique(blk[blk >= 0])))
    sizes = np.array(sizes)
    print(f"R={R:4d}: union mean {sizes.mean():7.1f} p90 {np.percentile(sizes, 90):7.1f} max {sizes.max():5d}"
          f"  per-row reads {(mv + 1):d} -> {sizes.mean() / R:6.2f} cols/row  ({(mv + 1) * R / sizes.mean():5.2f}x less)")
# random index order for comparison
for R in (16, 32):
    sizes = [len(np.unique(c[c >= 0])) for c in (np.concatenate([N, np.arange(n)[:, None]], axis=1)[b * R:(b + 1) * R].ravel() for b in range(0, n // R, n // R // 2000))]
    print(f"index order R={R}: union mean {np.mean(sizes):.1f}")
