"""Synthetic NOAA-shaped station x day data (host-side input generation).

Layout follows the reference simulator (simulate.cpp:32-51): stations uniform
in a box, every station observed on days 1..D, rows then ordered by
order_observations.  The response is a smooth random space-time field (random
Fourier features of a Gneiting-like spectrum) plus nugget noise: exact GP
draws are infeasible beyond the reference's own 20,000-point guard
(simulate.cpp:27-30), and the likelihood throughput does not depend on the
values of y.
"""
from __future__ import annotations

import numpy as np

# theta of PAPER.md section 4 (sigma2, sigma1_2, a, c, alpha, nu, beta, delta)
THETA_SEC4 = (0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2)
# NOAA temperature fit, Table 3; coordinates in metres
THETA_T3 = (1.539, 6.193, 0.090, 3.37e-6, 0.831, 1.5, 0.999, 1.667)

# BASELINE.json configs: (stations, days, box, theta)
CONFIGS = {
    "cfg1": dict(stations=500, days=20, box=(1.0, 1.0), theta=THETA_SEC4, m_v=10),
    "cfg2": dict(stations=1000, days=100, box=(1.0, 1.0), theta=THETA_SEC4, m_v=20),
    "cfg3": dict(stations=1000, days=100, box=(1.0, 1.0), theta=THETA_SEC4, m_v=20, m=200),
    "cfg4": dict(stations=10000, days=110, box=(4.6e6, 2.9e6), theta=THETA_T3, m_v=30, m=1000),
    "cfg5": dict(stations=10000, days=110, box=(4.6e6, 2.9e6), theta=THETA_T3, m=2000),
}


def station_day(stations: int, days: int, box=(1.0, 1.0), theta=THETA_SEC4, seed: int = 20260203,
                n_features: int = 64):
    """Unordered station x day points (x, y, t) and a synthetic response."""
    rng = np.random.default_rng(seed)
    sx = rng.uniform(0.0, box[0], stations)
    sy = rng.uniform(0.0, box[1], stations)
    t = np.repeat(np.arange(1, days + 1, dtype=np.float64), stations)
    x = np.tile(sx, days)
    y = np.tile(sy, days)
    sigma2, sigma1_2, a, c, alpha = theta[:5]
    # random Fourier features: spatial frequencies ~ c, temporal ~ sqrt(a)
    w = rng.normal(0.0, c, (n_features, 2))
    om = rng.normal(0.0, np.sqrt(a), n_features)
    ph = rng.uniform(0.0, 2 * np.pi, n_features)
    amp = np.sqrt(2.0 * sigma1_2 / n_features)
    field = np.zeros(len(t))
    for k in range(n_features):
        field += amp * np.cos(w[k, 0] * x + w[k, 1] * y + om[k] * t + ph[k])
    resp = field + rng.normal(0.0, np.sqrt(max(sigma2, 1e-12)), len(t))
    return x, y, t, resp


def config_data(name: str, seed: int = 20260203):
    c = CONFIGS[name]
    return station_day(c["stations"], c["days"], c["box"], c["theta"], seed)
