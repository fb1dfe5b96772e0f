"""order_observations (dataset.cpp:81-114): the engine's host permutation equals the oracle's, element for
element -- stable sort by t, then a seeded Fisher-Yates within each equal-t block from one
mt19937_64(mix_seed(seed, 0x0bde11)).  Runs on the CPU (host code of the C ABI, no device calls)."""
import numpy as np
import pytest

from oracle import oracle as O


@pytest.fixture(scope="module")
def S():
    import paper_2602_03609_b200 as S
    return S


@pytest.mark.parametrize("case", ["cfg4", "cfg2", "ties", "unsorted", "irregular", "single"])
def test_engine_order_equals_oracle(S, case):
    rng = np.random.default_rng(7)
    seed = 20260203
    if case == "cfg4":
        _, _, t, _ = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), seed=seed, n_features=1)
    elif case == "cfg2":
        _, _, t, _ = S.synth.station_day(1000, 100, seed=seed, n_features=1)
    elif case == "ties":
        t = rng.integers(0, 5, 5000).astype(np.float64)
    elif case == "unsorted":
        t = rng.permutation(np.repeat(np.arange(50.0), 37))
        seed = 3
    elif case == "irregular":
        t = np.round(rng.exponential(2.0, 4000), 3) - 1.5  # negative and fractional times, ties
    else:
        t = np.array([4.0])
    a = S.order_observations_perm(t, seed)
    b = O.order_observations(t, seed)
    assert (a == b).all()
    assert (np.diff(t[a]) >= 0).all()
