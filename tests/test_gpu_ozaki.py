"""FP64 products on the int8 tensor cores (csrc/ozaki.cu) against exact references.

The Ozaki slicing is error-free apart from the dropped low-order diagonals, so the error of each
entry is bounded by ~2^-(7 S) * k * max|A_r| * max|B_j| (S = 6 slices for the row form X = K^-1 V',
7 for the long reductions, by default).  The
reference is math.fsum over the rounded products (error k 2^-53 max|a| max|b|, far inside the bound).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROWS_SLICES = 6  # csrc/ozaki.cu slices_for("STGP_OZAKI_S_ROWS", 6)
ROWS_TOL = 2.0 ** -(7 * ROWS_SLICES - 3)  # truncation of both operands plus the dropped diagonals


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_03609_b200 as S
    return S.Context(0)


def _exact(A, B):
    out = np.empty((A.shape[0], B.shape[0]))
    for r in range(A.shape[0]):
        for j in range(B.shape[0]):
            out[r, j] = math.fsum(A[r] * B[j])  # rounded products: error <= k 2^-53 max|a||b|, far inside the bound
    return out


@pytest.mark.parametrize("n,m,k", [(37, 24, 40), (300, 48, 912)])
def test_ozaki_matches_exact_dot(ctx, n, m, k):
    rng = np.random.default_rng(n + k)
    # rows spanning many binades and signs, some zero rows
    A = rng.standard_normal((n, k)) * np.exp2(rng.integers(-30, 30, size=(n, 1)))
    B = rng.standard_normal((m, k)) * np.exp2(rng.integers(-20, 20, size=(m, 1)))
    A[3] = 0.0
    B[1, ::2] = 0.0
    C, _ = ctx.gemm_rows(A, B, emulated=True)
    ref = _exact(A[:40], B)
    scale = np.abs(A[:40]).max(axis=1)[:, None] * np.abs(B).max(axis=1)[None, :] * k
    err = np.abs(C[:40] - ref)
    assert (err <= ROWS_TOL * scale).all(), (err / np.maximum(scale, 1e-300)).max()
    assert (C[3] == 0.0).all()
    D, _ = ctx.gemm_rows(A, B, emulated=False)
    assert np.allclose(C, D, rtol=0, atol=2 * ROWS_TOL * np.abs(A).max(axis=1)[:, None] * np.abs(B).max(axis=1)[None, :] * k)


def test_ozaki_cfg4_shape_timing(ctx):
    # the X = K^{-1} V' shape of the VIF gradient (n x 912 rows against a 912 x 912 symmetric matrix)
    rng = np.random.default_rng(1)
    n, M = 200000, 912
    A = rng.standard_normal((n, M))
    B = rng.standard_normal((M, M))
    B = B + B.T
    C, ms_e = ctx.gemm_rows(A, B, emulated=True)
    D, ms_d = ctx.gemm_rows(A, B, emulated=False)
    scale = np.abs(A).max(axis=1)[:, None] * np.abs(B).max(axis=1)[None, :] * M
    assert (np.abs(C - D) <= 2 * ROWS_TOL * scale).all()
    print(f"ozaki {ms_e:.2f} ms vs DGEMM {ms_d:.2f} ms at n={n}")


TRMM_SLICES = 7  # csrc/ozaki.cu slices_for("STGP_OZAKI_S_TRMM", 7)
TRMM_TOL = 2.0 ** -(7 * TRMM_SLICES - 3)


@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("m,n", [(212, 1500), (912, 600)])
def test_ozaki_trmm(ctx, m, n, transpose):
    # W = L^{-1} U / omega = L^{-T} omega' shapes: T the inverse Cholesky factor of an ill-conditioned
    # SPD matrix (rows of very different magnitude, cancelling signs), B with columns over many binades
    rng = np.random.default_rng(m + n + transpose)
    P = rng.random((m, 2))
    Kc = np.exp(-np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1)) / 0.3) + 1e-6 * np.eye(m)
    T = np.tril(np.linalg.inv(np.linalg.cholesky(Kc)))
    B = rng.standard_normal((m, n)) * np.exp2(rng.integers(-20, 20, size=(1, n)))
    B[:, 5] = 0.0
    C1, _ = ctx.trmm(T, B, transpose, mode=1)
    C2, _ = ctx.trmm(T, B, transpose, mode=2)
    assert np.array_equal(C1, C2)  # the skipped K steps hold only zero digits: the int32 sums are identical
    assert (C1[:, 5] == 0.0).all()
    opT = T.T if transpose else T
    cols = list(range(0, n, max(1, n // 40)))
    ref = np.array([[math.fsum(opT[j] * B[:, r]) for r in cols] for j in range(m)])
    scale = np.abs(opT).max(axis=1)[:, None] * np.abs(B[:, cols]).max(axis=0)[None, :] * m
    err = np.abs(C1[:, cols] - ref)
    assert (err <= TRMM_TOL * scale).all(), (err / np.maximum(scale, 1e-300)).max()
    D, _ = ctx.trmm(T, B, transpose, mode=0)
    full = np.abs(opT).max(axis=1)[:, None] * np.abs(B).max(axis=0)[None, :] * m
    assert (np.abs(C1 - D) <= 2 * TRMM_TOL * full).all()


def test_ozaki_trmm_cfg4_timing(ctx):
    # the cfg4 shape (M = 912) over 200k columns: triangle-cut int8 product vs the DMMA TRMM
    rng = np.random.default_rng(3)
    m, n = 912, 200000
    T = np.tril(rng.standard_normal((m, m))) + m * np.eye(m)
    B = rng.standard_normal((m, n))
    C1, ms1 = ctx.trmm(T, B, False, mode=1)
    _, ms2 = ctx.trmm(T, B, False, mode=2)
    D, ms0 = ctx.trmm(T, B, False, mode=0)
    full = np.abs(T).max(axis=1)[:, None] * np.abs(B).max(axis=0)[None, :] * m
    assert (np.abs(C1 - D) <= 2 * TRMM_TOL * full).all()
    print(f"trmm ozaki {ms1:.2f} ms (full K {ms2:.2f}) vs DMMA {ms0:.2f} ms at n={n}")


@pytest.mark.parametrize("n,m", [(1000, 40), (300001, 96)])
def test_ozaki_long_reduction(ctx, n, m):
    # C = A^T B over n rows in exact int32 chunks (the K = S S^T and V' F^T shapes), per-chunk scales
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, m)) * np.exp2(rng.integers(-8, 8, size=(n, 1)))
    B = rng.standard_normal((n, m))
    C, _ = ctx.gemm_cols(A, B)
    ref = A.T @ B
    # slicing error is relative to the per-chunk row maxima: <= ~2^-46 n max|A[:, j]| max|B[:, i]|
    bound = 2.0 ** -44 * n * np.abs(A).max(axis=0)[:, None] * np.abs(B).max(axis=0)[None, :]
    assert (np.abs(C - ref) <= bound).all(), (np.abs(C - ref) / bound).max()
    G, _ = ctx.gemm_cols(A)  # A^T A: exactly symmetric
    assert (G == G.T).all()
    assert np.allclose(G, A.T @ A, rtol=0, atol=2.0 ** -44 * n * np.abs(A).max() ** 2)


def test_ozaki_long_reduction_timing(ctx):
    rng = np.random.default_rng(2)
    n, m = 400000, 912
    A = rng.standard_normal((n, m))
    B = rng.standard_normal((n, m))
    C, ms_e = ctx.gemm_cols(A, B)
    D, ms_d = ctx.gemm_cols(A, B, emulated=False)
    assert np.allclose(C, D, rtol=0, atol=2.0 ** -40 * n)
    print(f"ozaki cols {ms_e:.2f} ms vs DGEMM {ms_d:.2f} ms at n={n}")


_FITC_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_2602_03609_b200 as S
from oracle import oracle as O
x, y, t, yv, X = O.test_dataset(1, 1500, 47, n_times=8, p=1)
rng = np.random.default_rng(9)
Z = np.column_stack([rng.random(40), rng.random(40), 1 + 7 * rng.random(40)])
th = (0.2, 1.1, 0.8, 12.0, 0.6, 1.5, 0.3, 0.5)
s = S.build_fitc(S.SpaceTimeDataset(x, y, t), th, S.InducingSet.from_points(Z))
v, g = S.nll_and_grad(s, yv, X, np.array([-0.2]))
print(json.dumps({"nll": v, "grad": list(map(float, g))}))
"""


def test_ozaki_products_inside_fitc_match_oracle():
    # FITC's K, K^-1 W and W diag(phi) W^T forced onto the int8 path at test size
    import json
    import os
    import subprocess
    import sys
    from oracle import oracle as O
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, STGP_OZAKI_MIN_M="0")
    r = subprocess.run([sys.executable, "-c", _FITC_SCRIPT % dict(root=root)], env=env, capture_output=True, text=True,
                       timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    a = json.loads(r.stdout.strip().splitlines()[-1])
    x, y, t, yv, X = O.test_dataset(1, 1500, 47, n_times=8, p=1)
    rng = np.random.default_rng(9)
    Z = np.column_stack([rng.random(40), rng.random(40), 1 + 7 * rng.random(40)])
    th = (0.2, 1.1, 0.8, 12.0, 0.6, 1.5, 0.3, 0.5)
    om = O.OracleModel("fitc", x, y, t, th, Z=Z)
    beta = np.array([-0.2])
    gr, sc = om.nll_grad_scale(yv, X, beta)
    assert a["nll"] == pytest.approx(om.nll(yv, X, beta), rel=1e-8)
    g = np.array(a["grad"])
    assert O.grad_close(g, gr, sc), (g, gr, sc)
