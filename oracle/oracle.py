"""ctypes binding of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, where it is the checker or the
timed CPU baseline -- never the product path.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

ERRORS = {2: "ConfigError", 3: "DataError", 4: "NumericError", 1: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")


class Params(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("sigma2", "sigma1_2", "a", "c", "alpha", "nu", "beta", "delta")]


class Model(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("policy", C.c_int), ("n", C.c_int),
        ("x", C.c_void_p), ("y", C.c_void_p), ("t", C.c_void_p),
        ("nbr", C.c_void_p), ("m_v", C.c_int), ("M", C.c_int),
        ("zx", C.c_void_p), ("zy", C.c_void_p), ("zt", C.c_void_p),
        ("theta", Params),
    ]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_exp.restype = C.c_double
        _lib.orc_exp.argtypes = [C.c_double]
        _lib.orc_kernel_eval.restype = C.c_double
        _lib.orc_kernel_eval.argtypes = [C.POINTER(Params), C.c_double, C.c_double]
        _lib.orc_dc_pair.restype = C.c_double
        _lib.orc_dc_pair.argtypes = [C.POINTER(Params)] + [C.c_double] * 6
        _lib.orc_mix_seed.restype = C.c_uint64
        _lib.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _chk(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def params(theta) -> Params:
    if isinstance(theta, Params):
        return theta
    if isinstance(theta, dict):
        return Params(**theta)
    if hasattr(theta, "as_tuple"):
        return Params(*theta.as_tuple())
    return Params(*theta)


def set_threads(n: int) -> int:
    return lib().orc_set_threads(int(n))


def set_prune(on: bool):
    lib().orc_set_prune(int(bool(on)))


def kernel_eval(theta, h, u) -> float:
    return lib().orc_kernel_eval(C.byref(params(theta)), float(h), float(u))


def kernel_grad(theta, h, u) -> np.ndarray:
    g = np.zeros(6)
    _chk(lib().orc_kernel_grad(C.byref(params(theta)), C.c_double(h), C.c_double(u), _p(g)))
    return g


def effective_ranges(theta):
    tr, sr = C.c_double(), C.c_double()
    _chk(lib().orc_effective_ranges(C.byref(params(theta)), C.byref(tr), C.byref(sr)))
    return tr.value, sr.value


def mix_seed(seed: int, stream: int) -> int:
    return int(lib().orc_mix_seed(seed, stream))


def exp(x: float) -> float:
    return lib().orc_exp(float(x))


def exp_array(x) -> np.ndarray:
    """host glibc exp, element-wise (numpy's exp is not glibc's)."""
    x = _f64(x)
    out = np.zeros_like(x)
    lib().orc_exp_array(C.c_long(len(x)), _p(x), _p(out))
    return out


def order_observations(t, seed: int) -> np.ndarray:
    t = _f64(t)
    perm = np.zeros(len(t), dtype=np.int32)
    _chk(lib().orc_order_observations(C.c_int(len(t)), _p(t), C.c_uint64(seed), _p(perm)))
    return perm


def test_dataset(kind: int, n: int, seed: int, n_times: int = 10, p: int = 0):
    """Reference test-suite datasets (see orc_test_dataset)."""
    nn = n * n_times if kind == 2 else n
    x, y, t, yv = (np.zeros(nn) for _ in range(4))
    X = np.zeros((nn, max(p, 0)), order="F")
    _chk(lib().orc_test_dataset(kind, n, C.c_uint64(seed), n_times, p, _p(x), _p(y), _p(t), _p(yv),
                                _p(X) if p > 0 else None))
    return x, y, t, yv, X


def dc_pair(theta, a, b) -> float:
    return lib().orc_dc_pair(C.byref(params(theta)), *map(float, a), *map(float, b))


def dc_neighbors(x, y, t, theta, m_v: int, with_dist: bool = False):
    x, y, t = _f64(x), _f64(y), _f64(t)
    n = len(x)
    out = np.zeros((n, m_v), dtype=np.int32)
    dist = np.zeros((n, m_v)) if with_dist else None
    _chk(lib().orc_dc_neighbors(n, _p(x), _p(y), _p(t), C.byref(params(theta)), m_v, _p(out), _p(dist)))
    return (out, dist) if with_dist else out


def dc_neighbors_range(x, y, t, theta, m_v: int, q0: int, q1: int):
    x, y, t = _f64(x), _f64(y), _f64(t)
    out = np.zeros((q1 - q0, m_v), dtype=np.int32)
    _chk(lib().orc_dc_neighbors_range(len(x), _p(x), _p(y), _p(t), C.byref(params(theta)), m_v, q0, q1, _p(out)))
    return out


def dr_neighbors(x, y, t, theta, Z, m_v: int, with_dist: bool = False, with_w: bool = False):
    x, y, t = _f64(x), _f64(y), _f64(t)
    Z = np.asarray(Z, dtype=np.float64).reshape(-1, 3)
    zx, zy, zt = _f64(Z[:, 0]), _f64(Z[:, 1]), _f64(Z[:, 2])
    n, M = len(x), len(Z)
    out = np.zeros((n, m_v), dtype=np.int32)
    dist = np.zeros((n, m_v)) if with_dist else None
    W = np.zeros((n, M)) if with_w else None  # column-major M x n == row-major n x M
    resid = np.zeros(n) if with_w else None
    _chk(lib().orc_dr_neighbors(n, _p(x), _p(y), _p(t), C.byref(params(theta)), M, _p(zx), _p(zy), _p(zt),
                                m_v, _p(out), _p(dist), _p(W), _p(resid)))
    res = [out]
    if with_dist:
        res.append(dist)
    if with_w:
        res += [W, resid]
    return res[0] if len(res) == 1 else tuple(res)


def euclid_neighbors(x, y, t, m_v: int, ss: float, ts: float):
    x, y, t = _f64(x), _f64(y), _f64(t)
    n = len(x)
    out = np.zeros((n, m_v), dtype=np.int32)
    _chk(lib().orc_euclid_neighbors(n, _p(x), _p(y), _p(t), m_v, C.c_double(ss), C.c_double(ts), _p(out)))
    return out


def kmeanspp(points, k: int, seed: int) -> np.ndarray:
    P = np.asfortranarray(np.asarray(points, dtype=np.float64).reshape(len(points), -1))
    n, d = P.shape
    out = np.zeros((k, d), order="F")
    _chk(lib().orc_kmeanspp(_p(P), n, d, k, C.c_uint64(seed), _p(out)))
    return np.ascontiguousarray(out)


def sts_kmeanspp(x, y, t, m: int, seed: int):
    x, y, t = _f64(x), _f64(y), _f64(t)
    cap = max(m, 1) * 4 + 16
    out = np.zeros((cap, 3))
    ms, mt = C.c_int(), C.c_int()
    _chk(lib().orc_sts_kmeanspp(len(x), _p(x), _p(y), _p(t), m, C.c_uint64(seed), C.byref(ms), C.byref(mt), _p(out), cap))
    return out[: ms.value * mt.value].copy(), ms.value, mt.value


def joint_kmeanspp(x, y, t, m: int, ss: float, ts: float, seed: int):
    x, y, t = _f64(x), _f64(y), _f64(t)
    out = np.zeros((m, 3))
    k = C.c_int()
    _chk(lib().orc_joint_kmeanspp(len(x), _p(x), _p(y), _p(t), m, C.c_double(ss), C.c_double(ts), C.c_uint64(seed),
                                  C.byref(k), _p(out), m))
    return out[: k.value].copy()


KIND = {"vecchia": 0, "fitc": 1, "vif": 2}


class OracleModel:
    """A model description for the oracle's structure functions."""

    def __init__(self, kind, x, y, t, theta, nbr=None, Z=None, policy="observation"):
        self._keep = []
        self.x, self.y, self.t = _f64(x), _f64(y), _f64(t)
        self.n = len(self.x)
        self.nbr = None if nbr is None else np.ascontiguousarray(nbr, dtype=np.int32)
        m_v = 0 if self.nbr is None else self.nbr.shape[1]
        if self.nbr is None:
            self.nbr = np.zeros((self.n, 1), dtype=np.int32) - 1
            m_v = 1
        Z = np.zeros((0, 3)) if Z is None else np.asarray(Z, dtype=np.float64).reshape(-1, 3)
        self.zx, self.zy, self.zt = _f64(Z[:, 0]), _f64(Z[:, 1]), _f64(Z[:, 2])
        self.m = Model(KIND[kind] if isinstance(kind, str) else kind,
                       1 if policy in ("observation", 1) else 0, self.n,
                       _p(self.x), _p(self.y), _p(self.t), _p(self.nbr), m_v, len(Z),
                       _p(self.zx), _p(self.zy), _p(self.zt), params(theta))

    @staticmethod
    def _xb(n, X, beta):
        if X is None or beta is None or np.size(beta) == 0:
            return 0, None, None
        X = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(n, -1))
        return X.shape[1], X, _f64(beta)

    def rows(self):
        D = np.zeros(self.n)
        A = np.zeros(self.nbr.shape)
        _chk(lib().orc_build_rows(C.byref(self.m), _p(D), _p(A)))
        return D, A

    def fitc_diag(self):
        d = np.zeros(self.n)
        _chk(lib().orc_fitc_diag(C.byref(self.m), _p(d)))
        return d

    def nll(self, yv, X=None, beta=None) -> float:
        p, Xf, b = self._xb(self.n, X, beta)
        yv = _f64(yv)
        out = C.c_double()
        _chk(lib().orc_nll(C.byref(self.m), _p(yv), p, _p(Xf), _p(b), C.byref(out)))
        return out.value

    def nll_grad(self, yv, X=None, beta=None) -> np.ndarray:
        p, Xf, b = self._xb(self.n, X, beta)
        yv = _f64(yv)
        g = np.zeros(7)
        _chk(lib().orc_nll_grad(C.byref(self.m), _p(yv), p, _p(Xf), _p(b), _p(g)))
        return g

    def nll_grad_scale(self, yv, X=None, beta=None):
        """(gradient, scale): scale[k] = sum over rows of |row contribution to component k| (the
        conditioning of the gradient sum; parity tolerances are 1e-8 * scale)."""
        p, Xf, b = self._xb(self.n, X, beta)
        yv = _f64(yv)
        g, sc = np.zeros(7), np.zeros(7)
        _chk(lib().orc_nll_grad_scale(C.byref(self.m), _p(yv), p, _p(Xf), _p(b), _p(g), _p(sc)))
        return g, sc

    def gls_beta(self, yv, X) -> np.ndarray:
        X = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(self.n, -1))
        yv = _f64(yv)
        out = np.zeros(X.shape[1])
        _chk(lib().orc_gls_beta(C.byref(self.m), _p(yv), X.shape[1], _p(X), _p(out)))
        return out

    def predict(self, yv, targets, pred_m_v: int, X=None, beta=None, Xp=None):
        p, Xf, b = self._xb(self.n, X, beta)
        T = np.asarray(targets, dtype=np.float64).reshape(-1, 3)
        qx, qy, qt = _f64(T[:, 0]), _f64(T[:, 1]), _f64(T[:, 2])
        npred = len(T)
        Xpf = None if Xp is None or p == 0 else np.asfortranarray(np.asarray(Xp, dtype=np.float64).reshape(npred, -1))
        mu, var = np.zeros(npred), np.zeros(npred)
        yv = _f64(yv)
        _chk(lib().orc_predict(C.byref(self.m), _p(yv), p, _p(Xf), _p(b), npred, _p(qx), _p(qy), _p(qt), _p(Xpf),
                               pred_m_v, _p(mu), _p(var)))
        return mu, var


def dense_nll(x, y, t, theta, yv, X=None, beta=None) -> float:
    x, y, t, yv = _f64(x), _f64(y), _f64(t), _f64(yv)
    p, Xf, b = OracleModel._xb(len(x), X, beta)
    out = C.c_double()
    _chk(lib().orc_dense_nll(len(x), _p(x), _p(y), _p(t), C.byref(params(theta)), _p(yv), p, _p(Xf), _p(b), C.byref(out)))
    return out.value


def dense_predict(x, y, t, theta, yv, targets):
    x, y, t, yv = _f64(x), _f64(y), _f64(t), _f64(yv)
    T = np.asarray(targets, dtype=np.float64).reshape(-1, 3)
    qx, qy, qt = _f64(T[:, 0]), _f64(T[:, 1]), _f64(T[:, 2])
    mu, var = np.zeros(len(T)), np.zeros(len(T))
    _chk(lib().orc_dense_predict(len(x), _p(x), _p(y), _p(t), C.byref(params(theta)), _p(yv), len(T), _p(qx), _p(qy),
                                 _p(qt), _p(mu), _p(var)))
    return mu, var


def full_conditioning(n: int) -> np.ndarray:
    """test_approximations.cpp:34-43: N(i) = {0..i-1}."""
    nb = np.full((n, max(n - 1, 1)), -1, dtype=np.int32)
    for i in range(1, n):
        nb[i, :i] = np.arange(i)
    return nb


# ---------------------------------------------------------------------------
# fit (estimation.cpp:121-263, 423-619), Gaussian likelihood: the checker of the device fit driver.
# Data are the ordered arrays (FittedModel.data).  Objective values and gradients come from the
# oracle structures above; the selection is rebuilt with the oracle searches.
# ---------------------------------------------------------------------------
_BOUNDARY_EPS = 1e-6


def _sigmoid(z):
    if z >= 0.0:
        return 1.0 / (1.0 + math.exp(-z))
    e = math.exp(z)
    return e / (1.0 + e)


def _to_z(th):  # estimation.cpp:126-147
    s2, s1, a, c, al, nu, be, de = th
    lg = lambda p: math.log(p / (1.0 - p))  # noqa: E731
    return np.array([math.log(max(s2, 1e-12)), math.log(s1), math.log(a), math.log(c),
                     lg(min(max(al, _BOUNDARY_EPS), 1 - _BOUNDARY_EPS)), lg(min(max(be, _BOUNDARY_EPS), 1 - _BOUNDARY_EPS)),
                     math.log(max(de, 1e-8))])


def _exp(v):
    return math.exp(v) if v < 709.78 else math.inf


def _theta_of(z, nu):  # estimation.cpp:149-159; CovarianceParams::validate (covariance.cpp:34-46)
    th = (_exp(z[0]), _exp(z[1]), _exp(z[2]), _exp(z[3]),
          min(max(_sigmoid(z[4]), _BOUNDARY_EPS), 1.0), nu, min(max(_sigmoid(z[5]), 0.0), 1.0), _exp(z[6]))
    s2, s1, a, c, al, _, be, de = th
    ok = (0 <= s2 < math.inf and 0 < s1 < math.inf and 0 < a < math.inf and 0 < c < math.inf and 0 < al <= 1
          and 0 <= be <= 1 and 0 <= de < math.inf)
    if not ok:
        raise OracleError(2, "CovarianceParams: parameter out of range")
    return th


def _dtheta_dz(z):  # estimation.cpp:167-188
    sa, sb = _sigmoid(z[4]), _sigmoid(z[5])
    return np.array([math.exp(z[0]), math.exp(z[1]), math.exp(z[2]), math.exp(z[3]), sa * (1 - sa), sb * (1 - sb),
                     math.exp(z[6])])


class _Lbfgs:  # estimation.cpp:234-263
    def __init__(self):
        self.pairs = []

    def reset(self):
        self.pairs = []

    def push(self, s, y):
        if s.dot(y) > 1e-12 * np.linalg.norm(s) * np.linalg.norm(y):
            self.pairs.append((s, y))
            if len(self.pairs) > 10:
                self.pairs.pop(0)

    def direction(self, g):
        q = -g.copy()
        if not self.pairs:
            return q
        al = [0.0] * len(self.pairs)
        for i in range(len(self.pairs) - 1, -1, -1):
            s, y = self.pairs[i]
            al[i] = (1.0 / s.dot(y)) * s.dot(q)
            q = q - al[i] * y
        s, y = self.pairs[-1]
        q = q * (s.dot(y) / y.dot(y))
        for i, (s, y) in enumerate(self.pairs):
            bc = (1.0 / s.dot(y)) * y.dot(q)
            q = q + (al[i] - bc) * s
        return q


def _selection(x, y, t, method, m_v, m, seed, th):  # estimation.cpp:197-231
    tr, sr = effective_ranges(th)
    ss = sr if math.isfinite(sr) and sr > 0 else 1.0
    ts = tr if math.isfinite(tr) and tr > 0 else 1e6
    if method == "vecchia-euclid":
        return "vecchia", euclid_neighbors(x, y, t, m_v, ss, ts), None
    if method == "vecchia-corr":
        return "vecchia", dc_neighbors(x, y, t, th, m_v), None
    if method == "fitc-kmeanspp":
        return "fitc", None, joint_kmeanspp(x, y, t, m, ss, ts, seed)
    if method == "fitc-sts":
        return "fitc", None, sts_kmeanspp(x, y, t, m, seed)[0]
    Z = sts_kmeanspp(x, y, t, m, seed)[0]
    return "vif", dr_neighbors(x, y, t, th, Z, m_v), Z


def fit_gaussian(x, y, t, yv, X, method, m_v, m, seed, nu, init, max_iterations=200, tol_objective=1e-8,
                 tol_gradient=1e-5):
    """estimation.cpp:423-619 (Gaussian path) on ordered data; returns (theta, beta, f, converged, trace)."""
    n = len(x)
    p = 0 if X is None else np.asarray(X).reshape(n, -1).shape[1]
    X = None if p == 0 else np.asarray(X, dtype=np.float64).reshape(n, p)
    th0 = tuple(init)
    th0 = th0[:5] + (nu,) + th0[6:]
    z = _to_z(th0)
    beta = np.linalg.solve(X.T @ X, X.T @ yv) if p else None
    sel = None

    def model(zz):
        kind, nbr, Z = sel
        return OracleModel(kind, x, y, t, _theta_of(zz, nu), nbr=nbr, Z=Z)

    def value(zz):
        return model(zz).nll(yv, X, beta)

    def grad(zz):
        return model(zz).nll_grad(yv, X, beta) * _dtheta_dz(zz)

    lb = _Lbfgs()
    f, g = float("nan"), None
    have, done, conv, term = False, False, False, 0
    trace = []
    for it in range(1, max_iterations + 1):
        if done:
            break
        refreshed = False
        sched = (it & (it - 1)) == 0
        if sched or not have:
            sel = _selection(x, y, t, method, m_v, m, seed, _theta_of(z, nu))
            refreshed = sched
            fn = value(z)
            if have and abs(fn - f) > tol_objective * max(1.0, abs(f)):
                lb.reset()
            f = fn
            g = grad(z)
            have = True
        if p:
            beta = model(z).gls_beta(yv, X)
            f = value(z)
            g = grad(z)
        gn = float(np.abs(g).max())
        trace.append((it, f, gn, refreshed))
        if gn < tol_gradient and len(trace) >= 2 and abs(trace[-2][1] - f) < tol_objective * max(1.0, abs(f)):
            rs = _selection(x, y, t, method, m_v, m, seed, _theta_of(z, nu))
            old, sel = sel, rs
            fr = value(z)
            if abs(fr - f) <= tol_objective * max(1.0, abs(f)) or term >= 3:
                f = fr
                trace.append((it, f, gn, True))
                conv, done = True, True
                break
            f = fr
            g = grad(z)
            lb.reset()
            term += 1
            trace.append((it, f, gn, True))
            continue
        d = lb.direction(g)
        if d.dot(g) >= 0.0:
            d = -g
        step, slope, acc = 1.0, g.dot(d), False
        for _ in range(40):
            zn = z + step * d
            try:
                ft = value(zn)
            except OracleError as e:
                if e.code != 4:
                    raise
                step *= 0.5
                continue
            if math.isfinite(ft) and ft <= f + 1e-4 * step * slope:
                fnew, acc = ft, True
                break
            step *= 0.5
        if not acc:
            if gn < tol_gradient * 10.0:
                conv = True
            break
        gnew = grad(zn)
        lb.push(zn - z, gnew - g)
        z, f, g = zn, fnew, gnew
    return _theta_of(z, nu), beta, f, conv, trace


def dr_neighbors_rows(x, y, t, theta, Z, m_v: int, rows=None, with_dist: bool = False, by_dist: bool = False):
    """residual_neighbors for the given query rows (time-ordered data) with certified exact pruning
    (orc_dr_neighbors_rows); rows None = all rows.  Equal to dr_neighbors on those rows.  by_dist: each
    row's indices in (distance, index) order instead of ascending."""
    x, y, t = _f64(x), _f64(y), _f64(t)
    Z = np.asarray(Z, dtype=np.float64).reshape(-1, 3)
    zx, zy, zt = _f64(Z[:, 0]), _f64(Z[:, 1]), _f64(Z[:, 2])
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    nq = len(x) if r is None else len(r)
    out = np.zeros((nq, m_v), dtype=np.int32)
    dist = np.zeros((nq, m_v)) if with_dist else None
    _chk(lib().orc_dr_neighbors_rows(len(x), _p(x), _p(y), _p(t), C.byref(params(theta)), len(Z), _p(zx), _p(zy),
                                     _p(zt), m_v, nq, _p(r), _p(out), _p(dist), int(by_dist)))
    return (out, dist) if with_dist else out


def openblas_path():
    """the scipy-bundled OpenBLAS (LP64, scipy_* symbols) of this image, or None"""
    import glob
    import scipy
    libs = glob.glob(os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)), "scipy.libs",
                                  "libscipy_openblas-*.so"))
    return libs[0] if libs else None


def set_blas(on: bool = True, threads: int = 0) -> bool:
    """BLAS timing mode (orc_set_blas): the dense n x M^2 contractions go to OpenBLAS; off restores the
    sequential-order restatement the parity tests use.  Returns whether BLAS is active."""
    path = openblas_path() if on else None
    if on and path is None:
        return False
    _chk(lib().orc_set_blas(path.encode() if path else None, int(threads)))
    return on


def zcptn(y, mu, sigma, lam):
    """(loglik, d1, d2) of the ZC-PTN observation model (laplace.cpp:56-91)."""
    out = np.zeros(3)
    _chk(lib().orc_zcptn(C.c_double(y), C.c_double(mu), C.c_double(sigma), C.c_double(lam), _p(out)))
    return tuple(out)


def normal_tail(z):
    """(norm_cdf, log_norm_cdf, inverse_mills) (laplace.cpp:25-54)."""
    out = np.zeros(3)
    lib().orc_normal_tail(C.c_double(z), _p(out))
    return tuple(out)


def laplace_marginal(om: "OracleModel", yv, lik_sigma: float, lik_lambda: float, X=None, beta=None, warm=None):
    """laplace_marginal (laplace.cpp:115-203), ZC-PTN likelihood: (negative log-marginal, state dict)."""
    p, Xf, b = OracleModel._xb(om.n, X, beta)
    yv = _f64(yv)
    n = om.n
    mode, ga, w = np.zeros(n), np.zeros(n), np.zeros(n)
    out, it = C.c_double(), C.c_int()
    wm = None if warm is None else _f64(warm)
    _chk(lib().orc_laplace_marginal(C.byref(om.m), _p(yv), p, _p(Xf), _p(b), C.c_double(lik_sigma),
                                    C.c_double(lik_lambda), _p(wm), C.byref(out), _p(mode), _p(ga), _p(w),
                                    C.byref(it)))
    return out.value, {"mode": mode, "grad_at_mode": ga, "w": w, "iterations": it.value}


def zcptn_predict(om: "OracleModel", state, targets, lik_sigma: float, lik_lambda: float, pred_m_v: int,
                  n_samples: int, seed: int, Xp=None, beta=None):
    """zcptn_predict (laplace.cpp:205-259): latent moments, P(rain), Monte Carlo amounts and draws."""
    T = np.asarray(targets, dtype=np.float64).reshape(-1, 3)
    qx, qy, qt = _f64(T[:, 0]), _f64(T[:, 1]), _f64(T[:, 2])
    npred = len(T)
    p = 0 if Xp is None or beta is None else np.asarray(Xp).reshape(npred, -1).shape[1]
    Xpf = None if p == 0 else np.asfortranarray(np.asarray(Xp, dtype=np.float64).reshape(npred, -1))
    b = None if p == 0 else _f64(beta)
    outs = [np.zeros(npred) for _ in range(5)]
    samples = np.zeros((npred, n_samples), order="F")
    vscale = np.zeros(npred)
    _chk(lib().orc_zcptn_predict(C.byref(om.m), _p(_f64(state["grad_at_mode"])), _p(_f64(state["w"])), npred,
                                 _p(qx), _p(qy), _p(qt), _p(Xpf), p, _p(b), C.c_double(lik_sigma),
                                 C.c_double(lik_lambda), pred_m_v, n_samples, C.c_uint64(seed),
                                 *[_p(o) for o in outs], _p(samples), _p(vscale)))
    keys = ["mu_latent", "var_latent", "p_rain", "amount_mean", "amount_median"]
    d = dict(zip(keys, outs))
    d["var_scale"] = vscale
    d["samples"] = np.ascontiguousarray(samples)
    return d


def grad_close(g, gr, scale, rtol: float = 1e-8) -> bool:
    """Per-component gradient parity: |g_k - gr_k| <= rtol * scale_k, scale_k = sum over rows of
    |row contribution to k| (OracleModel.nll_grad_scale)."""
    g, gr, scale = np.asarray(g, dtype=np.float64), np.asarray(gr, dtype=np.float64), np.asarray(scale)
    return bool((np.abs(g - gr) <= rtol * scale).all())
