"""Python mirror of the reference's public C++ API for the hot path.

Names, argument meaning and error behaviour follow the reference headers
(proj/include/stgp/*.hpp); every call goes through the C ABI of the CUDA
engine (include/stgp_b200.h).  Exceptions: ConfigError / DataError /
NumericError as in types.hpp:26-38.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, astuple

import numpy as np

from . import _native as N
from ._native import ConfigError, DataError, NumericError, StgpError  # noqa: F401

LATENT, OBSERVATION = 0, 1
METRIC_EUCLID, METRIC_DC, METRIC_DR = 0, 1, 2


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class CovarianceParams:
    """covariance.hpp:23-38 (field order is the ABI order)."""
    sigma2: float = 0.0
    sigma1_2: float = 1.0
    a: float = 1.0
    c: float = 1.0
    alpha: float = 0.5
    nu: float = 1.5
    beta: float = 0.5
    delta: float = 0.5

    def as_tuple(self):
        return astuple(self)

    def c_struct(self) -> N.Params:
        return N.Params(*astuple(self))


def as_params(theta) -> CovarianceParams:
    if isinstance(theta, CovarianceParams):
        return theta
    if isinstance(theta, dict):
        return CovarianceParams(**theta)
    return CovarianceParams(*theta)


class Context:
    """One CUDA device + stream (+ optional NCCL communicator)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        N.call("stgp_ctx_create", device, C.byref(h))
        self.h = h
        self.device = device

    def set_shard(self, rank: int, world: int):
        N.call("stgp_ctx_set_shard", self.h, rank, world)

    def init_nccl(self, unique_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        N.call("stgp_ctx_init_nccl", self.h, buf, rank, world)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.call("stgp_nccl_unique_id", buf)
        return buf.raw

    def synchronize(self):
        N.call("stgp_ctx_synchronize", self.h)

    def set_host_allreduce(self, fn):
        """fn(buf: np.ndarray) sums buf across ranks in place (in-process ranks)."""
        def _cb(user, buf, count):
            try:
                fn(np.ctypeslib.as_array(buf, shape=(count,)))
                return 0
            except Exception:  # noqa: BLE001 - reported to the engine as a failed all-reduce
                return 1
        self._allreduce_cb = N.ALLREDUCE_FN(_cb)
        N.call("stgp_ctx_set_host_allreduce", self.h, C.cast(self._allreduce_cb, C.c_void_p), None)

    def stream_ptr(self) -> int:
        return int(N.lib().stgp_ctx_stream(self.h))

    def fp64_peak_tflops(self) -> float:
        out = C.c_double()
        N.call("stgp_debug_fp64_peak", self.h, C.byref(out))
        return out.value

    def profile_all(self) -> dict:
        """{region: (ms, count)} for every profiled region recorded so far."""
        buf = C.create_string_buffer(1 << 14)
        N.call("stgp_ctx_profile_names", self.h, buf, len(buf))
        names = [n for n in buf.value.decode().split("\n") if n]
        return {n: self.profile_get(n) for n in names}

    def dmma_peak_tflops(self) -> float:
        """Measured FP64 tensor-core (DMMA m8n8k4) throughput, TFLOP/s."""
        out = C.c_double()
        N.call("stgp_debug_dmma_peak", self.h, C.byref(out))
        return out.value

    def gemm_rows(self, A, B, emulated: bool = True):
        """C = A B^T (FP64) through the int8 Ozaki path (tcgen05) or the DMMA GEMM; returns (C, device ms)."""
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        n, k = A.shape
        m = B.shape[0]
        C_ = np.zeros((n, m))
        ms = C.c_double(0.0)
        N.call("stgp_debug_gemm_rows", self.h, int(emulated), n, m, k, _ptr(A), _ptr(B), _ptr(C_), C.byref(ms))
        return C_, ms.value

    def trmm(self, T, B, transpose: bool = False, mode: int = 1):
        """C = op(T) B for lower-triangular T (m x m) and B (m x n): mode 0 the DMMA TRMM, 1 the int8
        Ozaki rows form with the triangle's K ranges, 2 the same over the full K range; returns
        (C, device ms)."""
        T = np.asfortranarray(T, dtype=np.float64)
        B = np.asfortranarray(B, dtype=np.float64)
        m, n = B.shape
        C_ = np.zeros((m, n), order="F")
        ms = C.c_double(0.0)
        N.call("stgp_debug_trmm", self.h, int(mode), int(transpose), m, n, _ptr(T), _ptr(B), _ptr(C_), C.byref(ms))
        return C_, ms.value

    def gemm_cols(self, A, B=None, emulated: bool = True):
        """C = A^T B (A, B: n x m, i.e. m x n column-major), C[j][i] = sum_r A[r, j] B[r, i]; the
        int8 Ozaki path for the long reduction or the DMMA GEMM.  B None: A^T A."""
        A = np.ascontiguousarray(A, dtype=np.float64)
        n, m = A.shape
        Bc = A if B is None else np.ascontiguousarray(B, dtype=np.float64)
        C_ = np.zeros((m, m))
        ms = C.c_double(0.0)
        N.call("stgp_debug_gemm_cols", self.h, int(emulated), m, n, _ptr(A), _ptr(Bc), _ptr(C_), C.byref(ms))
        return C_, ms.value

    def profile(self, enable: bool = True):
        N.call("stgp_ctx_profile", self.h, int(enable))

    def profile_get(self, region: str):
        ms, cnt = C.c_double(), C.c_int64()
        N.call("stgp_ctx_profile_get", self.h, region.encode(), C.byref(ms), C.byref(cnt))
        return ms.value, cnt.value

    def profile_reset(self):
        N.call("stgp_ctx_profile_reset", self.h)

    def kernel_launches(self) -> int:
        return int(N.lib().stgp_ctx_kernel_launches(self.h))

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().stgp_ctx_destroy(self.h)
            self.h = None


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def mix_seed(seed: int, stream: int) -> int:
    return int(N.lib().stgp_mix_seed(seed, stream))


def order_observations_perm(t, seed: int) -> np.ndarray:
    """dataset.cpp:81-114: the permutation `ordering` of order_observations."""
    t = _f64(t)
    perm = np.zeros(len(t), dtype=np.int32)
    N.call("stgp_order_observations", len(t), _ptr(t), C.c_uint64(seed), _ptr(perm))
    return perm


def effective_ranges(theta):
    tr, sr = C.c_double(), C.c_double()
    p = as_params(theta).c_struct()
    N.call("stgp_effective_ranges", C.byref(p), C.byref(tr), C.byref(sr))
    return tr.value, sr.value


class HostAllreduce:
    """Sum all-reduce between in-process ranks (threads) through host buffers."""

    def __init__(self, world: int, timeout: float = 300.0):
        import threading
        self.world = world
        self.bufs = [None] * world
        self.barrier = threading.Barrier(world, timeout=timeout)

    def for_rank(self, rank: int):
        def fn(buf):
            self.bufs[rank] = buf.copy()
            self.barrier.wait()
            total = self.bufs[0].copy()
            for r in range(1, self.world):  # fixed rank order: identical bits on every rank
                total += self.bufs[r]
            self.barrier.wait()
            buf[:] = total
        return fn


class SpaceTimeDataset:
    """Device-resident ordered observations (dataset.hpp:22-41)."""

    def __init__(self, x, y, t, resp=None, X=None, ctx: Context | None = None, ordering=None):
        self.ctx = ctx or default_context()
        self.x, self.y, self.t = _f64(x), _f64(y), _f64(t)
        self.n = len(self.x)
        self.resp = None if resp is None else _f64(resp)
        self.X = None if X is None else np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(self.n, -1))
        self.ordering = np.arange(self.n) if ordering is None else np.asarray(ordering)
        h = C.c_void_p()
        N.call("stgp_dataset_create", self.ctx.h, self.n, _ptr(self.x), _ptr(self.y), _ptr(self.t), C.byref(h))
        self.h = h
        if self.resp is not None:
            p = 0 if self.X is None else self.X.shape[1]
            N.call("stgp_dataset_set_response", self.h, _ptr(self.resp), p, _ptr(self.X) if p else None)

    @property
    def p(self):
        return 0 if self.X is None else self.X.shape[1]

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().stgp_dataset_destroy(self.h)
            self.h = None


def order_observations(x, y, t, resp=None, X=None, seed: int = 0, ctx=None) -> SpaceTimeDataset:
    perm = order_observations_perm(t, seed)
    x, y, t = np.asarray(x)[perm], np.asarray(y)[perm], np.asarray(t)[perm]
    resp = None if resp is None else np.asarray(resp)[perm]
    X = None if X is None else np.asarray(X).reshape(len(perm), -1)[perm]
    return SpaceTimeDataset(x, y, t, resp, X, ctx=ctx, ordering=perm)


class NeighborSets:
    """neighbors.hpp:100-110 (device resident; .sets downloads lazily)."""

    def __init__(self, h, ds: SpaceTimeDataset):
        self.h = h
        self.ds = ds
        n, m, k = C.c_int(), C.c_int(), C.c_int()
        N.call("stgp_neighbors_shape", self.h, C.byref(n), C.byref(m), C.byref(k))
        self.n, self.m_v, self.metric_kind = n.value, m.value, k.value

    @classmethod
    def from_sets(cls, ds: SpaceTimeDataset, sets, metric_kind=METRIC_DC):
        arr = np.ascontiguousarray(sets, dtype=np.int32)
        h = C.c_void_p()
        N.call("stgp_neighbors_from_host", ds.h, arr.shape[1], _ptr(arr), metric_kind, C.byref(h))
        return cls(h, ds)

    def indices(self) -> np.ndarray:
        out = np.zeros((self.n, self.m_v), dtype=np.int32)
        N.call("stgp_neighbors_download", self.h, _ptr(out), None)
        return out

    def distances(self) -> np.ndarray:
        out = np.zeros((self.n, self.m_v))
        N.call("stgp_neighbors_download", self.h, None, _ptr(out))
        return out

    @property
    def sets(self):
        idx = self.indices()
        return [list(r[r >= 0]) for r in idx]

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().stgp_neighbors_destroy(self.h)
            self.h = None


def euclidean_neighbors(ds: SpaceTimeDataset, m_v: int, space_scale: float, time_scale: float) -> NeighborSets:
    h = C.c_void_p()
    N.call("stgp_euclidean_neighbors", ds.h, m_v, space_scale, time_scale, C.byref(h))
    return NeighborSets(h, ds)


def correlation_neighbors(ds: SpaceTimeDataset, theta, m_v: int) -> NeighborSets:
    h = C.c_void_p()
    p = as_params(theta).c_struct()
    N.call("stgp_correlation_neighbors", ds.h, C.byref(p), m_v, C.byref(h))
    return NeighborSets(h, ds)


def residual_neighbors(ds: SpaceTimeDataset, theta, inducing: "InducingSet", m_v: int) -> NeighborSets:
    h = C.c_void_p()
    p = as_params(theta).c_struct()
    N.call("stgp_residual_neighbors", ds.h, C.byref(p), inducing.h, m_v, C.byref(h))
    return NeighborSets(h, ds)


class InducingSet:
    """inducing.hpp:22-31."""

    def __init__(self, h, ctx: Context):
        self.h = h
        self.ctx = ctx
        M, ms, mt = C.c_int(), C.c_int(), C.c_int()
        N.call("stgp_inducing_size", self.h, C.byref(M), C.byref(ms), C.byref(mt))
        self.M, self.m_s, self.m_t = M.value, ms.value, mt.value

    @classmethod
    def from_points(cls, points, ctx: Context | None = None):
        ctx = ctx or default_context()
        P = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
        h = C.c_void_p()
        N.call("stgp_inducing_create", ctx.h, len(P), _ptr(P), C.byref(h))
        return cls(h, ctx)

    @property
    def points(self) -> np.ndarray:
        out = np.zeros((self.M, 3))
        N.call("stgp_inducing_download", self.h, _ptr(out))
        return out

    def size(self):
        return self.M

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().stgp_inducing_destroy(self.h)
            self.h = None


def sts_kmeanspp(ds: SpaceTimeDataset, m: int, seed: int) -> InducingSet:
    h = C.c_void_p()
    N.call("stgp_sts_kmeanspp", ds.h, m, C.c_uint64(seed), C.byref(h))
    return InducingSet(h, ds.ctx)


def joint_kmeanspp_inducing(ds: SpaceTimeDataset, m: int, space_scale: float, time_scale: float,
                            seed: int) -> InducingSet:
    h = C.c_void_p()
    N.call("stgp_joint_kmeanspp_inducing", ds.h, m, space_scale, time_scale, C.c_uint64(seed), C.byref(h))
    return InducingSet(h, ds.ctx)


def kmeanspp(points, k: int, seed: int, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    P = np.asfortranarray(np.asarray(points, dtype=np.float64).reshape(len(points), -1))
    out = np.zeros((k, P.shape[1]), order="F")
    N.call("stgp_kmeanspp", ctx.h, _ptr(P), P.shape[0], P.shape[1], k, C.c_uint64(seed), _ptr(out))
    return np.ascontiguousarray(out)


class Structure:
    """VecchiaStructure / FitcStructure / VifStructure (approximations.hpp:33-75)."""

    def __init__(self, h, ds: SpaceTimeDataset, kind: str, m_v: int):
        self.h = h
        self.data = ds
        self.kind = kind
        self.m_v = m_v

    @property
    def D(self) -> np.ndarray:
        out = np.zeros(self.data.n)
        N.call("stgp_structure_download_D", self.h, _ptr(out))
        return out

    @property
    def A(self) -> np.ndarray:
        out = np.zeros((self.data.n, self.m_v))
        N.call("stgp_structure_download_A", self.h, _ptr(out))
        return out

    @property
    def fitc_diag(self) -> np.ndarray:
        out = np.zeros(self.data.n)
        N.call("stgp_structure_download_fitc_diag", self.h, _ptr(out))
        return out

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().stgp_structure_destroy(self.h)
            self.h = None


def build_vecchia(ds, theta, neighbors: NeighborSets, policy=LATENT) -> Structure:
    h = C.c_void_p()
    p = as_params(theta).c_struct()
    N.call("stgp_build_vecchia", ds.h, C.byref(p), neighbors.h, int(policy), C.byref(h))
    return Structure(h, ds, "vecchia", neighbors.m_v)


def build_fitc(ds, theta, inducing: InducingSet) -> Structure:
    h = C.c_void_p()
    p = as_params(theta).c_struct()
    N.call("stgp_build_fitc", ds.h, C.byref(p), inducing.h, C.byref(h))
    return Structure(h, ds, "fitc", 1)


def build_vif(ds, theta, inducing: InducingSet, neighbors: NeighborSets, policy=LATENT) -> Structure:
    h = C.c_void_p()
    p = as_params(theta).c_struct()
    N.call("stgp_build_vif", ds.h, C.byref(p), inducing.h, neighbors.h, int(policy), C.byref(h))
    return Structure(h, ds, "vif", neighbors.m_v)


def _yxb(s: Structure, y, X, beta):
    n = s.data.n
    yv = None if y is None else _f64(y)
    if X is None or beta is None or np.size(beta) == 0:
        return yv, None, 0, None
    Xf = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(n, -1))
    return yv, Xf, Xf.shape[1], _f64(beta)


def nll(s: Structure, y=None, X=None, beta=None) -> float:
    yv, Xf, p, b = _yxb(s, y, X, beta)
    out = C.c_double()
    N.call("stgp_nll", s.h, _ptr(yv), _ptr(Xf), p, _ptr(b), C.byref(out))
    return out.value


def nll_grad(s: Structure, y=None, X=None, beta=None) -> np.ndarray:
    yv, Xf, p, b = _yxb(s, y, X, beta)
    g = np.zeros(7)
    N.call("stgp_nll_grad", s.h, _ptr(yv), _ptr(Xf), p, _ptr(b), _ptr(g))
    return g


def nll_and_grad(s: Structure, y=None, X=None, beta=None):
    yv, Xf, p, b = _yxb(s, y, X, beta)
    g = np.zeros(7)
    out = C.c_double()
    N.call("stgp_nll_and_grad", s.h, _ptr(yv), _ptr(Xf), p, _ptr(b), C.byref(out), _ptr(g))
    return out.value, g


def evaluate(s: Structure, theta, y=None, X=None, beta=None):
    """Rebuild at theta and return (nll, grad) in one device pass."""
    yv, Xf, p, b = _yxb(s, y, X, beta)
    g = np.zeros(7)
    out = C.c_double()
    pc = as_params(theta).c_struct()
    N.call("stgp_eval", s.h, C.byref(pc), _ptr(yv), _ptr(Xf), p, _ptr(b), C.byref(out), _ptr(g))
    return out.value, g


def gls_beta(s: Structure, y, X) -> np.ndarray:
    yv = _f64(y)
    Xf = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(s.data.n, -1))
    out = np.zeros(Xf.shape[1])
    N.call("stgp_gls_beta", s.h, _ptr(yv), _ptr(Xf), Xf.shape[1], _ptr(out))
    return out


@dataclass
class PredictiveDistribution:
    mu: np.ndarray
    var: np.ndarray


def predict(s: Structure, y, X, beta, targets, X_p=None, pred_m_v: int = 0) -> PredictiveDistribution:
    yv, Xf, p, b = _yxb(s, y, X, beta)
    T = np.ascontiguousarray(np.asarray(targets, dtype=np.float64).reshape(-1, 3))
    npred = len(T)
    Xp = None if (X_p is None or p == 0) else np.asfortranarray(np.asarray(X_p, dtype=np.float64).reshape(npred, -1))
    mu, var = np.zeros(npred), np.zeros(npred)
    N.call("stgp_predict", s.h, _ptr(yv), _ptr(Xf), p, _ptr(b), npred, _ptr(T), _ptr(Xp), pred_m_v, _ptr(mu), _ptr(var))
    return PredictiveDistribution(mu, var)


@dataclass
class LikelihoodParams:
    """LikelihoodParams (covariance.hpp:41-48): ZC-PTN noise sd and power."""
    sigma: float = 1.0
    lambda_: float = 1.0


@dataclass
class LaplaceState:
    """LaplaceState (laplace.hpp:37-44)."""
    mode: np.ndarray
    grad_at_mode: np.ndarray
    w: np.ndarray
    log_marginal: float
    converged: bool
    iterations: int


def laplace_marginal(s: Structure, y, X=None, beta=None, lik: LikelihoodParams | None = None, warm_start=None):
    """laplace_marginal (laplace.hpp:47-53): (negative Laplace log-marginal, LaplaceState) for the ZC-PTN
    likelihood on a latent-policy Vecchia / VIF structure or a FITC structure."""
    lik = lik or LikelihoodParams()
    yv, Xf, p, b = _yxb(s, y, X, beta)
    n = s.data.n
    mode, ga, w = np.zeros(n), np.zeros(n), np.zeros(n)
    out, it = C.c_double(), C.c_int()
    warm = None if warm_start is None else _f64(warm_start)
    N.call("stgp_laplace_marginal", s.h, _ptr(yv), _ptr(Xf), p, _ptr(b), float(lik.sigma), float(lik.lambda_),
           _ptr(warm), C.byref(out), _ptr(mode), _ptr(ga), _ptr(w), C.byref(it))
    return out.value, LaplaceState(mode, ga, w, -out.value, True, it.value)


@dataclass
class ZcptnPrediction:
    """ZcptnPrediction (laplace.hpp:55-62)."""
    mu_latent: np.ndarray
    var_latent: np.ndarray
    p_rain: np.ndarray
    amount_mean: np.ndarray
    amount_median: np.ndarray
    samples: np.ndarray


def zcptn_predict(state: LaplaceState, s: Structure, targets, X_p=None, beta=None,
                  lik: LikelihoodParams | None = None, pred_m_v: int = 0, n_samples: int = 200,
                  seed: int = 0) -> ZcptnPrediction:
    """zcptn_predict (laplace.hpp:67-72) from the Laplace state of laplace_marginal."""
    lik = lik or LikelihoodParams()
    T = np.ascontiguousarray(np.asarray(targets, dtype=np.float64).reshape(-1, 3))
    npred = len(T)
    p = 0 if X_p is None or beta is None or np.size(beta) == 0 else np.asarray(X_p).reshape(npred, -1).shape[1]
    Xp = None if p == 0 else np.asfortranarray(np.asarray(X_p, dtype=np.float64).reshape(npred, -1))
    b = None if p == 0 else _f64(beta)
    outs = [np.zeros(npred) for _ in range(5)]
    samples = np.zeros((npred, n_samples), order="F")
    N.call("stgp_zcptn_predict", s.h, _ptr(_f64(state.grad_at_mode)), _ptr(_f64(state.w)), npred, _ptr(T), _ptr(Xp), p,
           _ptr(b), float(lik.sigma), float(lik.lambda_), int(pred_m_v), int(n_samples), C.c_uint64(seed),
           *[_ptr(o) for o in outs], _ptr(samples))
    return ZcptnPrediction(*outs, np.ascontiguousarray(samples))


def debug_exp(x, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    x = _f64(x)
    out = np.zeros_like(x)
    N.call("stgp_debug_exp", ctx.h, len(x), _ptr(x), _ptr(out))
    return out


def debug_kernel(theta, h, u, ctx: Context | None = None, grad: bool = True):
    """Device GneitingKernel::eval (and ::grad unless grad=False; general nu raises NumericError there)."""
    ctx = ctx or default_context()
    h, u = _f64(h), _f64(u)
    cov, g = np.zeros(len(h)), (np.zeros((len(h), 6)) if grad else None)
    p = as_params(theta).c_struct()
    N.call("stgp_debug_kernel", ctx.h, C.byref(p), len(h), _ptr(h), _ptr(u), _ptr(cov), _ptr(g) if grad else None)
    return cov, g


# ---------------------------------------------------------------------------
# fit driver (estimation.hpp:23-110, estimation.cpp:423-619; Gaussian likelihood)
# ---------------------------------------------------------------------------
FIT_METHODS = {"vecchia-euclid": 0, "vecchia-corr": 1, "fitc-kmeanspp": 2, "fitc-sts": 3, "vif": 4}


class FitConfig(C.Structure):
    """FitConfig (estimation.hpp:23-56): method, m_v, m, max_iterations, tolerances, nu, seed."""
    _fields_ = [("method", C.c_int), ("m_v", C.c_int), ("m", C.c_int), ("max_iterations", C.c_int),
                ("tol_objective", C.c_double), ("tol_gradient", C.c_double), ("nu", C.c_double),
                ("seed", C.c_uint64)]

    def __init__(self, method="vecchia-corr", m_v=30, m=500, max_iterations=200, tol_objective=1e-8,
                 tol_gradient=1e-5, nu=1.5, seed=0):
        super().__init__(FIT_METHODS[method] if isinstance(method, str) else int(method), m_v, m, max_iterations,
                         tol_objective, tol_gradient, nu, seed)


class TraceRow(C.Structure):
    _fields_ = [("iteration", C.c_int), ("nll", C.c_double), ("grad_norm", C.c_double), ("refresh", C.c_int)]


@dataclass
class FittedModel:
    """FittedModel (estimation.hpp:68-83): parameters, coefficients, the ordered data and the trace."""
    theta: CovarianceParams
    beta: np.ndarray
    final_nll: float
    converged: bool
    trace: list
    data: "SpaceTimeDataset"


def default_init(ds: "SpaceTimeDataset", config: FitConfig, y=None, X=None) -> CovarianceParams:
    """default_init (estimation.cpp:68-114) on an ordered dataset."""
    yv = _f64(ds.resp if y is None else y)
    Xv = ds.X if X is None else np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(ds.n, -1))
    p = 0 if Xv is None else Xv.shape[1]
    out = N.Params()
    N.call("stgp_default_init", ds.h, _ptr(yv), _ptr(Xv) if p else None, p, C.byref(config), C.byref(out))
    return CovarianceParams(*[getattr(out, f) for f, _ in N.Params._fields_])


def fit(x, y, t, resp, X=None, config: FitConfig | None = None, init=None, ctx: Context | None = None,
        trace_cap: int = 4096) -> FittedModel:
    """fit (estimation.cpp:423-619): orders the observations with config.seed (FittedModel.data),
    then maximises the Gaussian likelihood on the device."""
    config = config or FitConfig()
    ds = order_observations(x, y, t, resp, X, seed=config.seed, ctx=ctx)
    yv = ds.resp
    p = ds.p
    theta = N.Params()
    beta = np.zeros(max(p, 1))
    fnll = C.c_double(0.0)
    conv = C.c_int(0)
    ntr = C.c_int(0)
    rows = (TraceRow * trace_cap)()
    init_p = as_params(init).c_struct() if init is not None else None
    N.call("stgp_fit", ds.h, _ptr(yv), _ptr(ds.X) if p else None, p, C.byref(config),
           C.byref(init_p) if init_p is not None else None, C.byref(theta), _ptr(beta), C.byref(fnll), C.byref(conv),
           C.cast(rows, C.c_void_p), trace_cap, C.byref(ntr))
    trace = [(r.iteration, r.nll, r.grad_norm, bool(r.refresh)) for r in rows[:min(ntr.value, trace_cap)]]
    th = CovarianceParams(*[getattr(theta, f) for f, _ in N.Params._fields_])
    return FittedModel(th, beta[:p].copy(), fnll.value, bool(conv.value), trace, ds)


# ---------------------------------------------------------------------------
# dataset CSV and neighbour audit (dataset.cpp:191-316, neighbors.cpp:336-355)
# ---------------------------------------------------------------------------
@dataclass
class DatasetTable:
    """read_dataset_csv's SpaceTimeDataset fields (host): points, value, X (n x p), stations."""
    x: np.ndarray
    y: np.ndarray
    t: np.ndarray
    value: np.ndarray
    X: np.ndarray
    stations: list
    covariate_names: list


def read_dataset_csv(path: str) -> DatasetTable:
    h = C.c_void_p()
    N.call("stgp_read_dataset_csv", str(path).encode(), C.byref(h))
    try:
        n, p, hs = C.c_int(), C.c_int(), C.c_int()
        N.call("stgp_table_shape", h, C.byref(n), C.byref(p), C.byref(hs))
        n, p = n.value, p.value
        x, y, t, v = (np.zeros(n) for _ in range(4))
        X = np.zeros((n, p), order="F")
        N.call("stgp_table_columns", h, _ptr(x), _ptr(y), _ptr(t), _ptr(v), _ptr(X) if p else None)
        L = N.lib()

        def text(fn, i):
            k = fn(h, i, None, 0)
            buf = C.create_string_buffer(k + 1)
            fn(h, i, buf, k + 1)
            return buf.value.decode()
        stations = [text(L.stgp_table_station, i) for i in range(n)] if hs.value else []
        names = [text(L.stgp_table_covariate_name, j) for j in range(p)]
        return DatasetTable(x, y, t, v, X, stations, names)
    finally:
        N.lib().stgp_table_destroy(h)


def write_dataset_csv(path: str, x, y, t, value, X=None, stations=None, header_comment: str = ""):
    x, y, t, value = _f64(x), _f64(y), _f64(t), _f64(value)
    n = len(x)
    Xf = None if X is None else np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(n, -1))
    p = 0 if Xf is None else Xf.shape[1]
    st = None
    if stations is not None:
        st = (C.c_char_p * n)(*[str(s).encode() for s in stations])
    N.call("stgp_write_dataset_csv", str(path).encode(), n, _ptr(x), _ptr(y), _ptr(t), _ptr(value), p,
           _ptr(Xf) if p else None, C.cast(st, C.c_void_p) if st is not None else None, header_comment.encode())


def write_neighbor_debug_csv(path: str, neighbors: "NeighborSets", ds: "SpaceTimeDataset", header_comment: str = ""):
    N.call("stgp_write_neighbor_debug_csv", str(path).encode(), neighbors.h, ds.h, header_comment.encode())
