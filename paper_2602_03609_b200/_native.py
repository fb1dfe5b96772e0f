"""ctypes loader for the in-tree CUDA engine (libstgp_b200.so).

There is no fallback: if the library is missing or no B200 is visible the
calls fail loudly.  Build it with `python -c "import __graft_entry__ as g; g.build()"`
or `make -C paper_2602_03609_b200/csrc`.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# STGP_LIB selects another build of the same library (the bounds-checked one: `make checks`)
LIB_PATH = os.environ.get("STGP_LIB") or os.path.join(_HERE, "libstgp_b200.so")


class StgpError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types (types.hpp:26-38)."""


class ConfigError(StgpError):
    pass


class DataError(StgpError):
    pass


class NumericError(StgpError):
    pass


_CODES = {2: ConfigError, 3: DataError, 4: NumericError}


class Params(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("sigma2", "sigma1_2", "a", "c", "alpha", "nu", "beta", "delta")]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)

# name -> argtypes (restype int unless noted)
_SIGS = {
    "stgp_version": [],
    "stgp_ctx_create": [C.c_int, C.POINTER(_P)],
    "stgp_ctx_synchronize": [_P],
    "stgp_ctx_set_shard": [_P, C.c_int, C.c_int],
    "stgp_nccl_unique_id": [_P],
    "stgp_ctx_init_nccl": [_P, _P, C.c_int, C.c_int],
    "stgp_order_observations": [C.c_int, _P, C.c_uint64, _P],
    "stgp_effective_ranges": [C.POINTER(Params), _D, _D],
    "stgp_dataset_create": [_P, C.c_int, _P, _P, _P, C.POINTER(_P)],
    "stgp_dataset_set_response": [_P, _P, C.c_int, _P],
    "stgp_euclidean_neighbors": [_P, C.c_int, C.c_double, C.c_double, C.POINTER(_P)],
    "stgp_correlation_neighbors": [_P, C.POINTER(Params), C.c_int, C.POINTER(_P)],
    "stgp_residual_neighbors": [_P, C.POINTER(Params), _P, C.c_int, C.POINTER(_P)],
    "stgp_neighbors_from_host": [_P, C.c_int, _P, C.c_int, C.POINTER(_P)],
    "stgp_neighbors_shape": [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "stgp_neighbors_download": [_P, _P, _P],
    "stgp_inducing_create": [_P, C.c_int, _P, C.POINTER(_P)],
    "stgp_sts_kmeanspp": [_P, C.c_int, C.c_uint64, C.POINTER(_P)],
    "stgp_joint_kmeanspp_inducing": [_P, C.c_int, C.c_double, C.c_double, C.c_uint64, C.POINTER(_P)],
    "stgp_kmeanspp": [_P, _P, C.c_int, C.c_int, C.c_int, C.c_uint64, _P],
    "stgp_inducing_size": [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "stgp_inducing_download": [_P, _P],
    "stgp_build_vecchia": [_P, C.POINTER(Params), _P, C.c_int, C.POINTER(_P)],
    "stgp_build_fitc": [_P, C.POINTER(Params), _P, C.POINTER(_P)],
    "stgp_build_vif": [_P, C.POINTER(Params), _P, _P, C.c_int, C.POINTER(_P)],
    "stgp_structure_download_D": [_P, _P],
    "stgp_structure_download_A": [_P, _P],
    "stgp_structure_download_fitc_diag": [_P, _P],
    "stgp_nll": [_P, _P, _P, C.c_int, _P, _D],
    "stgp_nll_grad": [_P, _P, _P, C.c_int, _P, _P],
    "stgp_nll_and_grad": [_P, _P, _P, C.c_int, _P, _D, _P],
    "stgp_gls_beta": [_P, _P, _P, C.c_int, _P],
    "stgp_predict": [_P, _P, _P, C.c_int, _P, C.c_int, _P, _P, C.c_int, _P, _P],
    "stgp_zcptn_predict": [_P, _P, _P, C.c_int, _P, _P, C.c_int, _P, C.c_double, C.c_double, C.c_int, C.c_int,
                           C.c_uint64, _P, _P, _P, _P, _P, _P],
    "stgp_laplace_marginal": [_P, _P, _P, C.c_int, _P, C.c_double, C.c_double, _P, _D, _P, _P, _P,
                              C.POINTER(C.c_int)],
    "stgp_eval": [_P, C.POINTER(Params), _P, _P, C.c_int, _P, _D, _P],
    "stgp_debug_exp": [_P, C.c_int, _P, _P],
    "stgp_debug_fp64_peak": [_P, _D],
    "stgp_debug_dmma_peak": [_P, _D],
    "stgp_read_dataset_csv": [C.c_char_p, C.POINTER(_P)],
    "stgp_table_shape": [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "stgp_table_columns": [_P, _P, _P, _P, _P, _P],
    "stgp_write_dataset_csv": [C.c_char_p, C.c_int, _P, _P, _P, _P, C.c_int, _P, _P, C.c_char_p],
    "stgp_write_neighbor_debug_csv": [C.c_char_p, _P, _P, C.c_char_p],
    "stgp_default_init": [_P, _P, _P, C.c_int, _P, C.POINTER(Params)],
    "stgp_fit": [_P, _P, _P, C.c_int, _P, _P, C.POINTER(Params), _P, _D, C.POINTER(C.c_int), _P, C.c_int,
                 C.POINTER(C.c_int)],
    "stgp_debug_gemm_rows": [_P, C.c_int, C.c_longlong, C.c_int, C.c_int, _P, _P, _P, _D],
    "stgp_debug_trmm": [_P, C.c_int, C.c_int, C.c_int, C.c_longlong, _P, _P, _P, _D],
    "stgp_debug_gemm_cols": [_P, C.c_int, C.c_int, C.c_longlong, _P, _P, _P, _D],
    "stgp_ctx_profile_names": [_P, C.c_char_p, C.c_int],
    "stgp_ctx_profile": [_P, C.c_int],
    "stgp_ctx_set_host_allreduce": [_P, _P, _P],
    "stgp_ctx_profile_get": [_P, C.c_char_p, _D, C.POINTER(C.c_int64)],
    "stgp_ctx_profile_reset": [_P],
    "stgp_debug_kernel": [_P, C.POINTER(Params), C.c_int, _P, _P, _P, _P],
}
_VOID = ["stgp_table_destroy", "stgp_ctx_destroy", "stgp_dataset_destroy", "stgp_neighbors_destroy", "stgp_inducing_destroy",
         "stgp_structure_destroy"]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"stgp_b200 CUDA engine not built: {LIB_PATH} is missing "
                              "(run __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        for name in _VOID:
            f = getattr(L, name)
            f.argtypes = [_P]
            f.restype = None
        L.stgp_last_error.restype = C.c_char_p
        L.stgp_last_error.argtypes = []
        L.stgp_mix_seed.restype = C.c_uint64
        L.stgp_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.stgp_ctx_kernel_launches.restype = C.c_int64
        L.stgp_ctx_kernel_launches.argtypes = [_P]
        for name in ("stgp_table_station", "stgp_table_covariate_name"):  # return a length, not a code
            getattr(L, name).restype = C.c_int
            getattr(L, name).argtypes = [_P, C.c_int, C.c_char_p, C.c_int]
        L.stgp_ctx_stream.restype = C.c_void_p
        L.stgp_ctx_stream.argtypes = [_P]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().stgp_last_error().decode()
        raise _CODES.get(rc, StgpError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def exported_symbols() -> list[str]:
    return sorted(list(_SIGS) + _VOID + ["stgp_last_error", "stgp_mix_seed", "stgp_ctx_kernel_launches", "stgp_ctx_stream",
                                         "stgp_table_station", "stgp_table_covariate_name"])
