"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol include/stgp_b200.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stgp_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stgp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    from paper_2602_03609_b200 import _native
    assert os.path.exists(_native.LIB_PATH), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (stgp_\w+)", out))
    assert set(declared()) <= exported


def test_python_binding_covers_header():
    from paper_2602_03609_b200 import _native
    assert set(declared()) <= set(_native.exported_symbols()) | {"stgp_ctx_release_comm"}


def test_no_oracle_in_product():
    # the product library must not link or reference the oracle
    from paper_2602_03609_b200 import _native
    out = subprocess.run(["nm", "-D", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out
    deps = subprocess.run(["ldd", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "liboracle" not in deps


def test_ctx_without_gpu_fails_loudly():
    import paper_2602_03609_b200 as S
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(S.StgpError):
        S.Context(0)
