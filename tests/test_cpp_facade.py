"""The C++ facade (include/stgp_b200.hpp) compiles against the C ABI and links
against the engine; on a GPU box the example runs end to end."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2602_03609_b200")


def _build(tmp_path):
    exe = str(tmp_path / "vif_eval")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "vif_eval.cpp"),
           "-L", PKG, "-l:libstgp_b200.so", "-Wl,-rpath," + PKG, "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_facade_example_runs(tmp_path):
    out = subprocess.run([_build(tmp_path), "200", "10"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "nll=" in out.stdout
