"""The header-only C++ facade (include/tucktree_b200.hpp) compiles with g++
against the engine library and reproduces the reference KATs through it."""
import os
import subprocess

import pytest

from paper_2501_06647_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path, eigen=False):
    """eigen=True compiles the facade's Eigen adaptor (tucktree::Matrix = Eigen::MatrixXd)
    against the Eigen-API headers of oracle/eigen_shim (Eigen itself is absent here)."""
    lib = B.build()
    exe = str(tmp_path / ("facade_check_eigen" if eigen else "facade_check"))
    extra = ["-DTUCKTREE_USE_EIGEN", "-I", os.path.join(ROOT, "oracle", "eigen_shim")] if eigen else []
    subprocess.check_call(["g++", "-std=c++17", "-O1", *extra, "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "facade_check.cpp"), lib,
                           "-Wl,-rpath," + os.path.dirname(lib), "-o", exe])
    return exe


@pytest.mark.parametrize("eigen", [False, True])
def test_facade_structure(tmp_path, eigen):
    exe = _compile(tmp_path, eigen)
    r = subprocess.run([exe], capture_output=True, text=True, cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("eigen", [False, True])
def test_facade_gpu(tmp_path, eigen):
    exe = _compile(tmp_path, eigen)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
