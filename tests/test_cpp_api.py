"""The C++ mirror of the reference API (include/fst_b200.hpp) compiles against the
C-ABI library (CPU) and passes the reference's stream/sketch tests on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2105_05879_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    f"-L{LIBDIR}", "-lfst_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_cpp_api_builds(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
