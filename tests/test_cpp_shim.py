"""The C++ drop-in layer (include/scenopt_b200.hpp, the reference's
namespace-scenopt API over the C-ABI), exercised by tests/cpp/test_shim.cpp:
reference-style cases for the oracles, FBE, L-BFGS and solvers. Host-only
cases run here; the device cases run under the gpu marker."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2107_01745_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "test_shim")


def _build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", SRC,
           f"-L{LIBDIR}", "-lscenopt_b200", f"-Wl,-rpath,{LIBDIR}", "-o", OUT]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return OUT


@pytest.fixture(scope="module")
def shim_binary(_built_libraries):
    return _build()


def test_shim_header_compiles_and_host_cases_pass(shim_binary):
    r = subprocess.run([shim_binary, "--host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout


@pytest.mark.gpu
def test_shim_device_cases(gpu, shim_binary):
    r = subprocess.run([shim_binary], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
