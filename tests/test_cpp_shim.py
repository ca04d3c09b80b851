"""The C++ drop-in layer (include/scenopt_b200.hpp, the reference's
namespace-scenopt API over the C-ABI), exercised by tests/cpp/test_shim.cpp:
reference-style cases for the oracles, FBE, L-BFGS and solvers. Host-only
cases run here; the device cases run under the gpu marker."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2107_01745_b200", "lib")
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")


def _build(name):
    os.makedirs(BUILD, exist_ok=True)
    out = os.path.join(BUILD, name)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), f"-L{LIBDIR}", "-lscenopt_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.fixture(scope="module")
def shim_binary(_built_libraries):
    return _build("test_shim")


@pytest.fixture(scope="module")
def sample_binary(_built_libraries):
    return _build("sample_markov")


def test_shim_header_compiles_and_host_cases_pass(shim_binary):
    r = subprocess.run([shim_binary, "--host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout


@pytest.mark.gpu
def test_shim_device_cases(gpu, shim_binary):
    r = subprocess.run([shim_binary], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


@pytest.mark.gpu
def test_reference_style_sample_solves_and_verifies(gpu, sample_binary):
    r = subprocess.run([sample_binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "verified 1" in r.stdout


def test_reference_style_sample_compiles(sample_binary):
    assert os.path.exists(sample_binary)
