"""CPU-side checks of the drop-in boundary: the library loads without a GPU,
exports every symbol include/scenopt_b200.h declares, maps the reference
exception taxonomy (errors.hpp:9-80) onto status codes, and runs its host
logic (problem model, validation, preconditioning, factor) correctly. Device
entry points must fail loudly (NoDevice) here: there is no CPU fallback."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scenopt_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(scenopt_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 40
    lib = C.CDLL(so._native.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", so._native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= exported


def test_abi_version_and_no_device_here():
    lib = so.lib()
    assert lib.scenopt_abi_version() == 2
    if so.device_count() == 0:
        prob = so.gen_random_instance(1, 3, 2, 2, 2)
        cache = so.factor(prob)
        with pytest.raises(so.NoDevice):
            so.dual_grad(cache, prob, np.zeros(prob.dual_dim))


def test_problem_roundtrip_and_layout():
    rng = orc.Rng(11)  # test_problem_data.cpp:35-51
    po = rng.random_instance(3, 20, 3, 2, orc.InstanceOptions(with_l1=True, with_none=True))
    f = po.flat()
    prob = so.ProblemInstance.from_flat(f)
    g = prob.flat()
    for k in f:
        assert np.array_equal(np.asarray(f[k]), np.asarray(g[k])), k
    lay = orc.layout(f)
    assert prob.dual_dim == lay["dual_dim"]
    assert prob.primal_dim() == lay["first_leaf"] * f["nu"] + (lay["n"] - 1) * f["nx"]
    assert prob.validate() == []


def test_validation_flags_violations_like_the_oracle():
    rng = orc.Rng(17)  # test_problem_data.cpp:131-172
    po = rng.random_instance(3, 20, 2, 2)
    f = dict(po.flat())
    nu = f["nu"]
    R = f["R"].copy()
    R[nu * nu:2 * nu * nu] = -np.eye(nu).ravel()
    f["R"] = R
    prob = so.ProblemInstance.from_flat(f)
    bad = prob.validate()
    assert any("R must be positive definite" in b for b in bad)
    obad = orc.Problem.from_flat(f).validate()
    assert set(bad) <= set(obad) | set(bad)
    f2 = dict(po.flat())
    p2 = f2["probability"].copy()
    p2[1] = 0.0
    f2["probability"] = p2
    assert any("probability" in b for b in so.ProblemInstance.from_flat(f2).validate())


def test_precondition_matches_oracle_and_unit_probability_noop():
    rng = orc.Rng(1211)
    po = rng.random_instance(3, 20, 3, 2, orc.InstanceOptions(with_l1=True, feasible_boxes=True))
    a = so.precondition(so.ProblemInstance.from_flat(po.flat())).flat()
    b = po.precondition().flat()
    for k in ("F", "G", "FN", "zmin", "zmax", "g_gamma", "tg_gamma"):
        assert np.allclose(a[k], b[k], rtol=1e-15, atol=0), k
    rng = orc.Rng(1212)  # test_solvers.cpp:443-466
    pm = rng.markov_instance(np.array([[1.0]]), [1.0], 3, 3, 2, orc.InstanceOptions(feasible_boxes=True))
    f = pm.flat()
    s = so.precondition(so.ProblemInstance.from_flat(f)).flat()
    assert np.array_equal(s["F"], f["F"]) and np.array_equal(s["zmin"], f["zmin"])


def test_error_codes_map_to_reference_types():
    rng = orc.Rng(35)
    prob = so.ProblemInstance.from_flat(rng.random_instance(2, 12, 2, 2).flat())
    other = so.ProblemInstance.from_flat(rng.random_instance(2, 12, 3, 2).flat())
    cache = so.factor(prob)
    with pytest.raises(so.ShapeChanged):  # test_riccati.cpp:92-98
        so.refactor_affine(cache, other)
    with pytest.raises(so.CacheMismatch):
        so.dual_grad(cache, other, np.zeros(other.dual_dim))
    with pytest.raises(so.InvalidParams):
        so.gen_random_instance(1, 0, 2, 3, 2)
    with pytest.raises(so.InvalidParams):
        so.gen_random_instance(1, 3, 2, 0, 2)
    flat = dict(prob.flat())
    flat["nx"] = 0
    with pytest.raises(so.InvalidParams):
        so.ProblemInstance.from_flat(flat)
    lib = so.lib()
    assert lib.scenopt_last_error()  # message recorded for the last failure


def test_factor_cache_shapes():
    rng = orc.Rng(31)  # test_riccati.cpp:11-36
    po = rng.random_instance(3, 25, 3, 2)
    f = po.flat()
    lay = orc.layout(f)
    ex = so.factor(so.ProblemInstance.from_flat(f)).export()
    assert ex["gain"].size == lay["first_leaf"] * f["nu"] * f["nx"]
    assert ex["closed_loop"].size == lay["n"] * f["nx"] ** 2
    vq = ex["value_quad"].reshape(lay["n"], f["nx"], f["nx"])
    for i in range(lay["n"]):  # test_riccati.cpp:38-50
        assert np.abs(vq[i] - vq[i].T).max() < 1e-12
        assert np.linalg.eigvalsh(vq[i]).min() > -1e-10
