"""Host-side factor (riccati.hpp:82-216) of the product against the CPU
oracle, and the instance generator against the oracle's restatement of
generators.hpp:255-328. CPU-only: these run in the driver's CPU suite."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc


def _cmp_factor(a: dict, b: dict, tol=1e-12):
    for k in a:
        n = min(a[k].size, b[k].size)
        if n:
            scale = 1.0 + np.abs(b[k][:n]).max()
            assert np.abs(a[k][:n] - b[k][:n]).max() <= tol * scale, k


def test_factor_matches_oracle_on_random_trees():
    rng = orc.Rng(41)
    for trial in range(20):
        stages = rng.integer(1, 5)
        po = rng.random_instance(stages, 40, rng.integer(1, 4), rng.integer(1, 4),
                                 orc.InstanceOptions(with_l1=True, with_none=True))
        prob = so.ProblemInstance.from_flat(po.flat())
        _cmp_factor(so.factor(prob).export(), orc.Factor(po).export())


def test_refactor_affine_matches_fresh_factor():
    rng = orc.Rng(34)  # test_riccati.cpp:66-90
    po = rng.random_instance(3, 25, 3, 2)
    flat = po.flat()
    prob = so.ProblemInstance.from_flat(flat)
    cache = so.factor(prob)
    f2 = dict(flat)
    n, nx, nu = flat["num_nodes"], flat["nx"], flat["nu"]
    f2["q"] = flat["q"] + np.r_[np.zeros(nx), rng.vector((n - 1) * nx)]
    f2["r"] = flat["r"] + np.r_[np.zeros(nu), rng.vector((n - 1) * nu)]
    f2["c"] = flat["c"] + np.r_[np.zeros(nx), rng.vector((n - 1) * nx)]
    f2["p"] = flat["p"] + rng.vector(flat["p"].size)
    prob2 = so.ProblemInstance.from_flat(f2)
    so.refactor_affine(cache, prob2)
    _cmp_factor(cache.export(), so.factor(prob2).export(), 1e-12)


def test_factor_rejects_singular_input_hessian():
    rng = orc.Rng(33)  # test_riccati.cpp:52-64
    po = rng.random_instance(2, 10, 2, 2)
    flat = dict(po.flat())
    nu, nx = flat["nu"], flat["nx"]
    kids = [i for i in range(1, flat["num_nodes"]) if flat["ancestor"][i] == 1]
    R, S, B = flat["R"].copy(), flat["S"].copy(), flat["B"].copy()
    for c in kids:
        R[c * nu * nu:(c + 1) * nu * nu] = (1e-14 * np.eye(nu)).ravel()
        S[c * nu * nx:(c + 1) * nu * nx] = 0.0
        B[c * nx * nu:(c + 1) * nx * nu] = 0.0
    flat.update(R=R, S=S, B=B)
    with pytest.raises(so.NotStronglyConvex):
        so.factor(so.ProblemInstance.from_flat(flat))
    with pytest.raises(orc.OracleError):
        orc.Factor(orc.Problem.from_flat(flat))


@pytest.mark.parametrize("shape", [(10, 5, 10, [2, 2, 2]), (3, 2, 3, [2, 2, 2]),
                                   (7, 3, 5, [3, 1, 2]), (16, 6, 4, [4, 4])])
def test_generator_matches_oracle_restatement(shape):
    nx, nu, N, br = shape
    a = so.gen_random_instance(1, nx, nu, N, br).flat()
    b = orc.gen_random(1, nx, nu, N, br).flat()
    for k in b:
        x, y = np.asarray(a[k], dtype=float), np.asarray(b[k], dtype=float)
        assert x.shape == y.shape, k
        # identical draw streams; only the spectral radius (QR iteration)
        # may differ in the last bits
        assert np.abs(x - y).max(initial=0.0) <= 1e-13 * (1 + np.abs(y).max(initial=0.0)), k


def test_generator_dims_and_feasible_origin():
    prob = so.gen_random_instance(1, 10, 5, 10, [2, 2, 2])
    flat = prob.flat()
    assert prob.num_nodes() == 71 and prob.num_leaves == 8 and prob.dual_dim == 148
    assert prob.validate() == []
    assert np.all(flat["zmin"] < 0) and np.all(flat["zmax"] > 0)
    nx = flat["nx"]
    for i in range(1, flat["num_nodes"]):
        A = flat["A"][i * nx * nx:(i + 1) * nx * nx].reshape((nx, nx), order="F")
        assert abs(np.abs(np.linalg.eigvals(A)).max() - 0.95) < 1e-12


def test_generator_reproduces_from_seed():
    a = so.gen_random_instance(42, 3, 2, 3, 2).flat()
    b = so.gen_random_instance(42, 3, 2, 3, 2).flat()
    c = so.gen_random_instance(43, 3, 2, 3, 2).flat()
    assert all(np.array_equal(a[k], b[k]) for k in a if isinstance(a[k], np.ndarray))
    assert not np.array_equal(a["A"], c["A"])


def test_c3_shape():
    """C3 of BASELINE.json: nx=50, nu=20, N=20, branching [8,8,8,2]."""
    n = 1 + 8 + 64 + 512 + 1024 * 17
    assert n == 17993
    prim = 16969 * 20 + (n - 1) * 50
    assert prim == 1_238_980
