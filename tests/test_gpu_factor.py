"""factor() on the device (K9, cuda/factor.cu) against
the CPU oracle's restatement of riccati.hpp:82-182: every FactorCache member
read back from the packed sweep layout, sweeps and solves of the
device-factored handle, and the strong-convexity rejection
(test_riccati.cpp:52-64)."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

pytestmark = pytest.mark.gpu


def _cmp(a: dict, b: dict, tol):
    for k in a:
        n = min(a[k].size, b[k].size)
        if n:
            scale = 1.0 + np.abs(b[k][:n]).max()
            err = np.abs(a[k][:n] - b[k][:n]).max() / scale
            assert err <= tol, (k, err)


def test_device_factor_matches_oracle_on_random_trees(gpu):
    rng = orc.Rng(41)
    for trial in range(12):
        po = rng.random_instance(rng.integer(1, 5), 40, rng.integer(1, 5), rng.integer(1, 4),
                                 orc.InstanceOptions(with_l1=True, with_none=True))
        prob = so.ProblemInstance.from_flat(po.flat())
        _cmp(so.factor_device(prob).export(), orc.Factor(po).export(), 1e-10)


@pytest.mark.parametrize("shape", [(10, 5, 10, [2, 2, 2]), (50, 20, 4, [8, 8]), (20, 8, 6, [3, 1, 4]),
                                   (120, 40, 2, [3])])
def test_device_factor_sweeps_and_solves_match_oracle(gpu, shape):
    nx, nu, N, br = shape
    prob = so.gen_random_instance(1, nx, nu, N, br)
    po = orc.Problem.from_flat(prob.flat())
    ofac = orc.Factor(po)
    cache = so.factor_device(prob)
    _cmp(cache.export(), ofac.export(), 1e-10)
    y = np.random.default_rng(2).uniform(-1, 1, prob.dual_dim)
    for fn, ofn in ((so.dual_grad, ofac.dual_grad), (so.hessian_vec, ofac.hessian_vec)):
        pt = fn(cache, prob, y)
        ox, ou = ofn(y)
        assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < 1e-9
    if nx <= 50:
        cfg = so.SolverConfig(nama_parallel_linesearch=True)
        rep = so.api._solve_direct("nama", prob, cache, cfg)
        orep = orc.solve(po, orc.SolverConfig(), 1)
        assert rep.status == "converged"
        assert abs(rep.iterations - orep["iterations"]) <= 1


def test_device_factor_rejects_singular_input_hessian(gpu):
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
        so.factor_device(so.ProblemInstance.from_flat(flat))


def _perturbed(flat, rng, root=True):
    f2 = dict(flat)
    n, nx, nu = flat["num_nodes"], flat["nx"], flat["nu"]
    f2["q"] = flat["q"] + np.r_[np.zeros(nx), rng.vector((n - 1) * nx)]
    f2["r"] = flat["r"] + np.r_[np.zeros(nu), rng.vector((n - 1) * nu)]
    f2["c"] = flat["c"] + np.r_[np.zeros(nx), rng.vector((n - 1) * nx)]
    f2["p"] = flat["p"] + rng.vector(flat["p"].size)
    if root:
        f2["root_state"] = flat["root_state"] + rng.vector(nx)
    return f2


def test_device_refactor_affine_matches_host_and_fresh_factor(gpu):
    rng = orc.Rng(34)  # test_riccati.cpp:66-90
    for trial in range(3):
        po = rng.random_instance(3, 40, 3, 2, orc.InstanceOptions(with_l1=True))
        flat = po.flat()
        prob = so.ProblemInstance.from_flat(flat)
        cache = so.factor_device(prob)
        prob2 = so.ProblemInstance.from_flat(_perturbed(flat, rng))
        so.refactor_affine(cache, prob2)
        host = so.factor(prob)
        so.refactor_affine(host, prob2)
        _cmp(cache.export(), host.export(), 1e-10)
        _cmp(cache.export(), so.factor_device(prob2).export(), 1e-10)
        # the updated handle sweeps the new problem (root state included)
        po2 = orc.Problem.from_flat(prob2.flat())
        ofac = orc.Factor(po2)
        y = rng.vector(prob.dual_dim)
        pt = so.dual_grad(cache, prob2, y)
        ox, ou = ofac.dual_grad(y)
        assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < 1e-9
        assert abs(so.fhat_value(cache, prob2, y) - ofac.fhat_value(y)) <= 1e-9 * (1 + abs(ofac.fhat_value(y)))


def test_mpc_style_resolve_after_refactor_affine(gpu):
    """Receding horizon: new initial state and linear terms each step, one
    device factor; each re-solve matches the oracle solve of that step."""
    prob = so.gen_random_instance(1, 10, 5, 10, [2, 2, 2])  # BASELINE C1 shape (well conditioned)
    cache = so.factor_device(prob)
    rng = orc.Rng(5)
    flat = prob.flat()
    for step in range(3):
        f2 = dict(flat)
        f2["root_state"] = 0.02 * rng.vector(flat["nx"])
        f2["q"] = flat["q"] * (1.0 + 0.05 * step)
        prob2 = so.ProblemInstance.from_flat(f2)
        so.refactor_affine(cache, prob2)
        rep = so.api._solve_direct("nama", prob2, cache, so.SolverConfig(nama_parallel_linesearch=True))
        orep = orc.solve(orc.Problem.from_flat(f2), orc.SolverConfig(), 1)
        assert rep.status == "converged"
        assert abs(rep.iterations - orep["iterations"]) <= 1
        assert np.abs(rep.x.x.ravel(order="F") - orep["x"]).max() < 1e-3 * (1 + np.abs(orep["x"]).max())


@pytest.mark.parametrize("flat", ["1", "0"])
def test_device_factor_flattened_top_on_c3(gpu, monkeypatch, flat):
    """Device-factored handle at C3: the flattened forward top's maps
    (G = CL G_p, L = (F + G'K_p) G_p, a' = CL a'_p + c, h' = (F + G'K_p) a'_p)
    computed on the device after K9 (factor_flat, cuda/factor.cu), against the
    oracle; then refactor_affine (new c / q / r / p_N / root state) recomputes
    the constants a' / h' and the handle sweeps the new problem."""
    monkeypatch.setenv("SCENOPT_FLAT_TOP", flat)
    prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
    cache = so.factor_device(prob)
    info = cache.dev_info()
    assert info["cut_stage"] == 4 and info["device_factor"] == 1 and info["flat_top"] == int(flat)
    rng = np.random.default_rng(12)
    y = rng.uniform(-1, 1, prob.dual_dim)
    r = rng.uniform(-1, 1, prob.dual_dim)
    flat_data = prob.flat()
    for step in range(2):
        po = orc.Problem.from_flat(prob.flat())
        ofac = orc.Factor(po)
        for affine in (True, False):
            pts, hs = so.sweep(cache, [y, r], affine)
            for v, pt, h in ((y, pts[0], hs[0]), (r, pts[1], hs[1])):
                ox, ou = ofac.sweep(v, affine)
                assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < 1e-9
                Hx = orc.apply_H(po, ox, ou)
                assert np.abs(h - Hx).max() <= 1e-9 * (1 + np.abs(Hx).max())
        if step == 0:
            prob = so.ProblemInstance.from_flat(_perturbed(flat_data, orc.Rng(5)))
            so.refactor_affine(cache, prob)
