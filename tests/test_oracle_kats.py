"""Pins the CPU oracle (test infrastructure) against every known-answer test
the reference suite holds for this path, and against the reference's own
ground-truth property oracles restated in numpy (tests/support.py).

KAT sources: test_prox.cpp:44-67, 82-101, 103-134, 136-164;
test_scenario_tree.cpp:20-64; test_lbfgs.cpp:177-192; SPEC.md scenario_tree
examples; test_tree_oracles.cpp:23-152; test_problem_data.cpp:87-130."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import support as sup

INF = float("inf")


def mixed_g():
    """test_prox.cpp:23-44: box on [-1,2]^2 (w .25), l1 (w .5, gamma .8), none."""
    return orc.Nonsmooth.from_blocks(6, [
        dict(offset=0, size=2, weight=0.25, kind=1, zmin=[-1, -1], zmax=[2, 2]),
        dict(offset=2, size=2, weight=0.5, kind=2, gamma=0.8),
        dict(offset=4, size=2, weight=0.25, kind=0)])


def test_prox_box_clamps_independently_of_scale():
    g = mixed_g()
    v = np.array([-3.0, 1.5, 0.0, 0.0, 7.0, -7.0])
    for scale in (0.3, 1.0, 10.0):
        out = g.prox(v, scale)
        assert out[0] == -1.0 and out[1] == 1.5 and out[4] == 7.0 and out[5] == -7.0


def test_prox_l1_soft_threshold():
    g = mixed_g()
    t = 2.0 * 0.5 * 0.8
    v = np.zeros(6)
    v[2], v[3] = 1.3, -t / 2
    out = g.prox(v, 2.0)
    assert out[2] == pytest.approx(1.3 - t) and out[3] == 0.0


def test_prox_optimality_fenchel_and_moreau():
    g = mixed_g()
    rng = orc.Rng(21)
    for _ in range(40):
        v = rng.vector(6, 4.0)
        s = rng.uniform(0.1, 3.0)
        z = g.prox(v, s)
        assert g.dist_subdiff_inf((v - z) / s, z) < 1e-12
    rng = orc.Rng(22)
    for _ in range(40):
        v = rng.vector(6, 3.0)
        z = g.prox(v, 1.0)
        w = v - z
        conj = g.conj(w)
        assert np.isfinite(conj)
        assert w @ z == pytest.approx(0.5 * 0.8 * np.abs(z[2:4]).sum() + conj, abs=1e-12)
    rng = orc.Rng(23)
    for lam in (0.2, 1.0, 4.0):
        v = rng.vector(6, 3.0)
        w = g.prox_conj(v, lam)
        assert g.dist_subdiff_inf(w, (v - w) / lam) < 1e-12


def test_conjugate_known_values():
    g = mixed_g()
    w = np.zeros(6)
    w[0], w[1] = -2.0, 3.0
    assert g.conj(w) == pytest.approx(8.0)
    w[2] = 0.4
    assert g.conj(w) == pytest.approx(8.0)
    w[2] = 0.5
    assert g.conj(w) == INF
    w[2] = 0.0
    w[4] = 1e-12
    assert np.isfinite(g.conj(w))
    w[4] = 0.1
    assert g.conj(w) == INF


def test_subdifferential_distance_known_values():
    g = mixed_g()
    z, y = np.zeros(6), np.zeros(6)
    z[0], y[0] = 0.5, 0.3
    assert g.dist_subdiff_inf(y, z) == pytest.approx(0.3)
    z[0] = 2.0
    assert g.dist_subdiff_inf(y, z) == 0.0
    y[0] = -0.2
    assert g.dist_subdiff_inf(y, z) == pytest.approx(0.2)
    y[0] = z[0] = 0.0
    z[2], y[2] = 1.0, 0.4
    assert g.dist_subdiff_inf(y, z) == 0.0
    y[2] = 0.1
    assert g.dist_subdiff_inf(y, z) == pytest.approx(0.3)
    z[2] = 0.0
    assert g.dist_subdiff_inf(y, z) == 0.0
    y[2] = -0.6
    assert g.dist_subdiff_inf(y, z) == pytest.approx(0.2)


def test_prox_argument_validation():
    g = mixed_g()
    with pytest.raises(orc.OracleError, match="InvalidParams"):
        g.prox(np.zeros(6), 0.0)
    with pytest.raises(orc.OracleError, match="InvalidParams"):
        g.prox_conj(np.zeros(6), -1.0)


def test_markov_tree_known_answers():
    P = np.array([[0.1, 0.9], [0.9, 0.1]])
    t = orc.tree_from_markov(P, [0.5, 0.5], 3)
    assert t["num_nodes"] == 15 and list(t["stage_offsets"]) == [0, 1, 3, 7, 15]
    assert t["probability"][0] == 1.0 and t["mode"][0] == -1
    assert t["mode"][1] == 0 and t["probability"][1] == pytest.approx(0.5)
    kids = [i for i in range(15) if t["ancestor"][i] == 1]
    assert t["probability"][kids[0]] == pytest.approx(0.05)
    assert t["probability"][kids[1]] == pytest.approx(0.45)
    t2 = orc.tree_from_markov(P, [0.5, 0.5], 2)  # SPEC.md example
    leaves = t2["probability"][t2["stage_offsets"][2]:]
    assert np.allclose(leaves, [0.05, 0.45, 0.45, 0.05])
    t3 = orc.tree_from_markov(np.array([[1.0, 0.0], [0.5, 0.5]]), [1.0, 0.0], 4)
    assert t3["num_nodes"] == 5 and np.all(t3["probability"] == 1.0)
    with pytest.raises(orc.OracleError, match="InvalidParams"):
        orc.tree_from_markov(P, [0.5, 0.5], 0)
    with pytest.raises(orc.OracleError, match="NonStochasticMatrix"):
        orc.tree_from_markov(np.array([[0.5, 0.6], [0.5, 0.5]]), [0.5, 0.5], 2)


def test_lbfgs_known_answers():
    rng = orc.Rng(87)  # test_lbfgs.cpp:177-192: gamma0 == 0.4
    buf = orc.Lbfgs(4, 1e-12)
    for _ in range(4):
        s = rng.vector(5)
        buf.push(s, 2.5 * s, 1.0)
    assert buf.gamma0() == pytest.approx(0.4, abs=1e-14)
    buf.clear()
    assert buf.size() == 0 and buf.gamma0() == 1.0
    rng = orc.Rng(83)
    for _ in range(5):
        dim, memory = rng.integer(4, 12), rng.integer(2, 6)
        b = orc.Lbfgs(memory, 1e-12)
        root = rng.matrix(dim, dim)
        spd = root @ root.T + 0.5 * np.eye(dim)
        acc = []
        for _ in range(memory + rng.integer(0, 3)):
            s = rng.vector(dim)
            assert b.push(s, spd @ s, 1.0)
            acc = (acc + [(s, spd @ s)])[-memory:]
        gam = acc[-1][0] @ acc[-1][1] / (acc[-1][1] @ acc[-1][1])
        inv = sup.dense_bfgs_inverse(acc, dim, gam)
        g = rng.vector(dim)
        assert np.abs(b.apply_direction(g) + inv @ g).max() < 1e-11 * (1 + np.abs(inv @ g).max())


def test_dual_grad_matches_dense_kkt():
    rng = orc.Rng(41)  # test_tree_oracles.cpp:23-36
    for trial in range(20):
        po = rng.random_instance(rng.integer(1, 5), 40, rng.integer(1, 4), rng.integer(1, 4))
        fac = orc.Factor(po)
        y = rng.vector(po.dual_dim, 2.0)
        x, u = fac.dual_grad(y)
        kx, ku = sup.kkt_dual_grad(po.flat(), y)
        assert sup.rel_gap(kx, ku, x, u) < 1e-8


def test_hessian_exact_symmetric_psd_and_fd():
    rng = orc.Rng(44)  # test_tree_oracles.cpp:83-126
    po = rng.random_instance(3, 30, 3, 2)
    fac = orc.Factor(po)
    for _ in range(5):
        y, r = rng.vector(po.dual_dim, 2.0), rng.vector(po.dual_dim, 2.0)
        gy = -orc.apply_H(po, *fac.dual_grad(y))
        gyr = -orc.apply_H(po, *fac.dual_grad(y + r))
        hr = -orc.apply_H(po, *fac.hessian_vec(r))
        assert np.abs(gyr - gy - hr).max() < 1e-9 * (1 + np.abs(hr).max())
        a, b = rng.vector(po.dual_dim), rng.vector(po.dual_dim)
        ab = a @ -orc.apply_H(po, *fac.hessian_vec(b))
        ba = b @ -orc.apply_H(po, *fac.hessian_vec(a))
        assert ab == pytest.approx(ba, rel=1e-9, abs=1e-12)
        assert r @ hr > -1e-10
    rng = orc.Rng(45)
    po = rng.random_instance(2, 15, 2, 2)
    fac = orc.Factor(po)
    for _ in range(5):
        y = rng.vector(po.dual_dim)
        d = rng.vector(po.dual_dim)
        d /= np.linalg.norm(d)
        h = 1e-4
        fd = (fac.fhat_value(y + h * d) - fac.fhat_value(y - h * d)) / (2 * h)
        an = -orc.apply_H(po, *fac.dual_grad(y)) @ d
        assert fd == pytest.approx(an, rel=1e-6, abs=1e-8)


def test_eval_f_infeasibility_and_apply_H_adjoint():
    rng = orc.Rng(16)  # test_problem_data.cpp:115-130, 66-77
    po = rng.random_instance(2, 10, 2, 1)
    f = po.flat()
    lay = orc.layout(f)
    x = np.zeros((f["nx"], lay["n"]))
    u = rng.matrix(f["nu"], lay["first_leaf"])
    x[:, 0] = f["root_state"]
    for i in range(1, lay["n"]):
        a = f["ancestor"][i]
        x[:, i] = (sup.node_mat(f, "A", i, f["nx"], f["nx"]) @ x[:, a]
                   + sup.node_mat(f, "B", i, f["nx"], f["nu"]) @ u[:, a] + sup.node_vec(f, "c", i, f["nx"]))
    xf, uf = x.ravel(order="F"), u.ravel(order="F")
    assert np.isfinite(orc.eval_f(po, xf, uf))
    x2 = x.copy()
    x2[:, 0] += 1e-3
    assert orc.eval_f(po, x2.ravel(order="F"), uf) == INF
    x3 = x.copy()
    x3[:, -1] += 1e-3
    assert orc.eval_f(po, x3.ravel(order="F"), uf) == INF
    H = sup.dense_H(f)
    z = orc.apply_H(po, xf, uf)
    assert np.abs(z - H @ np.r_[uf, xf]).max() < 1e-12
    y = rng.vector(po.dual_dim)
    ax, au = orc.apply_H_adjoint(po, y)
    assert z @ y == pytest.approx(np.r_[au, ax] @ np.r_[uf, xf], rel=1e-12)


def test_oracle_solvers_match_admm_reference():
    rng = orc.Rng(1202)  # test_solvers.cpp:229-246
    for trial in range(2):
        opt = orc.InstanceOptions(with_box=True, with_l1=trial == 1, with_none=trial == 1,
                                  feasible_boxes=True)
        po = rng.random_instance(rng.integer(2, 3), 12, rng.integer(2, 3), 2, opt)
        rx, ru = sup.admm_reference(po.flat(), sup.blocks_of(po.flat()))
        for kind in (0, 1, 2):
            rep = orc.solve(po, orc.SolverConfig(eps=1e-6), kind)
            assert rep["status"] == 0
            assert max(np.abs(rep["x"] - rx).max(), np.abs(rep["u"] - ru).max()) < 1e-4


def test_oracle_generator_spectral_radius_and_layout():
    po = orc.gen_random(9, 3, 2, 3, [2, 2, 2])
    f = po.flat()
    for i in range(1, f["num_nodes"]):
        A = sup.node_mat(f, "A", i, 3, 3)
        assert abs(np.abs(np.linalg.eigvals(A)).max() - 0.95) < 1e-12
    assert po.validate() == []
    assert np.all(f["zmin"] < 0) and np.all(f["zmax"] > 0)
