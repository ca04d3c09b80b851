"""Spring-mass benchmark generator (generators.hpp:39-234)
against the reference's own tests (test_generators.cpp:42-193) and the CPU
oracle's restatement. The oracle discretizes with the series exponential of
test_generators.cpp:23-38; the product uses Pade scaling and squaring, so
A_d / B_d agree to 1e-10 (the reference's bound) and everything else is
bit-identical. Host-only: no GPU needed."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup


def test_defaults_produce_the_benchmark_dimensions():
    f = so.gen_spring_mass(5).flat()  # test_generators.cpp:42-49
    assert (f["nx"], f["nu"], f["num_stages"], f["num_nodes"]) == (10, 4, 11, 4095)
    assert f["num_nodes"] - f["stage_offsets"][11] == 2048


def test_instance_carries_the_documented_structure():
    par = so.SpringMassParams(horizon=3)  # test_generators.cpp:51-93
    prob = so.gen_spring_mass(5, par)
    f = prob.flat()
    assert f["num_nodes"] == 15 and f["num_nodes"] - f["stage_offsets"][3] == 8
    assert prob.validate() == []
    assert prob.dual_dim == 14 * 9 + 8 * 5
    assert f["probability"][1] == 0.5 and f["probability"][2] == 0.5
    tree = orc.tree_from_markov(np.array([[0.1, 0.9], [0.9, 0.1]]), np.array([0.5, 0.5]), 3)
    assert np.array_equal(tree["ancestor"], f["ancestor"])
    assert np.array_equal(tree["probability"], f["probability"])
    lay = orc.layout(f)
    for i in range(1, 15):
        assert f["stage_rows"][i] == 9
        assert np.array_equal(sup.node_mat(f, "Q", i, 10, 10), 5.0 * np.eye(10))
        assert np.array_equal(sup.node_mat(f, "R", i, 4, 4), 2.0 * np.eye(4))
        assert not sup.node_mat(f, "S", i, 4, 10).any()
        mode = tree["mode"][i]
        assert np.array_equal(sup.node_vec(f, "c", i, 10), np.zeros(10) if mode == 0 else np.full(10, 0.1))
        assert f["g_kind"][i] == 1
        off = int(lay["dual_offset"][i])
        assert np.array_equal(f["zmin"][off:off + 5], np.full(5, -5.0))
        assert np.array_equal(f["zmax"][off:off + 5], np.full(5, 5.0))
        assert np.array_equal(f["zmin"][off + 5:off + 9], np.full(4, -2.0))
        assert np.array_equal(f["zmax"][off + 5:off + 9], np.full(4, 2.0))
        F, G = sup.con_F(f, lay, i), sup.con_G(f, lay, i)
        assert np.array_equal(F[:5, 5:], np.eye(5)) and not F[:5, :5].any() and not F[5:].any()
        assert np.array_equal(G[5:], np.eye(4)) and not G[:5].any()
    for l in range(8):
        assert f["terminal_rows"][l] == 5
        assert np.array_equal(sup.node_mat(f, "P", l, 10, 10), 100.0 * np.eye(10))
        off = int(lay["tdual_offset"][l])
        assert np.array_equal(f["zmax"][off:off + 5], np.full(5, 5.0))
        assert np.array_equal(sup.term_F(f, lay, l), np.eye(10)[5:])


@pytest.mark.parametrize("masses", [2, 3, 5])
def test_zero_order_hold_matches_the_series_exponential(masses):
    par = so.SpringMassParams(horizon=1)  # test_generators.cpp:95-115
    f = so.gen_spring_mass(masses, par).flat()
    nx, nu = 2 * masses, masses - 1
    Ac, Bc = orc.spring_mass_continuous(masses, par)
    Ap, Bp = so.spring_mass_continuous(masses, par)
    assert np.array_equal(Ac, Ap) and np.array_equal(Bc, Bp)
    aug = np.zeros((nx + nu, nx + nu))
    aug[:nx, :nx], aug[:nx, nx:] = Ac, Bc
    big = orc.expm_series(aug * par.sampling)
    assert np.abs(sup.node_mat(f, "A", 1, nx, nx) - big[:nx, :nx]).max() < 1e-10
    assert np.abs(sup.node_mat(f, "B", 1, nx, nu) - big[:nx, nx:]).max() < 1e-10
    Ad, Bd = so.discretize_zoh(Ac, Bc, par.sampling)
    assert np.abs(Ad - big[:nx, :nx]).max() < 1e-10 and np.abs(Bd - big[:nx, nx:]).max() < 1e-10


def test_expm_against_the_series_and_closed_forms():
    rng = np.random.default_rng(3)
    for n, scale in ((1, 0.01), (4, 0.1), (6, 1.0), (9, 3.0), (12, 12.0)):  # every Pade degree
        X = scale * rng.uniform(-1, 1, (n, n))
        E, R = so.expm(X), orc.expm_series(X)
        assert np.abs(E - R).max() <= 1e-12 * max(1.0, np.abs(R).max())
    th = 0.7  # rotation generator
    E = so.expm(np.array([[0.0, -th], [th, 0.0]]))
    assert np.abs(E - np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])).max() < 1e-15
    N = np.triu(np.ones((4, 4)), 1)  # nilpotent: exp = I + N + N^2/2 + N^3/6
    assert np.abs(so.expm(N) - (np.eye(4) + N + N @ N / 2 + N @ N @ N / 6)).max() < 1e-14


def test_free_particles_discretize_to_double_integrators():
    par = so.SpringMassParams(stiffness=0.0, damping=0.0, horizon=1)  # test_generators.cpp:117-130
    A = sup.node_mat(so.gen_spring_mass(4, par).flat(), "A", 1, 8, 8)
    eye = np.eye(4)
    assert np.abs(A[4:, 4:] - eye).max() < 1e-12 and np.abs(A[:4, :4] - eye).max() < 1e-12
    assert np.abs(A[:4, 4:] - par.sampling * eye).max() < 1e-12 and np.abs(A[4:, :4]).max() < 1e-12


def test_rejects_out_of_range_parameters():
    with pytest.raises(so.InvalidParams):  # test_generators.cpp:132-145
        so.gen_spring_mass(1)
    with pytest.raises(so.InvalidParams):
        so.gen_spring_mass(5, so.SpringMassParams(mass_kg=0.0))
    with pytest.raises(so.DimensionMismatch):
        so.gen_spring_mass(5, so.SpringMassParams(mode_values=np.zeros(3)))
    with pytest.raises(so.DimensionMismatch):
        so.gen_spring_mass(5, so.SpringMassParams(root_state=np.zeros(3)))
    with pytest.raises(so.InvalidParams):
        so.gen_spring_mass(5, so.SpringMassParams(sampling=0.0))
    with pytest.raises(so.NonStochasticMatrix):
        so.gen_spring_mass(5, so.SpringMassParams(transition=np.array([[0.5, 0.6], [0.5, 0.5]])))
    for bad in (dict(mass_kg=0.0), dict(mode_values=np.zeros(3)), dict(root_state=np.zeros(3))):
        with pytest.raises(orc.OracleError):
            orc.gen_spring_mass(5, so.SpringMassParams(**bad))


@pytest.mark.parametrize("masses,par", [
    (5, so.SpringMassParams(horizon=4)),
    (3, so.SpringMassParams(horizon=5, root_state=np.linspace(-1, 1, 6))),
    # three modes with a zero transition (pruned branches) and custom weights
    (4, so.SpringMassParams(horizon=4, initial_probs=np.array([0.2, 0.3, 0.5]),
                            transition=np.array([[0.5, 0.5, 0.0], [0.0, 0.4, 0.6], [0.3, 0.3, 0.4]]),
                            mode_values=np.array([0.0, -0.05, 0.1]), state_weight=0.0, sampling=0.2)),
])
def test_product_generator_matches_oracle_restatement(masses, par):
    a = so.gen_spring_mass(masses, par).flat()
    b = orc.gen_spring_mass(masses, par).flat()
    assert a.keys() == b.keys()
    for k in a:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.shape == y.shape, k
        if k in ("A", "B"):
            assert np.abs(x - y).max() < 1e-12, k
        else:
            assert np.array_equal(x, y), k


def test_initial_state_samples_stay_inside_the_half_bound_box():
    # test_generators.cpp:182-193 asserts |state| <= 2.5 for every component, but the
    # code it tests draws positions from +-velocity_bound (generators.hpp:228-231:
    # pos_box = 1.0 * velocity_bound); code over comment: positions <= 5, velocities <= 2.5.
    par = so.SpringMassParams()
    s = so.sample_initial_state(5, par, seed=3, count=20)
    assert s.shape == (20, 10)
    assert np.abs(s).max() <= 2.5 * 2  # positions in +-velocity_bound, velocities in +-half
    assert np.abs(s[:, 5:]).max() <= 2.5
    assert np.array_equal(so.sample_initial_state(5, par, seed=7), so.sample_initial_state(5, par, seed=7))
    assert np.array_equal(s, orc.sample_initial_states(5, par, 3, 20))


def test_spring_mass_gap_comes_from_sampling_and_residual_scaling():
    """PAPER §IV-A reports 84 % of MINFBE / NAMA runs within 50 oracle calls
    and a GPAD median of 188; the reference code computes far less
    (profiles/spring_mass_study_r02.md). On the CPU oracle (the reference's
    restatement) this pins the two reference lines that explain the
    MINFBE / NAMA gap -- positions drawn in +-velocity_bound
    (generators.hpp:226) where the doc comment says half of it, and the
    preconditioned solve's residual measured back in original units
    (solvers.hpp:117-120) -- and that GPAD stays within 2x of NAMA either way."""
    M, H, S = 5, 8, 16

    class Par:
        horizon = H
        root_state = None

    x = orc.sample_initial_states(M, Par, seed=1, count=S).reshape(S, 2 * M)
    assert np.abs(x[:, :M]).max() > 2.5  # positions reach past half the bound (generators.hpp:226)

    def frac(kind, half, scaled):
        calls = []
        for x0 in x:
            p = Par()
            p.root_state = x0 * np.r_[np.full(M, 0.5 if half else 1.0), np.ones(M)]
            prob = orc.gen_spring_mass(M, p)
            cfg = orc.SolverConfig(eps=5e-4)
            if scaled:
                pre = prob.precondition()
                rep = orc.solve_direct(pre, orc.Factor(pre), cfg, kind)
            else:
                cfg.precondition = True
                rep = orc.solve(prob, cfg, kind)
            assert rep["status"] == 0
            calls.append(rep["dual_grad_calls"] + rep["hessian_vec_calls"])
        return np.mean(np.array(calls) <= 50), float(np.median(calls))

    ref = {k: frac(k, False, False) for k in (0, 1, 2)}
    both = {k: frac(k, True, True) for k in (0, 1, 2)}
    for k in (0, 1):  # MINFBE, NAMA
        assert ref[k][0] < 0.74 <= both[k][0], (k, ref[k], both[k])
    for d in (ref, both):  # GPAD median never 3x NAMA's (paper: 188 vs <= 50)
        assert d[2][1] < 2.0 * d[1][1]
