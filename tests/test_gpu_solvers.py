"""GPU solver parity (solvers.hpp) against the CPU oracle and the
reference's own solver properties (test_solvers.cpp). North-star bar:
identical iteration counts within +-1 and iterates within the tolerance."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

pytestmark = pytest.mark.gpu

KIND = {"minfbe": 0, "nama": 1, "gpad": 2}


def fixture(rng, opt, stages=3, max_nodes=12):
    po = rng.random_instance(rng.integer(2, stages), max_nodes, rng.integer(2, 3), 2, opt)
    prob = so.ProblemInstance.from_flat(po.flat())
    return po, prob


def feasible_box():
    return orc.InstanceOptions(with_box=True, feasible_boxes=True)


def mixed():
    return orc.InstanceOptions(with_box=True, with_l1=True, with_none=True, feasible_boxes=True)


def cfgs(**kw):
    rule = {"original": 0, "simple": 1, "none": 2}[kw.get("backtracking_rule", "simple")]
    okw = dict(kw)
    okw["backtracking_rule"] = rule
    return so.SolverConfig(**kw), orc.SolverConfig(**okw)


def agree(rep, orep, iters_tol=1):
    assert rep.status == ("converged" if orep["status"] == 0 else "max_iters_exceeded")
    assert abs(rep.iterations - orep["iterations"]) <= iters_tol, (rep.iterations, orep["iterations"])
    if rep.iterations == orep["iterations"]:
        assert rep.stats.dual_grad_calls == orep["dual_grad_calls"]
        assert rep.stats.hessian_vec_calls == orep["hessian_vec_calls"]


@pytest.mark.parametrize("kind", ["minfbe", "nama", "gpad"])
def test_solve_matches_oracle_on_random_trees(gpu, kind):
    rng = orc.Rng(1202)
    for trial in range(5):
        po, prob = fixture(rng, feasible_box() if trial % 2 == 0 else mixed())
        c, oc = cfgs(eps=1e-6)
        rep = so.solve(prob, c, kind)
        orep = orc.solve(po, oc, KIND[kind])
        agree(rep, orep)
        assert rep.verified and orep["verified"]
        scale = 1 + np.abs(orep["x"]).max()
        assert np.abs(rep.x.x.ravel(order="F") - orep["x"]).max() <= 10 * c.eps * scale
        assert rep.lipschitz_estimate == pytest.approx(orep["lipschitz_estimate"], rel=1e-9)


def test_solvers_match_admm_reference(gpu):
    rng = orc.Rng(1202)  # test_solvers.cpp:229-246
    for trial in range(3):
        po, prob = fixture(rng, feasible_box() if trial % 2 == 0 else mixed())
        ref_x, ref_u = sup.admm_reference(po.flat(), sup.blocks_of(po.flat()))
        c, _ = cfgs(eps=1e-6)
        for kind in ("minfbe", "nama", "gpad"):
            rep = so.solve(prob, c, kind)
            assert rep.status == "converged"
            gap = max(np.abs(rep.x.u.ravel(order="F") - ref_u).max(),
                      np.abs(rep.x.x.ravel(order="F") - ref_x).max())
            assert gap < 1e-4


def test_unconstrained_duals_converge_immediately(gpu):
    rng = orc.Rng(1201)  # test_solvers.cpp:197-227
    opt = orc.InstanceOptions(with_box=False, with_none=True)
    for trial in range(3):
        po, prob = fixture(rng, opt)
        c, _ = cfgs()
        for kind in ("minfbe", "nama", "gpad"):
            rep = so.solve(prob, c, kind)
            assert rep.status == "converged" and rep.iterations == 0 and rep.residual_inf == 0.0
            assert rep.verified
        cache = so.factor(prob)
        y0 = rng.vector(prob.dual_dim)
        assert so.solve_minfbe(prob, cache, c, y0).iterations <= 2
        assert so.solve_nama(prob, cache, c, y0).iterations <= 2
        assert so.solve_gpad(prob, cache, c, y0).iterations <= 2


def test_oracle_sweeps_counted_exactly(gpu):
    rng = orc.Rng(1204)  # test_solvers.cpp:272-305
    po, prob = fixture(rng, mixed())
    lip = sup.dual_lipschitz_dense(orc.Factor(po))
    c, oc = cfgs(backtracking_rule="none", lambda0=0.8 / lip)
    cache = so.factor(prob)
    ofac = orc.Factor(po)
    for kind, fn in (("minfbe", so.solve_minfbe), ("nama", so.solve_nama)):
        rep = fn(prob, cache, c)
        orep = orc.solve_direct(po, ofac, oc, KIND[kind])
        assert rep.status == "converged" and rep.iterations > 0
        assert rep.stats.dual_grad_calls == rep.iterations + 1
        assert rep.stats.hessian_vec_calls == 2 * rep.iterations
        agree(rep, orep)
    rg = so.solve_gpad(prob, cache, c)
    assert rg.stats.dual_grad_calls == rg.iterations + 1 and rg.stats.hessian_vec_calls == 0
    assert len(rg.residual_trace) == rg.iterations + 1


@pytest.mark.parametrize("kind", ["minfbe", "nama"])
def test_direct_solvers_match_oracle_traces(gpu, kind):
    rng = orc.Rng(77)
    for trial in range(4):
        po, prob = fixture(rng, mixed(), stages=4, max_nodes=30)
        cache = so.factor(prob)
        ofac = orc.Factor(po)
        c, oc = cfgs(eps=1e-7)
        fn = so.solve_minfbe if kind == "minfbe" else so.solve_nama
        rep = fn(prob, cache, c)
        orep = orc.solve_direct(po, ofac, oc, KIND[kind])
        agree(rep, orep)
        n = min(len(rep.residual_trace), len(orep["residual_trace"]), 5)
        assert np.allclose(rep.residual_trace[:n], orep["residual_trace"][:n], rtol=1e-6, atol=1e-12)
        assert np.allclose(rep.fbe_trace[:n], orep["fbe_trace"][:n], rtol=1e-8, atol=1e-10)
        assert np.abs(rep.y - orep["y"]).max() <= 10 * c.eps * (1 + np.abs(orep["y"]).max())


def test_backtracking_rules(gpu):
    rng = orc.Rng(1206)  # test_solvers.cpp:307-348
    halved = 0
    for rule in ("simple", "original", "simple", "original"):
        while True:  # an instance with active constraints (y* != 0)
            po, prob = fixture(rng, mixed())
            if orc.solve(po, orc.SolverConfig(), 0)["iterations"] > 0:
                break
        lip = sup.dual_lipschitz_dense(orc.Factor(po))
        c, oc = cfgs(backtracking_rule=rule, lambda0=10.0 / lip)
        cache = so.factor(prob)
        rep = so.solve_minfbe(prob, cache, c)
        assert rep.status == "converged" and 0 < rep.lambda_final <= c.lambda0
        halved += rep.lambda_final < c.lambda0
        orep = orc.solve_direct(po, orc.Factor(po), oc, 0)
        assert rep.lambda_final == orep["lambda_final"]
        agree(rep, orep)
    assert halved >= 2
    po, prob = fixture(orc.Rng(1205), feasible_box())
    c, _ = cfgs(backtracking_rule="original")
    rep = so.solve(prob, c, "minfbe")
    assert rep.lambda_final == 0.9 / rep.lipschitz_estimate


def test_envelope_monotone_and_solvers_agree(gpu):
    rng = orc.Rng(1208)  # test_solvers.cpp:350-386
    for trial in range(3):
        po, prob = fixture(rng, mixed())
        c, _ = cfgs(eps=1e-5)
        reps = {k: so.solve(prob, c, k) for k in ("minfbe", "nama", "gpad")}
        for k in ("minfbe", "nama"):
            ft = reps[k].fbe_trace
            assert all(ft[i] <= ft[i - 1] + 1e-10 * (1 + abs(ft[i - 1])) for i in range(1, len(ft)))
        bound = 10 * c.eps * (1 + np.linalg.norm(reps["minfbe"].x.flatten()))
        for a, b in (("minfbe", "nama"), ("minfbe", "gpad"), ("nama", "gpad")):
            assert np.abs(reps[a].x.flatten() - reps[b].x.flatten()).max() <= bound


def test_parallel_linesearch_reproduces_serial(gpu):
    rng = orc.Rng(1213)  # test_solvers.cpp:468-484
    for trial in range(3):
        po, prob = fixture(rng, mixed())
        cache = so.factor(prob)
        y0 = rng.vector(prob.dual_dim, 0.3)
        c1, _ = cfgs()
        c2, _ = cfgs(nama_parallel_linesearch=True)
        rs = so.solve_nama(prob, cache, c1, y0)
        rp = so.solve_nama(prob, cache, c2, y0)
        assert rs.iterations == rp.iterations
        assert np.abs(rs.y - rp.y).max() <= 1e-12
        assert len(rs.residual_trace) == len(rp.residual_trace)


def test_preconditioning_and_warm_start(gpu):
    rng = orc.Rng(1211)  # test_solvers.cpp:388-466
    for trial in range(2):
        po, prob = fixture(rng, feasible_box())
        for kind in ("minfbe", "nama"):
            c, oc = cfgs(eps=1e-5)
            cp, ocp = cfgs(eps=1e-5, precondition=True)
            rp = so.solve(prob, c, kind)
            rs = so.solve(prob, cp, kind)
            assert rs.verified
            assert np.abs(rp.x.flatten() - rs.x.flatten()).max() < 1e-4
            agree(rs, orc.solve(po, ocp, KIND[kind]))
    po, prob = fixture(orc.Rng(1210), mixed())
    c, oc = cfgs(backtracking_rule="none", warm_start=True, warm_start_iters=5)
    rep = so.solve(prob, c, "nama")
    assert rep.status == "converged" and rep.stats.dual_grad_calls == rep.iterations + 1 + 5
    assert rep.lipschitz_calls > 0
    orep = orc.solve(po, oc, 1)
    agree(rep, orep)
    cache = so.factor(prob)
    ws, calls = so.warm_start(prob, cache, c, 0.5)
    ows, ocalls = orc.warm_start(po, orc.Factor(po), oc, 0.5)
    assert calls == ocalls == 5 and np.abs(ws - ows).max() < 1e-9 * (1 + np.abs(ows).max())


def test_verify_detects_corruption_and_config_errors(gpu):
    rng = orc.Rng(1203)  # test_solvers.cpp:248-270, 523-551
    po, prob = fixture(rng, mixed())
    c, _ = cfgs()
    rep = so.solve(prob, c, "nama")
    assert rep.verified and rep.verify_residual_inf <= c.eps * (1 + 1e-9)
    so.verify_report(prob, rep, z_override=rep.z + 10 * c.eps)
    assert not rep.verified
    for bad in (dict(lambda0=-1.0), dict(eps=0.0), dict(eps_bt=0.5), dict(beta_bt=1.0),
                dict(memory=0), dict(max_iters=0), dict(warm_start_iters=-1)):
        with pytest.raises(so.InvalidParams):
            so.solve(prob, so.SolverConfig(**bad), "minfbe")


@pytest.mark.parametrize("kind", ["minfbe", "nama"])
def test_c1_c2_small_tree_matches_oracle(gpu, kind):
    """BASELINE configs C1 (MINFBE) / C2 (NAMA): nx=10, nu=5, N=10, [2,2,2]."""
    prob = so.gen_random_instance(1, 10, 5, 10, [2, 2, 2])
    po = orc.Problem.from_flat(prob.flat())
    c, oc = cfgs()
    rep = so.solve(prob, c, kind)
    orep = orc.solve(po, oc, KIND[kind])
    agree(rep, orep)
    assert rep.verified and orep["verified"]
    assert np.abs(rep.x.flatten() - np.r_[orep["u"], orep["x"]]).max() <= 10 * c.eps * (
        1 + np.abs(orep["x"]).max())


def test_lipschitz_estimate_rounds_match_oracle(gpu):
    """estimate_dual_lipschitz (solvers.hpp:89-113): the device runs the power
    rounds in batches with a sticky stop flag; the stopping round (and so the
    sweep count) and the estimate must be the reference's."""
    rng = orc.Rng(1301)
    rounds = set()
    for trial in range(8):
        po, prob = fixture(rng, mixed() if trial % 2 else feasible_box(), stages=4, max_nodes=30)
        cache = so.factor(prob)
        est, calls = so.estimate_dual_lipschitz(cache, prob)
        oest, ocalls = orc.Factor(po).estimate_lipschitz()
        assert calls == ocalls, (trial, calls, ocalls)
        assert est == pytest.approx(oest, rel=1e-9)
        rounds.add(calls)
    assert len(rounds) > 2  # the instances stop at different rounds (batch boundaries exercised)
    # the solver's own count is the same rounds
    c, oc = cfgs()
    rep = so.solve(prob, c, "nama")
    assert rep.lipschitz_calls == calls


@pytest.mark.parametrize("rel_tol,max_rounds", [(1e-3, 100), (0.0, 7), (1e-9, 13), (1e-6, 0), (1e-6, 1)])
def test_lipschitz_optional_arguments_match_oracle(gpu, rel_tol, max_rounds):
    """estimate_dual_lipschitz(cache, prob, calls, rel_tol, max_rounds)
    (solvers.hpp:88-93): other tolerances and caps stop at the reference's
    round with the reference's estimate (max_rounds <= 0: no sweep, 1e-12)."""
    rng = orc.Rng(1302)
    for trial in range(3):
        po, prob = fixture(rng, feasible_box(), stages=4, max_nodes=30)
        est, calls = so.estimate_dual_lipschitz(so.factor(prob), prob, rel_tol, max_rounds)
        oest, ocalls = orc.Factor(po).estimate_lipschitz(rel_tol, max_rounds)
        assert calls == ocalls and calls <= max(max_rounds, 0)
        assert est == pytest.approx(oest, rel=1e-9)
