"""Randomised parity sweep of the device path against the CPU oracle (test
infrastructure): random trees (depth, branching, node budget), dimensions,
nonsmooth kinds and affine terms; dual_grad / hessian_vec / 2-RHS sweeps to
1e-9 relative, and solves of every kind to +-1 iteration. Prints the worst
gaps and every failure.  python tools/fuzz_parity.py [trials] [seed]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = orc.Rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
max_nodes = int(sys.argv[3]) if len(sys.argv) > 3 else 400  # >= ~600 per stage exercises the subtree cut
solves = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
device_factor = len(sys.argv) > 5 and sys.argv[5] == "dev"  # factor on the GPU (K9 + flattened-top maps)
cuts = {}
worst = {"dual_grad": 0.0, "hessian_vec": 0.0, "two_rhs": 0.0}
fails, iters_off = [], 0
t0 = time.time()
for t in range(trials):
    stages = rng.integer(1, 6)
    nx, nu = rng.integer(1, 14), rng.integer(1, 8)
    opt = orc.InstanceOptions(with_box=True, with_l1=rng.integer(0, 1) == 1, with_none=rng.integer(0, 1) == 1,
                              affine=rng.integer(0, 3) > 0, feasible_boxes=True,
                              stage_rows_lo=rng.integer(0, 1), stage_rows_hi=rng.integer(1, 4))
    if max_nodes > 0:
        po = rng.random_instance(stages, rng.integer(2, max_nodes), nx, nu, opt)
        prob = so.ProblemInstance.from_flat(po.flat())
    else:  # full-branching trees with stages of 500-5000 nodes: the subtree cut, flat top, owners
        depth = rng.integer(2, 5)
        br = [rng.integer(3, 9) for _ in range(depth)]
        br[0] = rng.integer(3, 40)  # wide first stages put the cut at stage 2 or 3
        horizon = depth + rng.integer(0, 4)
        prob = so.gen_random_instance(rng.integer(1, 10 ** 6), nx, nu, horizon, br)
        po = orc.Problem.from_flat(prob.flat())
    ofac = orc.Factor(po)
    cache = so.factor_device(prob) if device_factor else so.factor(prob)
    info = cache.dev_info()
    key = (info["cut_stage"], info["flat_top"])
    cuts[key] = cuts.get(key, 0) + 1
    y = rng.vector(prob.dual_dim, 1.0)
    r = rng.vector(prob.dual_dim, 1.0)
    try:
        pt = so.dual_grad(cache, prob, y)
        ox, ou = ofac.dual_grad(y)
        g1 = sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F"))
        ph = so.hessian_vec(cache, prob, r)
        hx, hu = ofac.hessian_vec(r)
        g2 = sup.rel_gap(hx, hu, ph.x.ravel(order="F"), ph.u.ravel(order="F"))
        pts, _ = so.sweep(cache, [y, r], False)
        yx, yu = ofac.hessian_vec(y)
        g3 = max(sup.rel_gap(yx, yu, pts[0].x.ravel(order="F"), pts[0].u.ravel(order="F")),
                 sup.rel_gap(hx, hu, pts[1].x.ravel(order="F"), pts[1].u.ravel(order="F")))
        for k, g in (("dual_grad", g1), ("hessian_vec", g2), ("two_rhs", g3)):
            worst[k] = max(worst[k], g)
            if not g < 1e-9:
                fails.append((t, k, g, stages, nx, nu, prob.num_nodes()))
        if solves and t % 3 == 0:
            for kind, code in (("minfbe", 0), ("nama", 1), ("gpad", 2)):
                rep = so.solve(prob, so.SolverConfig(eps=1e-5), kind)
                orep = orc.solve(po, orc.SolverConfig(eps=1e-5), code)
                d = abs(rep.iterations - orep["iterations"])
                if d > 1 or (rep.status == "converged") != (orep["status"] == 0):
                    # the oracle against itself: the same solve from y0 perturbed by 1e-14
                    sens = None
                    if code < 2:
                        oc = orc.SolverConfig(eps=1e-5, lambda0=0.9 / orep["lipschitz_estimate"])
                        a0 = orc.solve_direct(po, ofac, oc, code)
                        a1 = orc.solve_direct(po, ofac, oc, code, y0=1e-14 * rng.vector(prob.dual_dim))
                        sens = (a0["iterations"], a1["iterations"])
                    fails.append((t, kind, rep.iterations, orep["iterations"], prob.num_nodes(), "oracle y0 / y0+1e-14:", sens))
                iters_off += d > 0
    except Exception as e:  # noqa: BLE001 - report and continue
        fails.append((t, "exception", repr(e)[:200], stages, nx, nu))
print(f"{trials} trials in {time.time() - t0:.0f} s; worst rel gaps {worst}; solves off by one: {iters_off}")
print("(cut stage, flat top) -> trees:", cuts)
print("failures:", len(fails))
for f in fails[:20]:
    print("  ", f)
