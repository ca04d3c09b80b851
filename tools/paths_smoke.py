"""Small workload touching every device path (sweeps of 1 / 2 RHS, each solver, the device
factor, power iteration, the experiment harness) on tiny trees: a quick smoke run of the
whole library."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_01745_b200 as so
prob = so.gen_random_instance(3, 6, 3, 5, [3, 2, 2])
cache = so.factor(prob)
rng = np.random.default_rng(0)
y, r = rng.uniform(-1, 1, prob.dual_dim), rng.uniform(-1, 1, prob.dual_dim)
pts, hs = so.sweep(cache, [y, r], True)
pts, hs = so.sweep(cache, [y], False)
for kind in ("minfbe", "nama", "gpad"):
    rep = so.solve(prob, so.SolverConfig(eps=1e-5), kind)
    print(kind, rep.status, rep.iterations)
dc = so.factor_device(prob)
so.dual_grad(dc, prob, y)
est, calls = so.estimate_dual_lipschitz(cache, prob)
print("lipschitz", est, calls)
rep = so.run_experiment([("a", prob), ("b", so.gen_spring_mass(2, so.SpringMassParams(horizon=3)))],
                        ["minfbe", "pnama"], include_timing=False)
print(rep.csv())
