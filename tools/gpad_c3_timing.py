import os, sys, time
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.getcwd())
import paper_2107_01745_b200 as so
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
L, _ = so.estimate_dual_lipschitz(c, p)
cfg = so.SolverConfig(lambda0=0.95 / L)
so.api._solve_direct("gpad", p, c, cfg)
w = [so.api._solve_direct("gpad", p, c, cfg) for _ in range(3)]
print("gpad iters", w[0].iterations, "wall_ms", [round(r.wall_ms, 2) for r in w], "sweeps", w[0].stats.dual_grad_calls)
