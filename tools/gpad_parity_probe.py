import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2107_01745_b200 as so
from oracle import oracle as orc
prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
cache = so.factor(prob); cache.device()
L, _ = so.estimate_dual_lipschitz(cache, prob)
po = orc.Problem.from_flat(prob.flat()); of = orc.Factor(po)
cfg = dict(lambda0=0.95 / L)
rep = so.api._solve_direct("gpad", prob, cache, so.SolverConfig(**cfg))
rep = so.api._solve_direct("gpad", prob, cache, so.SolverConfig(**cfg))
t = time.time()
orep = orc.solve_direct(po, of, orc.SolverConfig(**cfg), 2)
print("GPU", rep.iterations, rep.status, f"{rep.wall_ms:.2f} ms", rep.stats.dual_grad_calls, "| CPU", orep["iterations"], orep["status"], f"{time.time()-t:.1f} s", orep["dual_grad_calls"])
yo = orep["y"]; print("y gap", np.abs(rep.y - yo).max(), "bound", 10 * 5e-4 * (1 + np.abs(yo).max()))
k = min(len(rep.residual_trace), len(orep["residual_trace"])); rt = np.array(rep.residual_trace[:k]); ort = np.array(orep["residual_trace"][:k])
print("trace max rel", np.max(np.abs(rt - ort) / (np.abs(ort) + 5e-4)))
