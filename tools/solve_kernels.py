"""One warm MINFBE / NAMA solve of C3 (for an ncu launch list of its kernels)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
kind = sys.argv[1] if len(sys.argv) > 1 else "minfbe"
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
L, _ = so.estimate_dual_lipschitz(c, p)
cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
so.api._solve_direct(kind, p, c, cfg)
t = time.perf_counter()
r = so.api._solve_direct(kind, p, c, cfg)
print(kind, "wall_ms", r.wall_ms, "iters", r.iterations, "host", (time.perf_counter() - t) * 1e3)
