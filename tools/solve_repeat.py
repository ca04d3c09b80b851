"""Warm MINFBE / NAMA solves of C3 repeated (median wall_ms), no diagnostics."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
L, _ = so.estimate_dual_lipschitz(c, p)
for kind in ("minfbe", "nama"):
    cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
    so.api._solve_direct(kind, p, c, cfg)
    ws = [so.api._solve_direct(kind, p, c, cfg) for _ in range(7)]
    print(kind, "iters", ws[0].iterations, "wall_ms median %.3f min %.3f" % (
        statistics.median(r.wall_ms for r in ws), min(r.wall_ms for r in ws)))
