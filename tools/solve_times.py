"""Median wall_ms of 5 warm C3 MINFBE and NAMA (p-NAMA) solves (one line)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so  # noqa: E402

p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
L, _ = so.estimate_dual_lipschitz(c, p)
out = []
for kind in ("minfbe", "nama"):
    cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
    so.api._solve_direct(kind, p, c, cfg)
    w = []
    for _ in range(5):
        r = so.api._solve_direct(kind, p, c, cfg)
        w.append(r.wall_ms)
    out.append(f"{kind} {statistics.median(w):.3f} ms ({r.iterations} it)")
print("solves: " + ", ".join(out))
