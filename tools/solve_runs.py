"""Per-run wall_ms of repeated warm C3 solves (distribution diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
L, _ = so.estimate_dual_lipschitz(c, p)
kind = sys.argv[1] if len(sys.argv) > 1 else "minfbe"
gap = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
so.api._solve_direct(kind, p, c, cfg)
out = []
for _ in range(10):
    if gap:
        time.sleep(gap)
    out.append(so.api._solve_direct(kind, p, c, cfg).wall_ms)
print(kind, "gap", gap, " ".join("%.2f" % w for w in out))
