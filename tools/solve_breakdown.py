"""C3 MINFBE / NAMA with SCN_SOLVE_TIMING=2: per-op GPU time between stream marks (stderr)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so  # noqa: E402

prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
cache = so.factor(prob)
L, _ = so.estimate_dual_lipschitz(cache, prob)
for kind in ("minfbe", "nama"):
    cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
    so.api._solve_direct(kind, prob, cache, cfg)
    for _ in range(2):
        rep = so.api._solve_direct(kind, prob, cache, cfg)
        print(f"{kind}: {rep.wall_ms:.3f} ms, {rep.iterations} iterations", file=sys.stderr, flush=True)
