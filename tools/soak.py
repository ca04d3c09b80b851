"""Soak test: repeated C3 MINFBE / NAMA solves and back-to-back sweeps on one
handle; every repetition must reproduce the first bit for bit (flags, epochs,
speculation and the scalar publish protocol under sustained load).
python tools/soak.py [solves] [sweeps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_01745_b200 as so
nsolve = int(sys.argv[1]) if len(sys.argv) > 1 else 40
nsweep = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
cache = so.factor(prob)
L, _ = so.estimate_dual_lipschitz(cache, prob)
t0 = time.time()
ref = {}
for i in range(nsolve):
    for kind in ("minfbe", "nama"):
        r = so.api._solve_direct(kind, prob, cache, so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=kind == "nama"))
        key = (r.iterations, r.y.tobytes(), r.x.x.tobytes(), r.z.tobytes())
        if kind not in ref:
            ref[kind] = key
        assert key == ref[kind], (kind, i)
y = np.random.default_rng(1).uniform(-1, 1, prob.dual_dim)
first = so.dual_grad(cache, prob, y)
for i in range(nsweep):
    pts, hs = so.sweep(cache, [y], True)
    if i % 97 == 0:
        assert np.array_equal(pts[0].x, first.x) and np.array_equal(pts[0].u, first.u), i
print(f"soak ok: {2 * nsolve} solves and {nsweep} sweeps bitwise stable in {time.time() - t0:.1f} s")
