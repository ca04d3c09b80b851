"""Soak test of the sharded solver with W emulated ranks on one GPU (one host
thread per rank, exchanges through host memory): repeated MINFBE / NAMA
solves on the same handles must reproduce the first reports bit for bit on
every rank. python tools/soak_sharded.py [world] [repetitions]"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_01745_b200 as so
world = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
group = so.ShardGroup(world)
caches = []
for r in range(world):
    c = so.factor(prob)
    c.shard_emulated(r, group, 0, 1)
    caches.append(c)
ref = {}
t0 = time.time()
for it in range(reps_n):
    for kind in ("minfbe", "nama"):
        cfg = so.SolverConfig(nama_parallel_linesearch=kind == "nama")
        out, errs = [None] * world, []

        def run(r):
            try:
                out[r] = so.api._solve_direct(kind, prob, caches[r], cfg)
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        if errs:
            raise errs[0]
        for r in range(world):
            key = (out[r].iterations, out[r].y.tobytes(), out[r].x.x.tobytes())
            ref.setdefault(kind, key)
            assert key == ref[kind], (kind, it, r)
print(f"sharded soak ok: world {world}, {2 * reps_n} solves per rank bitwise stable in {time.time() - t0:.1f} s")
