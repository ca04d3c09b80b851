import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2107_01745_b200 as so
prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
so.solve(prob, so.SolverConfig(nama_parallel_linesearch=True), "nama")  # warm-up (CUDA context, pools)
for rep_i in range(2):
    t = time.time(); c = so.factor(prob); t1 = time.time(); c.device(); t2 = time.time()
    print(f"host factor {t1-t:.3f} s, handle (pack+upload) {t2-t1:.3f} s")
    t = time.time(); cd = so.factor_device(prob); cd.device(); t3 = time.time()
    print(f"device-factor handle {t3-t:.3f} s")
    t = time.time(); r = so.solve(prob, so.SolverConfig(nama_parallel_linesearch=True), "nama"); t4 = time.time()
    print(f"solve() wall_ms {r.wall_ms:.1f}, call {t4-t:.3f} s, iterations {r.iterations}")
    t = time.time(); r = so.solve(prob, so.SolverConfig(nama_parallel_linesearch=True), "nama", shared_cache=c); t5 = time.time()
    print(f"solve(shared host cache) wall_ms {r.wall_ms:.1f}")
    t = time.time(); r = so.solve(prob, so.SolverConfig(nama_parallel_linesearch=True), "nama", shared_cache=cd); t5 = time.time()
    print(f"solve(shared device cache) wall_ms {r.wall_ms:.1f}")
