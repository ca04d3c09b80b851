"""estimate_dual_lipschitz at C3: wall time (median of 5) and rounds."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
so.estimate_dual_lipschitz(c, p)
ts = []
for _ in range(5):
    t = time.perf_counter()
    est, calls = so.estimate_dual_lipschitz(c, p)
    ts.append((time.perf_counter() - t) * 1e3)
print("lipschitz %.6g rounds %d  ms median %.3f min %.3f" % (est, calls, statistics.median(ts), min(ts)))
