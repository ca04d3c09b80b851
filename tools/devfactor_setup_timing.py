import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2107_01745_b200 as so
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
for i in range(3):
    t = time.time(); c = so.factor_device(p); c.device(); print(f"device-factor handle {time.time()-t:.3f} s", file=sys.stderr, flush=True)
    del c
