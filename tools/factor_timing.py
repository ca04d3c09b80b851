"""Host factor + pack vs device factor (K9) for the bench trees."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
for br in ([8, 8, 8, 2], [8, 8, 8, 8, 4]):
    p = so.gen_random_instance(1, 50, 20, 20, br)
    t0 = time.time(); c = so.factor(p); t1 = time.time(); c.device(); torch.cuda.synchronize(); t2 = time.time()
    del c
    t3 = time.time(); d = so.factor_device(p); torch.cuda.synchronize(); t4 = time.time()
    # device factor kernels alone: re-run on the existing handle
    lib = N.lib()
    t5 = time.time(); so.api.check(lib.scenopt_dev_refactor_device(d.device())); t6 = time.time()
    # MPC-style update: new linear terms / root state, affine terms recomputed on the device
    f2 = dict(p.flat())
    f2["root_state"] = f2["root_state"] + 0.01
    f2["q"] = f2["q"] * 1.01
    p2 = so.ProblemInstance.from_flat(f2)
    so.refactor_affine(d, p2)
    t7 = time.time(); so.refactor_affine(d, p2); t8 = time.time()
    print(br, p.num_nodes(), f"host factor {t1-t0:.2f}s + pack/upload {t2-t1:.2f}s | device-factor handle {t4-t3:.2f}s"
          f" (factor kernels {1e3*(t6-t5):.1f} ms) | device refactor_affine {1e3*(t8-t7):.1f} ms", flush=True)
    del d
