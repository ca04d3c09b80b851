"""Per-stage retirement timeline of one sweep (profiling build):
SCENOPT_LIBRARY=.../libscenopt_b200_prof.so python tools/timeline.py [c3|c4]"""
import ctypes as C, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
shapes = {"c3": (50, 20, 20, [8, 8, 8, 2]), "c4": (50, 20, 20, [8, 8, 8, 8, 4])}
nx, nu, H, br = shapes[sys.argv[1] if len(sys.argv) > 1 else "c3"]
p = so.gen_random_instance(1, nx, nu, H, br)
c = so.factor(p)
dev = c.device()
lib = N.lib()
n = lib.scenopt_debug_items(dev, None, 0)
it = np.zeros((n, 7), np.int32)
lib.scenopt_debug_items(dev, it.ctypes.data_as(C.POINTER(C.c_int32)), n)
tl = torch.zeros(n, dtype=torch.int64, device="cuda")
so.api.check(lib.scenopt_debug_sweep_timeline(C.c_void_p(tl.data_ptr())))
stage = np.searchsorted(p.flat()["stage_offsets"], it[:, 3], side="right") - 1
y = torch.randn(p.dual_dim, dtype=torch.float64, device="cuda")
h = torch.empty_like(y)
P = C.POINTER(C.c_double)
Y = (P * 2)(C.cast(y.data_ptr(), P), None)
H_ = (P * 2)(C.cast(h.data_ptr(), P), None)
for rep in range(4):
    tl.zero_()
    torch.cuda.synchronize()
    so.api.check(lib.scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H_))
    so.api.check(lib.scenopt_dev_synchronize(dev))
t = tl.cpu().numpy().astype(np.float64)
t0 = t.min()
t = (t - t0) / 1e3
print(f"items {n}, first retirement at 0, last at {t.max():.1f} us")
for ps, name in ((0, "bw"), (1, "fw")):
    order = range(H, -1, -1) if ps == 0 else range(0, H + 1)
    for s in order:
        m = (it[:, 2] == ps) & (stage == s)
        if m.any():
            print(f"{name} stage {s:2d}: {m.sum():5d} items  first {t[m].min():8.1f}  last {t[m].max():8.1f} us"
                  f"  local {np.mean(it[m, 5] >= 0):.2f} publish {np.mean(it[m, 6]):.2f}")
