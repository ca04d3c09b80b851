"""Per-item consumer-team step timing of one sweep (profiling build):
SCENOPT_LIBRARY=.../libscenopt_b200_prof.so python tools/trace.py [c3|c4]
Stamps: 0 loop top, 1 matrices (TMA) ready, 2 staged vectors ready,
3 phase A done, 4 phase A barrier, 5 phase B done, 6 end barrier, 7 done."""
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
tr = torch.zeros(8 * n, dtype=torch.int64, device="cuda")
so.api.check(lib.scenopt_debug_sweep_trace(C.c_void_p(tr.data_ptr())))
y = torch.randn(p.dual_dim, dtype=torch.float64, device="cuda")
h = torch.empty_like(y)
P = C.POINTER(C.c_double)
Y = (P * 2)(C.cast(y.data_ptr(), P), None)
H_ = (P * 2)(C.cast(h.data_ptr(), P), None)
for rep in range(3):
    so.api.check(lib.scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H_))
so.api.check(lib.scenopt_dev_synchronize(dev))
t = tr.cpu().numpy().reshape(n, 8).astype(np.float64)
names = ["wait_tma", "wait_stage", "phaseA", "syncA", "phaseB", "sync_end", "tail"]
for ps, nm in ((0, "bw"), (1, "fw")):
    m = it[:, 2] == ps
    d = np.diff(t[m], axis=1)
    print(nm, {names[i]: round(float(np.median(d[:, i])), 0) for i in range(7)},
          "total", round(float(np.median(t[m, 7] - t[m, 0])), 0),
          "loop-to-loop", round(float(np.median(np.diff(t[m, 0]))), 0))
