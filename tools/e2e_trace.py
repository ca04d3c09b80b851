"""Where the host-buffer dual_grad's kernel time goes (profiling build):
per-item retirement stamps (%globaltimer) of one pinned-buffer call on C3,
split into backward and forward pass, against a device-resident sweep.
  SCENOPT_LIBRARY=.../libscenopt_b200_prof.so python tools/e2e_trace.py"""
import ctypes as C, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
dev = c.device()
lib = N.lib()
n = lib.scenopt_debug_items(dev, None, 0)
it = np.zeros((n, 7), np.int32)
lib.scenopt_debug_items(dev, it.ctypes.data_as(C.POINTER(C.c_int32)), n)
tr = torch.zeros(12 * n, dtype=torch.int64, device="cuda")
so.api.check(lib.scenopt_debug_sweep_trace(C.c_void_p(tr.data_ptr())))
D = p.dual_dim
P = C.POINTER(C.c_double)
yh = torch.rand(D, dtype=torch.float64).pin_memory()
xh = torch.empty(50 * p.num_nodes(), dtype=torch.float64).pin_memory()
uh = torch.empty(20 * p.first_leaf, dtype=torch.float64).pin_memory()
yp, xp, up = (C.cast(t.data_ptr(), P) for t in (yh, xh, uh))
yd = yh.cuda()
hd = torch.empty_like(yd)
Y = (P * 2)(C.cast(yd.data_ptr(), P), None)
H = (P * 2)(C.cast(hd.data_ptr(), P), None)


def split(label):
    t = tr.cpu().numpy().reshape(n, 12).astype(np.float64) / 1e3
    t0 = t[:, 8].min()  # first producer start
    rel = t[:, 11] - t0  # retirement
    bw, fw = it[:, 2] == 0, it[:, 2] == 1
    print(f"{label}: backward done {rel[bw].max():7.1f} us, forward {rel[fw].min():7.1f}..{rel[fw].max():7.1f} us;"
          f" forward items retired by 25/50/75/100 %: "
          + " ".join(f"{np.percentile(rel[fw], q):.0f}" for q in (25, 50, 75, 100)))


for rep in range(3):
    so.api.check(lib.scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H))
    so.api.check(lib.scenopt_dev_synchronize(dev))
split("device-resident affine sweep")
for rep in range(3):
    so.api.check(lib.scenopt_dual_grad(dev, yp, xp, up, 1))
split("host-buffer dual_grad (zero-copy x/u)")
