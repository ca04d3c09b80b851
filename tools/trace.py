"""Per-item step timing of one sweep (profiling build, %globaltimer ns):
SCENOPT_LIBRARY=.../libscenopt_b200_prof.so python tools/trace.py [c3|c4]
Team stamps: 0 loop top, 1 matrices ready, 2 vectors ready, 3 phase A done,
4 phase A barrier, 5 phase B done, 6 end barrier, 7 done-arrive; producer:
8 start, 9 dependencies seen, 10 staged; publisher: 11 released."""
import ctypes as C, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
shapes = {"c3": (50, 20, 20, [8, 8, 8, 2]), "c4": (50, 20, 20, [8, 8, 8, 8, 4]), "c1": (10, 5, 10, [2, 2, 2]), "c5_1k": (10, 5, 20, [2] * 6),
          "c5b": (10, 5, 20, [4] * 8)}
nx, nu, H, br = shapes[sys.argv[1] if len(sys.argv) > 1 else "c3"]
p = so.gen_random_instance(1, nx, nu, H, br)
c = so.factor(p)
dev = c.device()
lib = N.lib()
n = lib.scenopt_debug_items(dev, None, 0)
it = np.zeros((n, 7), np.int32)
lib.scenopt_debug_items(dev, it.ctypes.data_as(C.POINTER(C.c_int32)), n)
tr = torch.zeros(12 * n, dtype=torch.int64, device="cuda")
so.api.check(lib.scenopt_debug_sweep_trace(C.c_void_p(tr.data_ptr())))
y = torch.randn(p.dual_dim, dtype=torch.float64, device="cuda")
h = torch.empty_like(y)
P = C.POINTER(C.c_double)
Y = (P * 2)(C.cast(y.data_ptr(), P), None)
H_ = (P * 2)(C.cast(h.data_ptr(), P), None)
for rep in range(3):
    so.api.check(lib.scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H_))
so.api.check(lib.scenopt_dev_synchronize(dev))
t = tr.cpu().numpy().reshape(n, 12).astype(np.float64) / 1e3  # us
t -= t[:, 0].min()
stage = np.searchsorted(p.flat()["stage_offsets"], it[:, 3], side="right") - 1
cols = ["top", "tma", "vec", "A", "Async", "B", "end", "done", "p_start", "p_deps", "p_staged", "released"]
print("steady-state medians (us):")
for ps, nm in ((0, "bw"), (1, "fw")):
    m = (it[:, 2] == ps) & (stage >= max(6, len(br) + 2)) & (stage <= H - 2)
    d = np.diff(t[m][:, :8], axis=1)
    print(" ", nm, {cols[i + 1]: round(float(np.median(d[:, i])), 2) for i in range(7)})
print("top levels: stage, last release, per item medians: deps->staged, staged->team vec ready, vec->done, done->released")
for ps in (0, 1):
    order = range(5, -1, -1) if ps == 0 else range(0, 6)
    for s in order:
        m = (it[:, 2] == ps) & (stage == s)
        if not m.any():
            continue
        x = t[m]
        print(f"  {'bw' if ps == 0 else 'fw'} {s}: n={m.sum():4d} first_deps {x[:, 9].min():7.2f} last_released {x[:, 11].max():7.2f}"
              f" | stage {np.median(x[:, 10] - x[:, 9]):5.2f} team_wakeup {np.median(x[:, 2] - x[:, 10]):5.2f}"
              f" compute {np.median(x[:, 7] - x[:, 2]):5.2f} publish {np.median(x[:, 11] - x[:, 7]):5.2f}"
              f" | A {np.median(x[:, 3] - x[:, 2]):4.2f} sync {np.median(x[:, 4] - x[:, 3]):4.2f}"
              f" B {np.median(x[:, 5] - x[:, 4]):4.2f} end {np.median(x[:, 6] - x[:, 5]):4.2f}"
              f" done {np.median(x[:, 7] - x[:, 6]):4.2f}")
