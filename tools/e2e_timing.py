"""Per-call time of the host-I/O dual_grad (the bench's e2e) on C3."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_01745_b200 as so
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
dev = c.device()
lib = so.lib()
D = p.dual_dim
y = torch.rand(D, dtype=torch.float64).pin_memory()
x = torch.empty(50 * p.num_nodes(), dtype=torch.float64).pin_memory()
u = torch.empty(20 * p.first_leaf, dtype=torch.float64).pin_memory()
P = C.POINTER(C.c_double)
yp, xp, up = (C.cast(t.data_ptr(), P) for t in (y, x, u))
for _ in range(5):
    so.api.check(lib.scenopt_dual_grad(dev, yp, xp, up, 1))
n = 50
t = time.perf_counter()
for _ in range(n):
    so.api.check(lib.scenopt_dual_grad(dev, yp, xp, up, 1))
dt = (time.perf_counter() - t) / n
print(f"host-I/O dual_grad: {dt*1e6:.1f} us per call ({1/dt:.0f}/s)")
