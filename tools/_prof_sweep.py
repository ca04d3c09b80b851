import sys, ctypes as C, numpy as np
sys.path.insert(0, '.')
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
if cfg == "c3":
    p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
else:
    p = so.gen_random_instance(1, 10, 5, 20, [2] * 13)
c = so.factor(p)
dev = c.device()
y = np.linspace(-1, 1, p.dual_dim)
for i in range(3):
    so.sweep(c, [y], False, want_primal=False)
print("ok", c.dev_info())
