import sys, numpy as np, faulthandler
faulthandler.enable()
sys.path.insert(0, '.')
import paper_2107_01745_b200 as so
from oracle import oracle as orc
print("devices", so.device_count(), flush=True)
p = so.gen_random_instance(1, 10, 5, 10, [2,2,2])
c = so.factor(p)
print("factor ok", flush=True)
print(c.dev_info(), flush=True)
y = np.linspace(-1, 1, p.dual_dim)
pt = so.dual_grad(c, p, y)
print("sweep ok", flush=True)
o = orc.Factor(orc.Problem.from_flat(p.flat()))
ox, ou = o.dual_grad(y)
print("max diff x", np.abs(pt.x.ravel(order='F') - ox).max(), "u", np.abs(pt.u.ravel(order='F') - ou).max(), flush=True)
