import sys, os, ctypes as C, numpy as np, time
sys.path.insert(0, '.')
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p); dev = c.device(); info = c.dev_info()
y = np.linspace(-1, 1, p.dual_dim)
prof = (C.c_ulonglong * 16)()
so.sweep(c, [y], False, want_primal=False)
N.lib().scenopt_debug_sweep_profile(prof, 1)
t0 = time.time(); so.sweep(c, [y], False, want_primal=False); dt = time.time() - t0
N.lib().scenopt_debug_sweep_profile(prof, 1)
items = info['items_bw'] + info['items_fw']
cyc = dt * 1.965e9 * info['grid_ctas']
names = ["prod_empty", "prod_stage", "prod_dep", "cons_full", "pub_done", "pub_fence", "cons_tail", "bwA", "bwSync", "bwB", "fwA", "fwSync", "fwB", "endSync"]
per_item = {names[i]: prof[i] / items * info['grid_ctas'] / info['grid_ctas'] for i in range(14)}
print(f"grid={info['grid_ctas']} wall {dt*1e3:.1f} ms, {dt/items*1e6*info['grid_ctas']:.2f} us/item/CTA | cycles per item: " + " ".join(f"{k}={v:.0f}" for k, v in per_item.items()))
