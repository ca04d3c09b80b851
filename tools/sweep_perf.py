"""Sweep timing of one shape (SHAPE=c3|c4|c5a|...); with a profiling build, per-role counters (SCN_DBG)."""
import sys, os, ctypes as C, numpy as np
os.environ.setdefault("SCN_DBG", "4")  # per-role counters on unless chosen
sys.path.insert(0, '.')
import torch
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
shape = os.environ.get("SHAPE", "c3")
shapes = {"c3": (50, 20, 20, [8, 8, 8, 2]), "c5a": (10, 5, 20, [2] * 13), "c5b": (10, 5, 20, [4] * 8),
          "c5c": (50, 20, 20, [4] * 6), "c1": (10, 5, 10, [2, 2, 2]), "c4": (50, 20, 20, [8, 8, 8, 8, 4])}
nx, nu, N_, br = shapes[shape]
p = so.gen_random_instance(1, nx, nu, N_, br)
c = so.factor(p)
dev = c.device()
info = c.dev_info()
s = C.c_void_p(); N.lib().scenopt_dev_stream(dev, C.byref(s))
stream = torch.cuda.ExternalStream(s.value)
D = p.dual_dim
ys = [torch.randn(D, dtype=torch.float64, device='cuda') for _ in range(2)]
hs = [torch.empty(D, dtype=torch.float64, device='cuda') for _ in range(2)]
P = C.POINTER(C.c_double)
def arr(ts): return (P*2)(*[C.cast(t.data_ptr(), P) for t in ts] + [None]*(2-len(ts)))
torch.cuda.synchronize()
prof = (C.c_ulonglong * 16)()
items = info['items_bw'] + info['items_fw']
names = ["prod_sempty", "prod_stage", "prod_dep", "team_full", "team_sfull", "team_compute", "team_tail", "pub_fence",
         "lc_wait_tma", "lc_wait_vec", "lc_compute", "lc_endbar", "lc_release", "-", "-", "lc_loop"]
for nrhs, aff in ((1, 0), (1, 1), (2, 0)):
    Y = arr(ys[:nrhs]); H = arr(hs[:nrhs])
    for _ in range(3):
        so.lib().scenopt_dev_sweep_async(dev, nrhs, aff, Y, None, None, H)
    N.lib().scenopt_dev_synchronize(dev)
    N.lib().scenopt_debug_sweep_profile(prof, 1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record(stream)
    for _ in range(K):
        so.lib().scenopt_dev_sweep_async(dev, nrhs, aff, Y, None, None, H)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / K
    b = info['sweep_bytes_aff' if aff else ('sweep_bytes_hom2' if nrhs == 2 else 'sweep_bytes_hom')]
    N.lib().scenopt_debug_sweep_profile(prof, 1)
    per = {names[i]: prof[i] / (items * K) for i in range(len(names)) if names[i] != "-"}
    print(f"{shape} nrhs={nrhs} aff={aff}: {ms*1e3:.1f} us, {b/ms/1e6:.0f} GB/s ({b/ms/1e6/6455.3:.1%}) | cyc/item " + " ".join(f"{k}={v:.0f}" for k, v in per.items()), flush=True)
print({k: info[k] for k in ('grid_ctas', 'slots', 'items_bw', 'items_fw', 'nodes_per_item_max', 'slot_bytes')})
