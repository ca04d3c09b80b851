"""Per-CTA balance of one C3 sweep (profiling build): when each CTA finishes
its local backward / whole forward, against its local chain count and item
count. SCENOPT_LIBRARY=.../libscenopt_b200_prof.so python tools/cta_balance.py"""
import ctypes as C, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
c = so.factor(p)
dev = c.device()
info = c.dev_info()
cut = info["cut_stage"]
lib = N.lib()
n = lib.scenopt_debug_items(dev, None, 0)
it = np.zeros((n, 7), np.int32)
lib.scenopt_debug_items(dev, it.ctypes.data_as(C.POINTER(C.c_int32)), n)
tl = torch.zeros(n, dtype=torch.int64, device="cuda")
so.api.check(lib.scenopt_debug_sweep_timeline(C.c_void_p(tl.data_ptr())))
so_ = p.flat()["stage_offsets"]
stage = np.searchsorted(so_, it[:, 3], side="right") - 1
y = torch.randn(p.dual_dim, dtype=torch.float64, device="cuda")
h = torch.empty_like(y)
P = C.POINTER(C.c_double)
Y = (P * 2)(C.cast(y.data_ptr(), P), None)
H_ = (P * 2)(C.cast(h.data_ptr(), P), None)
ends = []
for rep in range(5):
    tl.zero_()
    torch.cuda.synchronize()
    so.api.check(lib.scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H_))
    so.api.check(lib.scenopt_dev_synchronize(dev))
    t = tl.cpu().numpy().astype(np.float64)
    t = (t - t.min()) / 1e3
    G = it[:, 1].max() + 1
    bw_local_end = np.zeros(G); fw_end = np.zeros(G); chains = np.zeros(G, int); top_items = np.zeros(G, int)
    nodes = np.zeros(G, int)
    for g in range(G):
        m = it[:, 1] == g
        bl = m & (it[:, 2] == 0) & (stage >= cut)
        bw_local_end[g] = t[bl].max() if bl.any() else 0
        fw_end[g] = t[m & (it[:, 2] == 1)].max()
        chains[g] = it[bl & (stage == cut), 4].sum()
        top_items[g] = (m & (stage < cut)).sum()
        nodes[g] = it[m, 4].sum()
    ends.append((bw_local_end, fw_end))
bw = np.median([e[0] for e in ends], axis=0)
fw = np.median([e[1] for e in ends], axis=0)
print(f"cut {cut}, grid {G}; median over 5 sweeps (profiling build, ~1.37x slower)")
for k in sorted(set(chains)):
    m = chains == k
    print(f"  CTAs with {k} chains: {m.sum():3d}  bw-local end median {np.median(bw[m]):6.1f} "
          f"[{bw[m].min():6.1f}, {bw[m].max():6.1f}]  fw end median {np.median(fw[m]):6.1f} "
          f"[{fw[m].min():6.1f}, {fw[m].max():6.1f}]  top items {top_items[m].mean():.2f}")
print("  slowest 10 CTAs by fw end:", np.argsort(fw)[-10:], np.round(np.sort(fw)[-10:], 1))
print("  fastest 10 CTAs by fw end:", np.argsort(fw)[:10], np.round(np.sort(fw)[:10], 1))
print("  bw-local end by CTA index (8 groups of 18):", [round(float(np.median(bw[i:i + 18])), 1) for i in range(0, G, 18)])
