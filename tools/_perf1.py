import sys, time, ctypes as C, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
t0 = time.time()
p = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
t1 = time.time()
c = so.factor(p)
t2 = time.time()
dev = c.device()
t3 = time.time()
info = c.dev_info()
print(f"gen {t1-t0:.1f}s factor {t2-t1:.1f}s upload {t3-t2:.1f}s", info, flush=True)
s = C.c_void_p()
N.lib().scenopt_dev_stream(dev, C.byref(s))
stream = torch.cuda.ExternalStream(s.value)
D = p.dual_dim
ys = [torch.randn(D, dtype=torch.float64, device='cuda') for _ in range(2)]
hs = [torch.empty(D, dtype=torch.float64, device='cuda') for _ in range(2)]
P = C.POINTER(C.c_double)
def arr(ts): return (P*2)(*[C.cast(t.data_ptr(), P) for t in ts] + [None]*(2-len(ts)))
torch.cuda.synchronize()
for nrhs, aff in ((1, 1), (1, 0), (2, 0)):
    Y = arr(ys[:nrhs]); H = arr(hs[:nrhs])
    for _ in range(5):
        so.lib().scenopt_dev_sweep_async(dev, nrhs, aff, Y, None, None, H)
    N.lib().scenopt_dev_synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    K = 50
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(K):
            so.lib().scenopt_dev_sweep_async(dev, nrhs, aff, Y, None, None, H)
        e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / K
    b = info['sweep_bytes_aff' if aff else ('sweep_bytes_hom2' if nrhs == 2 else 'sweep_bytes_hom')]
    mats = info['matrix_bytes_bw'] + info['matrix_bytes_fw']
    print(f"nrhs={nrhs} affine={aff}: {ms*1e3:.1f} us/sweep, algo {b/ms/1e6:.0f} GB/s ({b/ms/1e6/6455.3:.1%}), matrices-only {mats/ms/1e6:.0f} GB/s", flush=True)
