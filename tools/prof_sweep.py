"""Back-to-back sweeps of one shape for ncu captures: SHAPE (c3, c5b, ...),
NRHS (1/2), AFF (0/1), K sweeps after 5 warm-up sweeps.
  ncu -k regex:sweep_kernel --launch-skip 5 --launch-count 1 ... python tools/prof_sweep.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2107_01745_b200 as so  # noqa: E402
from paper_2107_01745_b200 import _native as N  # noqa: E402

SHAPES = {"c3": (50, 20, 20, [8, 8, 8, 2]), "c5a": (10, 5, 20, [2] * 13), "c5b": (10, 5, 20, [4] * 8),
          "c5c": (50, 20, 20, [4] * 6), "c4": (50, 20, 20, [8, 8, 8, 8, 4])}
shape = os.environ.get("SHAPE", "c3")
nrhs = int(os.environ.get("NRHS", "1"))
aff = int(os.environ.get("AFF", "1"))
K = int(os.environ.get("K", "10"))
nx, nu, Nh, br = SHAPES[shape]
p = so.gen_random_instance(1, nx, nu, Nh, br)
c = so.factor(p)
dev = c.device()
info = c.dev_info()
s = C.c_void_p()
N.lib().scenopt_dev_stream(dev, C.byref(s))
stream = torch.cuda.ExternalStream(s.value)
D = p.dual_dim
ys = [torch.randn(D, dtype=torch.float64, device="cuda") for _ in range(2)]
hs = [torch.empty(D, dtype=torch.float64, device="cuda") for _ in range(2)]
P = C.POINTER(C.c_double)


def arr(ts):
    return (P * 2)(*[C.cast(t.data_ptr(), P) for t in ts] + [None] * (2 - len(ts)))


Y, H = arr(ys[:nrhs]), arr(hs[:nrhs])
for _ in range(5 + K):
    so.api.check(so.lib().scenopt_dev_sweep_async(dev, nrhs, aff, Y, None, None, H))
so.api.check(N.lib().scenopt_dev_synchronize(dev))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(K):
    so.api.check(so.lib().scenopt_dev_sweep_async(dev, nrhs, aff, Y, None, None, H))
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / K
b = info["sweep_bytes_aff" if aff else ("sweep_bytes_hom2" if nrhs == 2 else "sweep_bytes_hom")]
print(f"{shape} nrhs={nrhs} aff={aff}: {ms * 1e3:.1f} us/sweep, {b / ms / 1e6:.0f} GB/s algorithmic, "
      f"{b} B; nodes {p.num_nodes()}, grid {info['grid_ctas']}, slots {info['slots']}, "
      f"items {info['items_bw']}+{info['items_fw']}, nodes/item <= {info['nodes_per_item_max']}, "
      f"slot {info['slot_bytes']} B", flush=True)
