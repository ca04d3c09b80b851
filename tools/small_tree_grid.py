"""Sweep time of small (latency-bound) trees against the grid size
(SCENOPT_GRID): C1, a C5 small case and the spring-mass benchmark tree."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
shapes = {"c1": lambda: so.gen_random_instance(1, 10, 5, 10, [2, 2, 2]),
          "c5_1k": lambda: so.gen_random_instance(1, 10, 5, 20, [2] * 6),
          "c5_12k": lambda: so.gen_random_instance(1, 10, 5, 20, [2] * 10),
          "spring": lambda: so.gen_spring_mass(5)}
P = C.POINTER(C.c_double)
for name, mk in shapes.items():
    prob = mk()
    c = so.factor(prob)
    dev = c.device()
    s = C.c_void_p(); N.lib().scenopt_dev_stream(dev, C.byref(s))
    stream = torch.cuda.ExternalStream(s.value)
    y = torch.randn(prob.dual_dim, dtype=torch.float64, device="cuda")
    h = torch.empty_like(y)
    Y = (P * 2)(C.cast(y.data_ptr(), P), None)
    H = (P * 2)(C.cast(h.data_ptr(), P), None)
    for _ in range(5):
        so.lib().scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(50):
        so.lib().scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H)
    e1.record(stream); e1.synchronize()
    info = c.dev_info()
    print(f"{name:7s} nodes {prob.num_nodes():6d} grid {info['grid_ctas']:3d} cut {info['cut_stage']:2d}: "
          f"{e0.elapsed_time(e1) / 50 * 1e3:7.1f} us/sweep", flush=True)
