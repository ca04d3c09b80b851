"""BASELINE config 5: dual-gradient oracle microbench over node counts
(SURVEY.md §8d C5): affine sweeps back to back on device-resident inputs,
CUDA events on the handle's stream, algorithmic bytes (§8d formula) / time
vs the measured HBM peak. Trees whose packed matrices fit in L2 are flagged.

  python tools/microbench_c5.py [--max-nodes N] [--device-factor] [--out profiles/c5_microbench_r02.json]
"""
import argparse, ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N

SHAPES = [  # (nx, nu, N, branching) -- SURVEY §8d C5
    (10, 5, 20, [2] * 6), (10, 5, 20, [2] * 10), (10, 5, 20, [2] * 13), (10, 5, 20, [4] * 8),
    (10, 5, 20, [4] * 9), (10, 5, 20, [4] * 10),
    (50, 20, 20, [4] * 3), (50, 20, 20, [4] * 5), (50, 20, 20, [4] * 6), (50, 20, 20, [8, 8, 8, 2]),
    (50, 20, 20, [4] * 7), (50, 20, 20, [8, 8, 8, 8, 4]),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-nodes", type=int, default=4_000_000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="comma-separated indices into SHAPES")
    ap.add_argument("--device-factor", action="store_true",
                    help="factor on the device (no host factor: the 11.9M-node point needs ~110 GB of host RAM "
                         "with it)")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6455.3) \
        if os.path.exists("MEASURED_PEAKS.json") else 6455.3
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    rows = []
    sel = [SHAPES[int(i)] for i in a.only.split(",")] if a.only else SHAPES
    for nx, nu, H, br in sel:
        n = 1
        w = 1
        for t in range(H):
            w *= br[t] if t < len(br) else 1
            n += w
        if n > a.max_nodes:
            continue
        t0 = time.time()
        p = so.gen_random_instance(1, nx, nu, H, br)
        c = so.factor_device(p) if a.device_factor else so.factor(p)
        dev = c.device()
        info = c.dev_info()
        setup = time.time() - t0
        s = C.c_void_p()
        N.lib().scenopt_dev_stream(dev, C.byref(s))
        st = torch.cuda.ExternalStream(s.value)
        y = torch.rand(p.dual_dim, dtype=torch.float64, device="cuda")
        h = torch.empty_like(y)
        P = C.POINTER(C.c_double)
        Y = (P * 2)(C.cast(y.data_ptr(), P), None)
        H_ = (P * 2)(C.cast(h.data_ptr(), P), None)
        for _ in range(3):
            so.api.check(N.lib().scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H_))
        so.api.check(N.lib().scenopt_dev_synchronize(dev))
        bytes_ = info["sweep_bytes_aff"]
        k = max(5, min(200, int(2e9 / max(bytes_, 1))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(k):
            so.api.check(N.lib().scenopt_dev_sweep_async(dev, 1, 1, Y, None, None, H_))
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / k
        gbs = bytes_ / (ms * 1e-3) / 1e9
        packed = info["matrix_bytes_bw"] + info["matrix_bytes_fw"]
        row = dict(nx=nx, nu=nu, horizon=H, branching=br, nodes=p.num_nodes(), sweeps=k, us_per_sweep=ms * 1e3,
                   algorithmic_bytes=bytes_, gbs=gbs, frac_of_peak=gbs / peak, l2_resident=packed < l2,
                   nodes_per_item_max=info["nodes_per_item_max"], slots=info["slots"],
                   items_global=info["items_global"], producer_warps=info["producer_warps"], setup_s=round(setup, 1),
                   factor="device" if a.device_factor else "host")
        rows.append(row)
        print(json.dumps(row), flush=True)
        del c, p
        torch.cuda.empty_cache()
    if a.out:
        json.dump({"peak_gbs": peak, "l2_bytes": l2, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
