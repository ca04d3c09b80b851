#!/usr/bin/env python3
"""Benchmark of the B200 MINFBE / NAMA hot path (BASELINE.json).

Metric: dual-gradient (Alg. 3) evaluations per second on the ~1M-variable
scenario tree C3 (nx=50, nu=20, N=20, branching [8,8,8,2]), as a fraction of
the measured HBM roofline; time-to-tolerance of MINFBE and NAMA on the same
tree is reported beside it.

A step is one dual-gradient evaluation: one fused backward/forward sweep
with apply_H (the hot kernel) on device-resident inputs. The working set
(1.2 GB of packed matrices) is ~10x the 126 MB L2, so every step streams
from HBM without an explicit flush.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (nx, nu, N, branching, label)
    "c3": (50, 20, 20, [8, 8, 8, 2], "C3: MINFBE/NAMA ~1M-variable tree (nx=50, nu=20, N=20, branching [8,8,8,2])"),
    "c1": (10, 5, 10, [2, 2, 2], "C1: small tree (nx=10, nu=5, N=10, branching [2,2,2])"),
    "c4": (50, 20, 20, [8, 8, 8, 8, 4], "C4: NAMA ~20M-variable tree (nx=50, nu=20, N=20, branching [8,8,8,8,4])"),
    "c5a": (10, 5, 20, [2] * 13, "C5: oracle microbench, 73,727 nodes (nx=10, nu=5, N=20, [2]x13)"),
    "c5b": (10, 5, 20, [4] * 8, "C5: oracle microbench, 873,813 nodes (nx=10, nu=5, N=20, [4]x8)"),
    "c5c": (50, 20, 20, [4] * 6, "C5: oracle microbench, 60,074 nodes (nx=50, nu=20, N=20, [4]x6)"),
}
METRIC = "time-to-tolerance & dual-grad evals/s on 1M-var tree; % of HBM roofline"


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for name, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def cpu_solves(orc, po, fac, lam0s, gpu_ttt=None):
    """The CPU oracle's MINFBE and NAMA (p-NAMA: the reference's second thread,
    solvers.hpp:411-418) from y0 = 0 at the given lambda0, with the
    reference's wall_ms semantics (solvers.hpp:240, 166-168)."""
    out = {}
    for kind, code in (("minfbe", 0), ("nama", 1)):
        cfg = orc.SolverConfig(lambda0=lam0s[kind], nama_parallel_linesearch=(kind == "nama"))
        rep = orc.solve_direct(po, fac, cfg, code)
        row = {"ms": rep["wall_ms"], "iterations": rep["iterations"],
               "status": "converged" if rep["status"] == 0 else "max_iters_exceeded",
               "dual_grad_calls": rep["dual_grad_calls"], "hessian_vec_calls": rep["hessian_vec_calls"],
               "residual_inf": rep["residual_inf"], "lambda0": lam0s[kind],
               "threads": 2 if kind == "nama" else 1}
        if gpu_ttt and kind in gpu_ttt:
            g = gpu_ttt[kind]
            row["gpu_iterations"] = g["iterations"]
            row["iterations_within_1"] = abs(g["iterations"] - rep["iterations"]) <= 1
            if "y" in g:
                yo = rep["y"]
                row["y_gap_inf"] = float(np.abs(g.pop("y") - yo).max())
                row["y_gap_bound"] = 10 * cfg.eps * (1 + float(np.abs(yo).max()))
            row["gpu_speedup"] = rep["wall_ms"] / g["ms"] if g.get("ms") else None
        out[kind] = row
    return out


def cpu_baseline(flat, lam0s=None, gpu_ttt=None, target_s=10.0):
    """The CPU oracle (restatement of the reference, built -O3 -march=native
    on this host; single thread, as the reference's serial node loops) on a
    bounded sample of the workload, plus its MINFBE / NAMA time-to-tolerance
    at the device's lambda0."""
    from oracle import oracle as orc

    native = orc.use_native()
    po = orc.Problem.from_flat(flat)
    fac = orc.Factor(po)
    t1 = fac.time_sweeps(1, True)
    n = max(2, min(200, int(math.ceil(target_s / max(t1, 1e-6)))))
    t = fac.time_sweeps(n, True)
    out = {"value": 1.0 / t, "unit": "dual-grad evals/s", "cores": 1, "kind": "port",
           "build": "g++ -O3 -march=native (built on this host)" if native else "portable -O3 (native build failed)",
           "host_cpu": host_cpu(),
           "sample": f"{n} affine sweeps (dual_grad) of the same instance on one host thread, "
                     f"{t * 1e3:.1f} ms each; MINFBE and NAMA solved to tolerance once each"}
    if lam0s:
        out["time_to_tolerance"] = cpu_solves(orc, po, fac, lam0s, gpu_ttt)
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (oracle port, since the
    reference does not compile without Eigen) on this box's host cores."""
    if rank != 0:
        return
    from oracle import oracle as orc

    native = orc.use_native()
    nx, nu, N, br, label = CONFIGS[args.config]
    t0 = time.time()
    po = orc.gen_random(1, nx, nu, N, br)
    fac = orc.Factor(po)
    setup_s = time.time() - t0
    t1 = fac.time_sweeps(1, True)
    # All host threads: the reference's sweep is serial (tree_oracles.hpp:54-88),
    # so the CPU path's throughput comes from independent evaluations running
    # side by side on the shared (read-only) factor, one per core. Each step is
    # one round of `threads` concurrent sweeps.
    import threading

    threads = max(1, min(os.cpu_count() or 1, 64))

    def round_of(k):
        ts = [threading.Thread(target=fac.time_sweeps, args=(k, True)) for _ in range(threads)]
        tt = time.perf_counter()
        for th in ts:
            th.start()
        for th in ts:
            th.join()
        return time.perf_counter() - tt

    budget = 60.0  # seconds of timed CPU work
    w = min(args.warmup, 3)  # warm-up rounds (the arm's own W >= 3, bounded: each round is ~0.15 s)
    round_of(w)
    tr = round_of(1)  # one concurrent sweep per thread
    k = min(args.steps, max(2, int(budget / max(tr, 1e-6))))
    wall = round_of(k)
    t = wall / (k * threads)  # seconds per evaluation, aggregate
    value = 1.0 / t
    # time-to-tolerance as solve() runs it (solvers.hpp:668-679): L by power
    # iteration once (reported apart), then each solver from y0 = 0
    ttt = None
    if args.config in ("c1", "c3"):
        tl = time.perf_counter()
        L, lip_sweeps = fac.estimate_lipschitz()
        ttt = {"lipschitz": {"ms": (time.perf_counter() - tl) * 1e3, "sweeps": lip_sweeps, "estimate": L}}
        ttt.update(cpu_solves(orc, po, fac, {"minfbe": 0.9 / L, "nama": 0.9 / L}))
    out = {"metric": METRIC, "value": value, "unit": "dual-grad evals/s", "impl": "reference",
           "n_gpus": world, "steps": k, "warmup": w, "ms_per_step": t * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded gen_random_instance, seed 1)",
           "config": {"workload": label, "nodes": po.flat()["num_nodes"], "dual_dim": po.dual_dim,
                      "setup_s": setup_s},
           "cpu_baseline": {"value": value, "unit": "dual-grad evals/s", "cores": threads, "kind": "port",
                            "build": "g++ -O3 -march=native (built on this host)" if native else "portable -O3",
                            "host_cpu": host_cpu(),
                            "sample": f"{k} rounds of {threads} concurrent affine sweeps (one per host "
                                      f"thread, {wall / k * 1e3:.0f} ms per round) of the CPU oracle "
                                      "(Eigen-free restatement of the reference; serial single-thread "
                                      f"sweep {t1 * 1e3:.1f} ms)"},
           "time_to_tolerance": ttt,
           "e2e": {"value": value, "unit": "dual-grad evals/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--solves", type=int, default=5, help="timed solves per solver (median reported)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-shard", action="store_true",
                    help="use the sharded (NCCL) handle even at one GPU (exercises the N>1 path)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = one tree of N config-sized subtrees (default); strong = the "
                         "config's own tree sharded over N GPUs (BASELINE config 4: --config c4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    # NCCL's version banner goes to stdout, where only the JSON line belongs
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    import torch
    import torch.distributed as dist

    import paper_2107_01745_b200 as so
    from paper_2107_01745_b200 import _native as Nat

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local if world > 1 else 0
    torch.cuda.set_device(device)

    nx, nu, N, br, label = CONFIGS[args.config]
    units = 1  # config-sized evaluations per sweep of the benchmarked tree
    sharded = world > 1 or args.force_shard
    if sharded and args.scaling == "weak":
        # Weak scaling over subtree shards: N GPUs solve ONE tree
        # of N config-sized subtrees, branching [8N, ...] (N = 1 is exactly the
        # config), sharded at stage 1 -- each rank owns 8 of the 8N stage-1
        # subtrees and replicates the root. Per sweep: one NCCL allreduce of
        # the stage-1 exchange buffer; per dual-kernel reduction: one
        # allgather of the ranks' partial sums. x / u / Hx stay on their owners.
        br = [br[0] * world] + list(br[1:])
        units = world
        label = f"{label}; x{world} sharded: one tree [{', '.join(map(str, br))}] over {world} GPUs"
    elif sharded:
        label = f"{label}; strong scaling: the same tree sharded over {world} GPUs"
    t0 = time.time()
    if sharded:
        # each rank builds only its part of the instance (its subtrees, the
        # top and the stage-1 nodes; bit-identical to the full instance there)
        # and factors it on the device: no rank holds the whole tree or a
        # host factor
        prob = so.gen_random_instance_shard(1, nx, nu, N, br, rank, world, 1)
        nid = [so.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(nid, src=0)
        cache = so.DeviceFactorCache.sharded(prob, rank, world, nid[0], device=device, stage=1)
    else:
        prob = so.gen_random_instance(1, nx, nu, N, br)
        cache = so.factor(prob)
    dev = cache.device(device)
    setup_s = time.time() - t0
    info = cache.dev_info()
    lib = so.lib()
    s = C.c_void_p()
    so.api.check(lib.scenopt_dev_stream(dev, C.byref(s)))
    stream = torch.cuda.ExternalStream(s.value, device=device)
    D = prob.dual_dim
    gen = torch.Generator(device="cpu").manual_seed(7)
    y = torch.rand(D, dtype=torch.float64, generator=gen).mul_(2).sub_(1).to(f"cuda:{device}")
    x = torch.empty(nx * prob.num_nodes(), dtype=torch.float64, device=f"cuda:{device}")
    u = torch.empty(nu * max(prob.first_leaf, 1), dtype=torch.float64, device=f"cuda:{device}")
    hx = torch.empty(D, dtype=torch.float64, device=f"cuda:{device}")
    P = C.POINTER(C.c_double)
    Y = (P * 2)(C.cast(y.data_ptr(), P), None)
    X = (P * 2)(C.cast(x.data_ptr(), P), None)
    U = (P * 2)(C.cast(u.data_ptr(), P), None)
    H = (P * 2)(C.cast(hx.data_ptr(), P), None)

    def step():
        # sharded: the primal stays on its owners (no gather inside the step)
        so.api.check(lib.scenopt_dev_sweep_async(dev, 1, 1, Y, None if sharded else X, None if sharded else U, H))

    for _ in range(args.warmup):
        step()
    so.api.check(lib.scenopt_dev_synchronize(dev))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        e1.synchronize()
        # e2e through the reference-facing call (dual_grad with host I/O)
        yh = torch.empty(D, dtype=torch.float64, pin_memory=True)
        yh.copy_(y.cpu())
        xh = torch.empty(nx * prob.num_nodes(), dtype=torch.float64, pin_memory=True)
        uh = torch.empty(nu * max(prob.first_leaf, 1), dtype=torch.float64, pin_memory=True)
        yp, xp, up = (C.cast(t.data_ptr(), P) for t in (yh, xh, uh))
        for _ in range(3):
            so.api.check(lib.scenopt_dual_grad(dev, yp, xp, up, 1))
        ke = max(10, args.steps // 4)
        te = time.perf_counter()
        for _ in range(ke):
            so.api.check(lib.scenopt_dual_grad(dev, yp, xp, up, 1))
        e2e_s = (time.perf_counter() - te) / ke
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
        dist.barrier()
    value = units * 1e3 / ms
    e2e_value = units / e2e_s

    # time-to-tolerance: MINFBE and NAMA from y0 = 0 with the reference
    # defaults. As in solve() (solvers.hpp:668-679), L is estimated once by
    # power iteration and lambda0 = 0.9 / L is passed to the loop; the
    # report's wall_ms (solvers.hpp:240, 166-168) then covers the iterations
    # only, and the power iteration is reported beside it.
    ttt = {}
    y_last = {}
    if not args.no_solve:
        so.estimate_dual_lipschitz(cache, prob)  # untimed: module load
        torch.cuda.synchronize()
        tl = time.perf_counter()
        L, lip_sweeps = so.estimate_dual_lipschitz(cache, prob)
        lip_ms = (time.perf_counter() - tl) * 1e3
        ttt["lipschitz"] = {"ms": lip_ms, "sweeps": lip_sweeps, "estimate": L}
        for kind in ("minfbe", "nama"):
            cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
            so.api._solve_direct(kind, prob, cache, cfg)  # untimed: workspace, module load
            # each report is dropped before the next solve: a caller holding
            # every result would hand each download fresh (faulting) host pages
            walls = []
            for _ in range(max(args.solves, 1)):
                rep = so.api._solve_direct(kind, prob, cache, cfg)
                walls.append(rep.wall_ms)
            walls.sort()
            ttt[kind] = {"ms": statistics.median(walls), "ms_min": walls[0], "ms_runs": walls,
                         "iterations": rep.iterations, "status": rep.status,
                         "dual_grad_calls": rep.stats.dual_grad_calls,
                         "hessian_vec_calls": rep.stats.hessian_vec_calls,
                         "residual_inf": rep.residual_inf,
                         "lambda0": cfg.lambda0}
            y_last[kind] = rep.y.copy()

    peaks, peak_src = measured_peaks()
    bytes_step = info["sweep_bytes_aff"]  # algorithmic bytes of the whole tree
    achieved = bytes_step / world / (ms * 1e-3) / 1e9  # per GPU
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(args.config, {}).get("dram_bytes_per_launch") if not sharded else None
        except (OSError, ValueError):
            traffic = None
    out = {
        "metric": METRIC, "value": value, "unit": "dual-grad evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded gen_random_instance, seed 1; random-system tree)",
        "config": {"workload": label, "nodes": prob.num_nodes(), "primal_dim": prob.primal_dim(),
                   "dual_dim": D,
                   "parallelism": (f"subtree shards x{world} (stage {info['shard_stage']}; per sweep one NCCL "
                                   f"allreduce of {8 * info.get('exchange_doubles', 0)} B; per dual-kernel "
                                   "reduction one allgather of partial sums)") if sharded else "1 GPU",
                   "value_units": ("C3-sized dual-grad evaluations (a sweep of the x{0} tree counts {0})"
                                   .format(units)) if sharded else "dual-grad evaluations of the tree",
                   "l2": "inputs larger than L2 (packed matrices %.2f GB vs 126 MB L2)"
                         % ((info["matrix_bytes_bw"] + info["matrix_bytes_fw"]) / 1e9),
                   "setup_s": round(setup_s, 2), "grid_ctas": info["grid_ctas"],
                   "slots": info["slots"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_step},
        "e2e": {"value": e2e_value, "unit": "dual-grad evals/s",
                "h2d_bytes_per_step": 8 * D,
                "d2h_bytes_per_step": 8 * (nx * prob.num_nodes() + nu * prob.first_leaf)},
        "gpu_launches": args.steps * (2 if sharded else 1),
        "time_to_tolerance": ttt,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # CPU solver at the device's lambda0; compared with the device's
        # iterates (iterations within 1, y within 10 eps), then dropped
        gpu = {k: dict(v, y=y_last[k]) for k, v in ttt.items() if k in y_last}
        lam0s = {k: v["lambda0"] for k, v in ttt.items() if k in ("minfbe", "nama")}
        out["cpu_baseline"] = cpu_baseline(prob.flat(), lam0s or None, gpu)
    if rank == 0:
        print(json.dumps(out), flush=True)
    # release the handle (and with it the library's own NCCL communicator)
    # while every rank is still alive, before the process group goes away
    del dev, cache
    import gc

    gc.collect()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
