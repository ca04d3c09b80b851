"""C4 (18.35M variables) sharded at stage 1 over W emulated ranks on one GPU
(per-rank instances, device factor), NAMA and MINFBE against the unsharded
device-factor handle: iterations within 1, y within 10 eps, every rank's
report bitwise equal. python tools/c4_emulated_check.py [W]"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_01745_b200 as so
W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
shape = (1, 50, 20, 20, [8, 8, 8, 8, 4])
t0 = time.time()
full = so.gen_random_instance(*shape)
fcache = so.factor_device(full)
print(f"full instance + device factor {time.time() - t0:.1f} s", flush=True)
group = so.ShardGroup(W)
parts = [so.gen_random_instance_shard(*shape, r, W, 1) for r in range(W)]
caches = [None] * W


def build(r):
    caches[r] = so.DeviceFactorCache.sharded(parts[r], r, W, group=group, stage=1)
    caches[r].device()


ts = [threading.Thread(target=build, args=(r,)) for r in range(W)]
[t.start() for t in ts]
[t.join() for t in ts]
print(f"{W} sharded handles {time.time() - t0:.1f} s", flush=True)
for kind in ("nama", "minfbe"):
    cfg = so.SolverConfig(nama_parallel_linesearch=kind == "nama")
    ref = so.api._solve_direct(kind, full, fcache, cfg)
    out = [None] * W

    def run(r):
        out[r] = so.api._solve_direct(kind, parts[r], caches[r], cfg)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(W)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for r in range(1, W):
        assert out[r].iterations == out[0].iterations and np.array_equal(out[r].y, out[0].y)
    gap = np.abs(out[0].y - ref.y).max()
    bound = 10 * cfg.eps * (1 + np.abs(ref.y).max())
    print(f"{kind}: unsharded {ref.iterations} it {ref.wall_ms:.1f} ms | {W} emulated ranks {out[0].iterations} it "
          f"{out[0].wall_ms:.1f} ms | y gap {gap:.2e} (bound {bound:.1e})", flush=True)
    assert abs(out[0].iterations - ref.iterations) <= 1 and gap <= bound
print("ok")
