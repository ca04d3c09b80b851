"""Subtree sharding on one B200.

* world = 1 with a real NCCL communicator: the two-launch sharded sweep
  (local backward | exchange allreduce | top + forward) must reproduce the
  single-launch handle bitwise, and so must whole solves (every reduction
  of the dual-space kernels goes through the phase / allgather path).
* W emulated ranks on the phase API (handles without a communicator,
  exchange done here on the host): each rank packs only its own subtrees;
  summing the ranks' exchange buffers and Hx must reproduce the unsharded
  Hx (1e-12: the per-item summation order depends on how a shard's nodes
  are grouped into items).
* W emulated ranks of a shard group (one host thread per rank, exchanges
  through host memory after stream synchronisation): the whole sharded
  solver, dual vectors sharded by row ownership, against the unsharded
  solver and the oracle.
Kernels of different ranks never wait on one another: every exchange sits
between launches."""
import ctypes as C

import numpy as np
import pytest

import paper_2107_01745_b200 as so
from paper_2107_01745_b200 import _native as N
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
P = C.POINTER(C.c_double)


def shapes():
    rng = orc.Rng(77)
    return [so.gen_random_instance(2, 6, 3, 9, [3, 1, 4, 2]),
            so.gen_random_instance(3, 5, 2, 8, [2, 2, 2, 2, 2]),
            so.ProblemInstance.from_flat(rng.random_instance(6, 400, 3, 2,
                                                             orc.InstanceOptions(with_l1=True)).flat())]


def both_handles(prob, world=1, rank=0, nccl=True, stage=-1):
    full = so.factor(prob)
    shard = so.factor(prob)
    shard.shard(rank, world, so.nccl_unique_id() if nccl else None, 0, stage)
    return full, shard


@pytest.mark.parametrize("stage", [-1, 2])
def test_world1_sharded_sweep_is_bitwise_the_single_launch(gpu, stage):
    for prob in shapes():
        full, shard = both_handles(prob, stage=stage)
        info = shard.dev_info()
        assert info["world"] == 1 and info["shard_stage"] == (1 if stage < 0 else stage)
        rng = np.random.default_rng(3)
        y = rng.uniform(-1, 1, prob.dual_dim)
        r = rng.uniform(-1, 1, prob.dual_dim)
        for affine in (True, False):
            pf, hf = so.sweep(full, [y, r], affine)
            ps, hs = so.sweep(shard, [y, r], affine)
            for k in range(2):
                assert np.array_equal(hf[k], hs[k])
        a = so.dual_grad(full, prob, y)
        b = so.dual_grad(shard, prob, y)
        assert np.array_equal(a.x, b.x) and np.array_equal(a.u, b.u)


def test_world1_sharded_solves_reproduce_the_single_launch(gpu):
    prob = so.gen_random_instance(5, 6, 3, 8, [3, 3, 2])
    full, shard = both_handles(prob)
    for kind in ("minfbe", "nama"):
        cfg = so.SolverConfig(nama_parallel_linesearch=(kind == "nama"))
        a = so.api._solve_direct(kind, prob, full, cfg)
        b = so.api._solve_direct(kind, prob, shard, cfg)
        assert a.status == b.status == "converged"
        assert a.iterations == b.iterations
        assert np.array_equal(a.y, b.y) and np.array_equal(a.x.x, b.x.x)
        assert a.stats.dual_grad_calls == b.stats.dual_grad_calls


class EmulatedRank:
    def __init__(self, prob, rank, world, stage):
        self.cache = so.factor(prob)
        self.cache.shard(rank, world, None, 0, stage)
        self.dev = self.cache.device()
        self.lib = N.lib()
        self.D = prob.dual_dim
        self.y = [self._alloc(self.D) for _ in range(2)]
        self.h = [self._alloc(self.D) for _ in range(2)]
        buf, n = P(), C.c_size_t()
        so.api.check(self.lib.scenopt_shard_exchange_buffer(self.dev, C.byref(buf), C.byref(n)))
        self.xbuf, self.nx = C.cast(buf, C.c_void_p).value, n.value

    def _alloc(self, n):
        p = C.c_void_p()
        so.api.check(self.lib.scenopt_dev_alloc(self.dev, C.c_size_t(8 * n), C.byref(p)))
        return p.value

    def put(self, dst, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        so.api.check(self.lib.scenopt_dev_memcpy(self.dev, C.c_void_p(dst), a.ctypes.data_as(C.c_void_p),
                                                 C.c_size_t(a.nbytes), 1))

    def get(self, src, n):
        a = np.empty(n)
        so.api.check(self.lib.scenopt_dev_memcpy(self.dev, a.ctypes.data_as(C.c_void_p), C.c_void_p(src),
                                                 C.c_size_t(8 * n), 2))
        return a

    def phase(self, ph, nrhs, affine):
        Y = (P * 2)(*[C.cast(C.c_void_p(p), P) for p in self.y])
        H = (P * 2)(*[C.cast(C.c_void_p(p), P) for p in self.h])
        so.api.check(self.lib.scenopt_shard_sweep_phase(self.dev, ph, nrhs, int(affine), Y, H))
        so.api.check(self.lib.scenopt_dev_synchronize(self.dev))


@pytest.mark.parametrize("world,stage,grid", [(2, -1, 0), (3, 2, 0), (4, 3, 6), (2, 4, 3)])
def test_emulated_ranks_reassemble_the_unsharded_sweep(gpu, monkeypatch, world, stage, grid):
    if grid:
        monkeypatch.setenv("SCENOPT_GRID", str(grid))  # force CTA-level cuts inside the shards
        monkeypatch.setenv("SCENOPT_MIN_SUBTREES", "1")
    for prob in shapes():
        counts = np.diff(prob.flat()["stage_offsets"])
        st = stage if stage > 0 else int(np.argmax(counts >= world))
        if st > prob.num_stages or counts[st] < world:
            continue
        full = so.factor(prob)
        ranks = [EmulatedRank(prob, r, world, st) for r in range(world)]
        infos = [rk.cache.dev_info() for rk in ranks]
        assert infos[0]["shard_first"] == prob.flat()["stage_offsets"][st]
        assert all(infos[i]["shard_past"] == infos[i + 1]["shard_first"] for i in range(world - 1))
        rng = np.random.default_rng(world)
        ys = [rng.uniform(-1, 1, prob.dual_dim) for _ in range(2)]
        for nrhs, affine in ((1, True), (2, False), (2, True)):
            for rk in ranks:
                for k in range(nrhs):
                    rk.put(rk.y[k], ys[k])
                    rk.put(rk.h[k], np.full(prob.dual_dim, np.nan))  # rows nobody zeroes or writes show up
                rk.phase(0, nrhs, affine)
            total = sum(rk.get(rk.xbuf, nrhs * rk.nx) for rk in ranks)
            for rk in ranks:
                rk.put(rk.xbuf, total)
                rk.phase(1, nrhs, affine)
            _, want = so.sweep(full, ys[:nrhs], affine)
            for k in range(nrhs):
                got = sum(rk.get(rk.h[k], prob.dual_dim) for rk in ranks)
                err = np.abs(got - want[k]).max() / (1.0 + np.abs(want[k]).max())
                assert err < 1e-12, (world, st, nrhs, affine, err)


def _emulated_solve(prob, world, stage, kind, cfg):
    """W sharded handles of one emulated group (one host thread per rank,
    exchanges through host memory), all solving the same problem."""
    import threading

    group = so.ShardGroup(world)
    caches = []
    for r in range(world):
        c = so.factor(prob)
        c.shard_emulated(r, group, 0, stage)
        caches.append(c)
    reps, errs = [None] * world, []

    def run(r):
        try:
            reps[r] = so.api._solve_direct(kind, prob, caches[r], cfg)
        except Exception as e:  # noqa: BLE001 - re-raised below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return reps, caches


@pytest.mark.parametrize("world,stage", [(2, -1), (3, 2), (4, 1)])
def test_emulated_ranks_solve_like_the_unsharded_handle(gpu, world, stage):
    """The sharded solver with W ranks on one GPU (emulated group): dual and
    primal vectors sharded by subtree, one exchange allreduce per sweep and
    one allgather of partial sums per reduction. Every rank takes the same
    decisions (bitwise-identical reports), and the result is the unsharded
    solver's: iterations within 1, iterates within the tolerance, oracle
    counts equal when the iterations are."""
    prob = so.gen_random_instance(5, 6, 3, 8, [4, 3, 2])
    po = orc.Problem.from_flat(prob.flat())
    full = so.factor(prob)
    for kind in ("minfbe", "nama"):
        cfg = so.SolverConfig(eps=1e-6, nama_parallel_linesearch=(kind == "nama"))
        ref = so.api._solve_direct(kind, prob, full, cfg)
        reps, caches = _emulated_solve(prob, world, stage, kind, cfg)
        assert caches[0].dev_info()["world"] == world
        for rep in reps[1:]:
            assert rep.iterations == reps[0].iterations
            assert np.array_equal(rep.y, reps[0].y) and np.array_equal(rep.x.x, reps[0].x.x)
        rep = reps[0]
        assert rep.status == ref.status == "converged"
        assert abs(rep.iterations - ref.iterations) <= 1
        if rep.iterations == ref.iterations:
            assert rep.stats.dual_grad_calls == ref.stats.dual_grad_calls
            assert rep.stats.hessian_vec_calls == ref.stats.hessian_vec_calls
        assert rep.lipschitz_estimate == pytest.approx(ref.lipschitz_estimate, rel=1e-9)
        assert np.abs(rep.y - ref.y).max() <= 10 * cfg.eps * (1 + np.abs(ref.y).max())
        assert np.abs(rep.x.x - ref.x.x).max() <= 10 * cfg.eps * (1 + np.abs(ref.x.x).max())
        # and the CPU oracle's iteration count
        orep = orc.solve(po, orc.SolverConfig(eps=1e-6, nama_parallel_linesearch=cfg.nama_parallel_linesearch),
                         {"minfbe": 0, "nama": 1}[kind])
        assert abs(rep.iterations - orep["iterations"]) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_ranks_solve_c3(gpu, world):
    """C3 (1.24M variables) sharded at stage 1 over 2 / 3 emulated ranks:
    NAMA (p-NAMA, 2-RHS sweeps) and MINFBE reach the unsharded handle's
    iterates with the same iteration counts."""
    prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
    full = so.factor(prob)
    L, _ = so.estimate_dual_lipschitz(full, prob)
    for kind in ("nama", "minfbe"):
        cfg = so.SolverConfig(lambda0=0.9 / L, nama_parallel_linesearch=(kind == "nama"))
        ref = so.api._solve_direct(kind, prob, full, cfg)
        reps, _ = _emulated_solve(prob, world, 1, kind, cfg)
        rep = reps[0]
        assert rep.status == "converged" and abs(rep.iterations - ref.iterations) <= 1
        assert np.abs(rep.y - ref.y).max() <= 10 * cfg.eps * (1 + np.abs(ref.y).max())
        assert rep.residual_inf <= cfg.eps


def test_world1_sharded_device_factor_is_bitwise_the_device_factor(gpu):
    """K9 on a sharded handle (world 1, NCCL): own subtrees, the exchange of
    the shard-stage value matrices, the replicated top -- the same factor,
    sweeps and solves as the unsharded device factor, bit for bit."""
    prob = so.gen_random_instance(5, 6, 3, 8, [3, 3, 2])
    full = so.factor_device(prob)
    shard = so.DeviceFactorCache.sharded(prob, 0, 1, so.nccl_unique_id())
    assert shard.dev_info()["device_factor"] == 1 and shard.dev_info()["world"] == 1
    y = np.random.default_rng(2).uniform(-1, 1, prob.dual_dim)
    a, b = so.dual_grad(full, prob, y), so.dual_grad(shard, prob, y)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.u, b.u)
    for kind in ("minfbe", "nama"):
        cfg = so.SolverConfig(nama_parallel_linesearch=(kind == "nama"))
        ra = so.api._solve_direct(kind, prob, full, cfg)
        rb = so.api._solve_direct(kind, prob, shard, cfg)
        assert ra.iterations == rb.iterations and np.array_equal(ra.y, rb.y)


@pytest.mark.parametrize("world,stage,shape", [(2, -1, (5, 6, 3, 8, [4, 3, 2])), (3, 2, (5, 6, 3, 8, [4, 3, 2])),
                                               (4, 1, (7, 5, 2, 9, [4, 2, 2, 2]))])
def test_emulated_ranks_factor_on_the_device(gpu, world, stage, shape):
    """Every rank factors only its own subtrees plus the replicated top on
    the device (no host factor anywhere): sweeps reassemble the host
    factor's, and the sharded solves match the unsharded solver."""
    import threading

    prob = so.gen_random_instance(*shape)
    full = so.factor(prob)
    group = so.ShardGroup(world)
    caches = [None] * world
    errs = []

    def make(r):
        try:
            caches[r] = so.DeviceFactorCache.sharded(prob, r, group=group, stage=stage)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=make, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    y = np.random.default_rng(world).uniform(-1, 1, prob.dual_dim)
    ref = so.dual_grad(full, prob, y)
    outs = [None] * world

    def grad(r):
        outs[r] = so.dual_grad(caches[r], prob, y)

    ts = [threading.Thread(target=grad, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for pt in outs:
        scale = 1 + np.abs(ref.x).max()
        assert np.abs(pt.x - ref.x).max() <= 1e-9 * scale and np.abs(pt.u - ref.u).max() <= 1e-9 * scale
    for kind in ("minfbe", "nama"):
        cfg = so.SolverConfig(eps=1e-6, nama_parallel_linesearch=(kind == "nama"))
        want = so.api._solve_direct(kind, prob, full, cfg)
        reps = [None] * world

        def run(r):
            reps[r] = so.api._solve_direct(kind, prob, caches[r], cfg)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert all(rp is not None for rp in reps)
        rep = reps[0]
        assert rep.status == "converged" and abs(rep.iterations - want.iterations) <= 1
        assert np.abs(rep.y - want.y).max() <= 10 * cfg.eps * (1 + np.abs(want.y).max())


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_ranks_with_per_rank_instances(gpu, world):
    """Each rank builds only its part of the instance
    (gen_random_instance_shard) and factors it on the device; nobody holds
    the whole tree. The sharded solves reach the full instance's iterates."""
    import threading

    shape = (5, 6, 3, 8, [4, 3, 2])
    full_prob = so.gen_random_instance(*shape)
    want_cache = so.factor(full_prob)
    group = so.ShardGroup(world)
    parts = [so.gen_random_instance_shard(*shape, rank=r, world=world) for r in range(world)]
    caches, errs = [None] * world, []

    def make(r):
        try:
            caches[r] = so.DeviceFactorCache.sharded(parts[r], r, group=group)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=make, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    for kind in ("minfbe", "nama"):
        cfg = so.SolverConfig(eps=1e-6, nama_parallel_linesearch=(kind == "nama"))
        want = so.api._solve_direct(kind, full_prob, want_cache, cfg)
        reps = [None] * world

        def run(r):
            reps[r] = so.api._solve_direct(kind, parts[r], caches[r], cfg)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        rep = reps[0]
        assert rep is not None and rep.status == "converged"
        assert abs(rep.iterations - want.iterations) <= 1
        assert np.abs(rep.y - want.y).max() <= 10 * cfg.eps * (1 + np.abs(want.y).max())
        assert np.abs(rep.x.x - want.x.x).max() <= 10 * cfg.eps * (1 + np.abs(want.x.x).max())
