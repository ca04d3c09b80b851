"""GPU parity of the fused sweep (dual_grad / hessian_vec, tree_oracles.hpp:
33-114) against the CPU oracle, plus the reference's property tests
(test_tree_oracles.cpp) run through the CUDA path. Tolerance: 1e-9
relative (north_star), using the reference's rel_gap metric."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

pytestmark = pytest.mark.gpu

TOL = 1e-9


def both(prob_o):
    """Same instance bytes on both sides."""
    flat = prob_o.flat()
    prob = so.ProblemInstance.from_flat(flat)
    return prob, so.factor(prob), orc.Factor(prob_o)


def test_dual_grad_matches_oracle_on_random_trees(gpu):
    rng = orc.Rng(41)  # test_tree_oracles.cpp:23-36
    for trial in range(20):
        stages = rng.integer(1, 5)
        po = rng.random_instance(stages, 40, rng.integer(1, 4), rng.integer(1, 4))
        prob, cache, ofac = both(po)
        y = rng.vector(prob.dual_dim, 2.0)
        fast = so.dual_grad(cache, prob, y)
        ox, ou = ofac.dual_grad(y)
        gap = sup.rel_gap(ox, ou, fast.x.ravel(order="F"), fast.u.ravel(order="F"))
        assert gap < TOL, (trial, gap)
        kx, ku = sup.kkt_dual_grad(po.flat(), y)
        assert sup.rel_gap(kx, ku, fast.x.ravel(order="F"), fast.u.ravel(order="F")) < 1e-8


def test_hessian_vec_matches_oracle_and_homogeneity(gpu):
    rng = orc.Rng(43)  # test_tree_oracles.cpp:64-81
    for trial in range(10):
        po = rng.random_instance(rng.integer(1, 4), 30, 3, 2)
        prob, cache, ofac = both(po)
        y = rng.vector(prob.dual_dim, 2.0)
        r = rng.vector(prob.dual_dim, 2.0)
        hom = so.hessian_vec(cache, prob, r)
        ox, ou = ofac.hessian_vec(r)
        assert sup.rel_gap(ox, ou, hom.x.ravel(order="F"), hom.u.ravel(order="F")) < TOL
        a = so.dual_grad(cache, prob, y)
        b = so.dual_grad(cache, prob, y + r)
        dx, du = (b.x - a.x).ravel(order="F"), (b.u - a.u).ravel(order="F")
        assert sup.rel_gap(dx, du, hom.x.ravel(order="F"), hom.u.ravel(order="F")) < TOL


@pytest.mark.parametrize("opt", [dict(), dict(with_l1=True, with_none=True),
                                 dict(affine=False, stage_rows_lo=0, stage_rows_hi=3)])
def test_fused_apply_H_matches_oracle(gpu, opt):
    rng = orc.Rng(12)
    for trial in range(6):
        po = rng.random_instance(rng.integer(1, 4), 60, rng.integer(1, 5), rng.integer(1, 4),
                                 orc.InstanceOptions(**opt))
        prob, cache, ofac = both(po)
        y = rng.vector(prob.dual_dim, 1.5)
        for affine in (True, False):
            pts, hs = so.sweep(cache, [y], affine)
            ox, ou = ofac.sweep(y, affine)
            Hx = orc.apply_H(po, ox, ou)
            assert np.abs(hs[0] - Hx).max() <= TOL * (1 + np.abs(Hx).max())


def test_two_rhs_sweep_is_bitwise_two_single_sweeps(gpu):
    rng = orc.Rng(1213)
    po = rng.random_instance(4, 120, 4, 3, orc.InstanceOptions(with_l1=True, with_none=True))
    prob, cache, _ = both(po)
    a = rng.vector(prob.dual_dim)
    b = rng.vector(prob.dual_dim)
    for affine in (False, True):
        pts2, hs2 = so.sweep(cache, [a, b], affine)
        pa, ha = so.sweep(cache, [a], affine)
        pb, hb = so.sweep(cache, [b], affine)
        assert np.array_equal(hs2[0], ha[0]) and np.array_equal(hs2[1], hb[0])
        assert np.array_equal(pts2[0].x, pa[0].x) and np.array_equal(pts2[1].u, pb[0].u)


@pytest.mark.parametrize("shape", [(10, 5, 10, [2, 2, 2]), (6, 3, 6, [3, 1, 4]),
                                   (20, 8, 5, [8, 8]), (50, 20, 3, [8, 8])])
def test_generated_configs_match_oracle(gpu, shape):
    nx, nu, N, br = shape
    prob = so.gen_random_instance(1, nx, nu, N, br)
    po = orc.Problem.from_flat(prob.flat())
    cache = so.factor(prob)
    ofac = orc.Factor(po)
    rng = np.random.default_rng(5)
    y = rng.uniform(-1, 1, prob.dual_dim)
    for fn, ofn in ((so.dual_grad, ofac.dual_grad), (so.hessian_vec, ofac.hessian_vec)):
        pt = fn(cache, prob, y)
        ox, ou = ofn(y)
        assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < TOL


def test_repeated_sweeps_are_deterministic(gpu):
    prob = so.gen_random_instance(3, 12, 4, 8, [3, 3, 2])
    cache = so.factor(prob)
    y = np.linspace(-1, 1, prob.dual_dim)
    first = so.dual_grad(cache, prob, y)
    for _ in range(20):
        again = so.dual_grad(cache, prob, y)
        assert np.array_equal(first.x, again.x) and np.array_equal(first.u, again.u)


def test_oracle_errors_mirror_reference(gpu):
    rng = orc.Rng(47)  # test_tree_oracles.cpp:143-152
    prob = so.ProblemInstance.from_flat(rng.random_instance(2, 12, 2, 2).flat())
    other = so.ProblemInstance.from_flat(rng.random_instance(2, 12, 3, 2).flat())
    cache = so.factor(prob)
    with pytest.raises(so.CacheMismatch):
        so.dual_grad(cache, other, np.zeros(other.dual_dim))
    with pytest.raises(so.DimensionMismatch):
        so.hessian_vec(cache, prob, np.zeros(prob.dual_dim + 1))


@pytest.mark.parametrize("grid,min_sub", [(4, 1), (8, 2), (16, 4), (3, 1), (16, 0)])
def test_subtree_ownership_schedule_matches_oracle(gpu, monkeypatch, grid, min_sub):
    """The per-CTA subtree schedule (local dependencies through the retire
    counter, global flags above the cut) at several grid sizes and cuts, on
    regular, irregular and random trees; the reduced grids force a cut on
    trees small enough for the oracle."""
    monkeypatch.setenv("SCENOPT_GRID", str(grid))
    monkeypatch.setenv("SCENOPT_MIN_SUBTREES", str(min_sub))
    rng = orc.Rng(900 + grid)
    cases = [orc.Problem.from_flat(so.gen_random_instance(2, 6, 3, 9, [3, 1, 4, 2]).flat()),
             orc.Problem.from_flat(so.gen_random_instance(4, 5, 2, 12, [2] * 7).flat()),
             rng.random_instance(6, 300, 3, 2, orc.InstanceOptions(with_l1=True, with_none=True))]
    for po in cases:
        prob, cache, ofac = both(po)
        info = cache.dev_info()
        assert info["grid_ctas"] == grid
        if min_sub == 0:
            assert info["cut_stage"] == -1
        y = rng.vector(prob.dual_dim, 1.5)
        r = rng.vector(prob.dual_dim, 1.5)
        for affine in (True, False):
            pts, hs = so.sweep(cache, [y, r], affine)
            for v, pt, h in ((y, pts[0], hs[0]), (r, pts[1], hs[1])):
                ox, ou = ofac.sweep(v, affine)
                assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < TOL
                Hx = orc.apply_H(po, ox, ou)
                assert np.abs(h - Hx).max() <= TOL * (1 + np.abs(Hx).max())


def test_default_grid_uses_subtree_ownership_on_c3(gpu):
    prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])  # BASELINE C3 shape
    info = so.factor(prob).dev_info()
    assert info["grid_ctas"] == info["sm_count"]
    assert info["cut_stage"] == 4  # 1024 subtrees >= 4 per CTA


@pytest.mark.parametrize("mode", [dict(SCENOPT_SLOT_KB="4"), dict(SCENOPT_STAGE="consumer"),
                                  dict(SCENOPT_SLOT_KB="6", SCENOPT_STAGE="consumer"),
                                  dict(SCENOPT_SLOT_KB="4", SCENOPT_GRID="5", SCENOPT_MIN_SUBTREES="1")])
def test_fallback_layouts_match_oracle(gpu, monkeypatch, mode):
    """Items larger than a shared-memory slot read their node blocks from HBM
    in place (kGlobalBlocks); very wide states stage vectors per consumer
    team. Forced on ordinary trees, 1- and 2-RHS."""
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    rng = orc.Rng(4242)
    cases = [orc.Problem.from_flat(so.gen_random_instance(3, 9, 4, 7, [3, 2, 2]).flat()),
             rng.random_instance(5, 200, 4, 3, orc.InstanceOptions(with_l1=True, with_none=True))]
    n_global = 0
    for po in cases:
        prob, cache, ofac = both(po)
        info = cache.dev_info()
        n_global += info["items_global"]
        if "SCENOPT_STAGE" in mode:
            assert info["consumer_stage"] == 1
        y = rng.vector(prob.dual_dim, 1.5)
        r = rng.vector(prob.dual_dim, 1.5)
        for affine in (True, False):
            pts, hs = so.sweep(cache, [y, r], affine)
            for v, pt, h in ((y, pts[0], hs[0]), (r, pts[1], hs[1])):
                ox, ou = ofac.sweep(v, affine)
                assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < TOL
                Hx = orc.apply_H(po, ox, ou)
                assert np.abs(h - Hx).max() <= TOL * (1 + np.abs(Hx).max())
    if "SCENOPT_SLOT_KB" in mode:
        assert n_global > 0


@pytest.mark.parametrize("dims", [(120, 60, [3, 2]), (300, 40, [2, 2])])
def test_wide_states_match_oracle(gpu, dims):
    """States far wider than the benchmark's (a node block of several
    hundred KB): the sweep picks the HBM-block / consumer-staged layouts by
    itself and still matches the oracle."""
    nx, nu, br = dims
    prob = so.gen_random_instance(7, nx, nu, 3, br)
    po = orc.Problem.from_flat(prob.flat())
    cache = so.factor(prob)
    ofac = orc.Factor(po)
    info = cache.dev_info()
    assert info["items_global"] > 0
    y = np.random.default_rng(1).uniform(-1, 1, prob.dual_dim)
    for fn, ofn in ((so.dual_grad, ofac.dual_grad), (so.hessian_vec, ofac.hessian_vec)):
        pt = fn(cache, prob, y)
        ox, ou = ofn(y)
        assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < TOL
    rep = so.solve(prob, so.SolverConfig(), "nama")
    assert rep.status == "converged" and rep.verified


def test_pinned_host_outputs_match_pageable_and_stay_in_bounds(gpu):
    """Pinned (mapped) caller buffers: the forward pass writes x / u into them
    over PCIe while it runs. The result must equal the pageable path bit for
    bit, and nothing may be written past u's nu*first_leaf elements (leaves
    carry no input) or past x's nx*n elements: guard zones around both
    buffers keep their sentinel."""
    import ctypes as C

    import torch

    from paper_2107_01745_b200 import _native as N

    prob = so.gen_random_instance(2, 12, 5, 9, [3, 3, 2])
    cache = so.factor(prob)
    y = np.random.default_rng(4).uniform(-1, 1, prob.dual_dim)
    ref = so.dual_grad(cache, prob, y)
    nx, nu, n, F = prob.nx, prob.nu, prob.num_nodes(), prob.first_leaf
    guard = 64
    P = C.POINTER(C.c_double)
    for _ in range(3):
        xb = torch.full((nx * n + 2 * guard,), 7.25, dtype=torch.float64).pin_memory()
        ub = torch.full((nu * F + 2 * guard,), 7.25, dtype=torch.float64).pin_memory()
        yb = torch.from_numpy(y.copy()).pin_memory()
        xp = C.cast(xb.data_ptr() + 8 * guard, P)
        up = C.cast(ub.data_ptr() + 8 * guard, P)
        so.api.check(N.lib().scenopt_dual_grad(cache.device(), C.cast(yb.data_ptr(), P), xp, up, 1))
        xs, us = xb.numpy(), ub.numpy()
        assert np.all(xs[:guard] == 7.25) and np.all(xs[guard + nx * n:] == 7.25)
        assert np.all(us[:guard] == 7.25) and np.all(us[guard + nu * F:] == 7.25)
        assert np.array_equal(xs[guard:guard + nx * n], ref.x.ravel(order="F"))
        assert np.array_equal(us[guard:guard + nu * F], ref.u.ravel(order="F"))


@pytest.mark.parametrize("shift", [1, 2])
def test_pinned_outputs_of_any_alignment(gpu, shift):
    """The forward pass writes mapped x / u rows with 16-byte stores, so zero
    copy needs 16-byte-aligned buffers: a pinned buffer shifted by one double
    (8-byte aligned) takes the copy path instead; both give the pageable
    path's bits and stay inside their buffers."""
    import ctypes as C

    import torch

    from paper_2107_01745_b200 import _native as N

    prob = so.gen_random_instance(2, 12, 6, 9, [3, 3, 2])
    cache = so.factor(prob)
    y = np.random.default_rng(4).uniform(-1, 1, prob.dual_dim)
    ref = so.dual_grad(cache, prob, y)
    nx, nu, n, F = prob.nx, prob.nu, prob.num_nodes(), prob.first_leaf
    guard = 64
    P = C.POINTER(C.c_double)
    xb = torch.full((nx * n + 2 * guard + 2,), 7.25, dtype=torch.float64).pin_memory()
    ub = torch.full((nu * F + 2 * guard + 2,), 7.25, dtype=torch.float64).pin_memory()
    yb = torch.from_numpy(y.copy()).pin_memory()
    off = guard + shift
    so.api.check(N.lib().scenopt_dual_grad(cache.device(), C.cast(yb.data_ptr(), P),
                                           C.cast(xb.data_ptr() + 8 * off, P), C.cast(ub.data_ptr() + 8 * off, P), 1))
    xs, us = xb.numpy(), ub.numpy()
    assert np.all(xs[:off] == 7.25) and np.all(xs[off + nx * n:] == 7.25)
    assert np.all(us[:off] == 7.25) and np.all(us[off + nu * F:] == 7.25)
    assert np.array_equal(xs[off:off + nx * n], ref.x.ravel(order="F"))
    assert np.array_equal(us[off:off + nu * F], ref.u.ravel(order="F"))


@pytest.mark.parametrize("flat", ["1", "0"])
def test_flattened_forward_top_matches_oracle_on_c3(gpu, monkeypatch, flat):
    """The forward top above the cut (stages 1..3 at C3) computed in one level
    from the ancestors' u_off with precomputed affine maps, against the
    oracle and against the per-stage chain (SCENOPT_FLAT_TOP=0)."""
    monkeypatch.setenv("SCENOPT_FLAT_TOP", flat)
    prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
    po = orc.Problem.from_flat(prob.flat())
    cache = so.factor(prob)
    assert cache.dev_info()["cut_stage"] == 4
    ofac = orc.Factor(po)
    rng = np.random.default_rng(11)
    y = rng.uniform(-1, 1, prob.dual_dim)
    r = rng.uniform(-1, 1, prob.dual_dim)
    for affine in (True, False):
        pts, hs = so.sweep(cache, [y, r], affine)
        for v, pt, h in ((y, pts[0], hs[0]), (r, pts[1], hs[1])):
            ox, ou = ofac.sweep(v, affine)
            assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < TOL
            Hx = orc.apply_H(po, ox, ou)
            assert np.abs(h - Hx).max() <= TOL * (1 + np.abs(Hx).max())


def test_mapped_host_outputs_are_bitwise_the_copied_ones(gpu):
    """Pinned (mapped) host buffers: the forward pass writes x / u over PCIe
    while it runs; pageable buffers get the copy after the sweep. Same bits,
    1 and 2 right-hand sides, affine and homogeneous."""
    import ctypes as C
    import torch
    prob = so.gen_random_instance(2, 12, 4, 6, [3, 2, 2])
    cache = so.factor(prob)
    dev = cache.device()
    lib = so.lib()
    f = prob.flat()
    nx, nu, n, F = prob.nx, prob.nu, prob.num_nodes(), prob.first_leaf
    P = C.POINTER(C.c_double)
    rng = np.random.default_rng(5)
    ys = [rng.uniform(-1, 1, prob.dual_dim) for _ in range(2)]

    def ptr(a):
        return C.cast(a.data_ptr(), P) if isinstance(a, torch.Tensor) else a.ctypes.data_as(P)

    for pinned in (False, True):
        mk = (lambda k: torch.zeros(k, dtype=torch.float64).pin_memory()) if pinned else (lambda k: np.zeros(k))
        # pinned inputs are read in place by the sweep (no H2D copy)
        yin = [torch.from_numpy(v).pin_memory() if pinned else v for v in ys]
        x1, u1 = mk(nx * n), mk(nu * F)
        so.api.check(lib.scenopt_dual_grad(dev, ptr(yin[0]), ptr(x1), ptr(u1), 1))
        X = [mk(nx * n), mk(nx * n)]
        U = [mk(nu * F), mk(nu * F)]
        Hs = [np.zeros(prob.dual_dim), np.zeros(prob.dual_dim)]
        so.api.check(lib.scenopt_dev_sweep(dev, 2, 0, (P * 2)(*[ptr(v) for v in yin]),
                                           (P * 2)(*[ptr(a) for a in X]), (P * 2)(*[ptr(a) for a in U]),
                                           (P * 2)(*[h.ctypes.data_as(P) for h in Hs]), 1))
        res = [np.asarray(a).copy() for a in (x1, u1, *X, *U, *Hs)]
        if not pinned:
            ref = res
    for a, b in zip(ref, res):
        assert np.array_equal(a, b)
    po = orc.Problem.from_flat(f)
    ox, ou = orc.Factor(po).dual_grad(ys[0])
    assert sup.rel_gap(ox, ou, res[0], res[1]) < 1e-9


@pytest.mark.parametrize("shape,item_kb", [((10, 5, 9, [2] * 7), 48), ((10, 5, 9, [2] * 7), 96),
                                           ((12, 4, 6, [2] * 6), 96)])
def test_oversized_staging_ring_falls_back_to_team_staging(gpu, monkeypatch, shape, item_kb):
    """Items of many small nodes whose staged vectors make the 12-deep
    producer staging ring larger than shared memory (found by
    tools/layout_fuzz.py: the fallback slot size used to wrap around in
    unsigned arithmetic, giving a negative slot and an illegal access). The
    layout must fall back to per-team staging and match the oracle."""
    monkeypatch.setenv("SCENOPT_ITEM_KB", str(item_kb))
    monkeypatch.setenv("SCENOPT_ITEM_MAX_NODES", "64")
    nx, nu, N, br = shape
    prob = so.gen_random_instance(3, nx, nu, N, br)
    po = orc.Problem.from_flat(prob.flat())
    cache = so.factor(prob)
    info = cache.dev_info()
    assert info["slot_bytes"] > 0
    ofac = orc.Factor(po)
    rng = np.random.default_rng(5)
    y, r = rng.uniform(-1, 1, prob.dual_dim), rng.uniform(-1, 1, prob.dual_dim)
    for affine in (True, False):
        pts, _ = so.sweep(cache, [y, r], affine)
        for v, pt in ((y, pts[0]), (r, pts[1])):
            ox, ou = ofac.sweep(v, affine)
            assert sup.rel_gap(ox, ou, pt.x.ravel(order="F"), pt.u.ravel(order="F")) < TOL


@pytest.mark.parametrize("shape", [(10, 5, 12, [4, 4, 4, 4]), (50, 20, 6, [8, 8]), (6, 3, 9, [3, 3, 3, 3])])
def test_sweep_geometries_are_bitwise_identical(gpu, monkeypatch, shape):
    """The six-producer geometry of the sweep kernel (picked for layouts of
    many-node items) differs from the default only in how vectors are staged:
    the consumer teams, and so every product's summation order, are the same,
    so both give the same bits for every sweep kind."""
    nx, nu, N, br = shape
    prob = so.gen_random_instance(7, nx, nu, N, br)
    rng = np.random.default_rng(11)
    y, r = rng.uniform(-1, 1, prob.dual_dim), rng.uniform(-1, 1, prob.dual_dim)
    out = {}
    for p in ("4", "6"):
        monkeypatch.setenv("SCENOPT_SWEEP_PRODUCERS", p)
        cache = so.factor(prob)
        assert cache.dev_info()["producer_warps"] == int(p)
        res = []
        for affine in (False, True):
            pts, hs = so.sweep(cache, [y, r], affine)
            res += [pts[0].x, pts[0].u, pts[1].x, pts[1].u, hs[0], hs[1]]
            pts1, hs1 = so.sweep(cache, [y], affine)
            res += [pts1[0].x, pts1[0].u, hs1[0]]
        for kind in ("minfbe", "nama"):  # the fused FB finish and the 2-RHS sweep in whole solves
            rep = so.api._solve_direct(kind, prob, cache, so.SolverConfig(nama_parallel_linesearch=kind == "nama"))
            assert rep.status == "converged"
            res += [rep.y, rep.x.x, rep.x.u, np.array([rep.iterations, rep.wall_ms * 0])]
        out[p] = res
    for a, b in zip(out["4"], out["6"]):
        assert np.array_equal(a, b)
    monkeypatch.delenv("SCENOPT_SWEEP_PRODUCERS")
    assert so.factor(prob).dev_info()["producer_warps"] == 4  # small trees keep the default geometry


def test_large_small_state_tree_takes_six_producers_bitwise(gpu, monkeypatch):
    """On a bandwidth-bound nx = 10 tree (873,813 nodes, 3.4 GB of packed
    matrices, items of up to 18 nodes) the default rule picks the
    six-producer geometry, and its sweeps equal the four-producer
    geometry's bit for bit (device factor, so no host factor is built)."""
    prob = so.gen_random_instance(1, 10, 5, 20, [4] * 8)
    rng = np.random.default_rng(3)
    y = rng.uniform(-1, 1, prob.dual_dim)
    out = {}
    for force in (None, "4"):
        if force:
            monkeypatch.setenv("SCENOPT_SWEEP_PRODUCERS", force)
        cache = so.factor_device(prob)
        info = cache.dev_info()
        assert info["producer_warps"] == (4 if force else 6), info["producer_warps"]
        pts, hs = so.sweep(cache, [y], True)
        out[force] = (pts[0].x, pts[0].u, hs[0])
        del cache
    for a, b in zip(out[None], out["4"]):
        assert np.array_equal(a, b)
