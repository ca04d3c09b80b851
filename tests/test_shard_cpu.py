"""Host logic of subtree sharding over world_size 2 on CPU
(gloo): both ranks derive the same shard plan from the C-ABI
(scenopt_shard_plan, host-only), their node sets partition the tree below
the shard stage with the top replicated, and the row ownership the library
uses (scenopt_shard_rows) is that partition. On the oracle's vectors: the
gathers of sharded results (sum-allreduce of disjoint row sets, top on rank
0) reassemble the full x, u and Hx exactly; the sweep's exchange of the
shard-stage dual rows gives every rank all of them; and a dual-kernel
reduction done the sharded way (partial sums over counted rows, allgather,
rank-order combine) gives every rank the same bits, equal to the full sum."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(2, 6, 3, 9, [3, 1, 4, 2], -1), (3, 5, 2, 8, [2, 2, 2, 2, 2], 3), (4, 4, 2, 6, [5, 3], 2)]


def _owned(flat, stage, lo, hi, rank):
    """Node mask of one rank: its shard-stage subtrees, plus the top on rank 0."""
    n = flat["num_nodes"]
    so_ = flat["stage_offsets"]
    anc = flat["ancestor"]
    mine = np.zeros(n, bool)
    mine[: so_[stage]] = rank == 0
    mine[lo:hi] = True
    for c in range(so_[stage + 1], n):
        mine[c] = mine[anc[c]]
    return mine


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2107_01745_b200 as so
        from oracle import oracle as orc
        for seed, nx, nu, N, br, stage in CASES:
            prob = so.gen_random_instance(seed, nx, nu, N, br)
            flat = prob.flat()
            st = C.c_int32()
            bounds = (C.c_int32 * (world + 1))()
            so.api.check(so.lib().scenopt_shard_plan(prob._h, world, stage, C.byref(st), bounds))
            plan = (st.value, list(bounds))
            allp = [None] * world
            dist.all_gather_object(allp, plan)
            assert all(p == plan for p in allp), allp
            s, b = plan
            so_ = flat["stage_offsets"]
            assert b[0] == so_[s] and b[-1] == so_[s + 1] and all(b[i] < b[i + 1] for i in range(world))
            mine = _owned(flat, s, b[rank], b[rank + 1], rank)
            # every node is owned exactly once (top on rank 0 only)
            cnt = torch.tensor(mine.astype(np.int64))
            dist.all_reduce(cnt)
            assert (cnt.numpy() == 1).all()
            # the oracle's sweep outputs, rank-local parts summed == full
            po = orc.Problem.from_flat(flat)
            fac = orc.Factor(po)
            y = np.random.default_rng(seed).uniform(-1, 1, prob.dual_dim)
            ox, ou = fac.sweep(y, True)
            hx = orc.apply_H(po, ox, ou)
            X = ox.reshape(-1, nx)          # node-major columns of the reference's nx x n
            U = ou.reshape(-1, nu)
            F = flat["stage_offsets"][N]
            rows = np.zeros(prob.dual_dim, bool)
            doff = np.concatenate([[0], np.cumsum(flat["stage_rows"][1:])])
            for c in range(1, flat["num_nodes"]):
                if mine[c]:
                    rows[doff[c - 1]: doff[c - 1] + flat["stage_rows"][c]] = True
            toff = doff[-1] + np.concatenate([[0], np.cumsum(flat["terminal_rows"])])
            for l in range(flat["num_nodes"] - F):
                if mine[F + l]:
                    rows[toff[l]: toff[l + 1]] = True
            for full, mask in ((hx, rows), (X, mine[:, None]), (U, mine[:F, None])):
                part = torch.from_numpy(np.where(mask, full, 0.0))
                dist.all_reduce(part)
                assert np.array_equal(part.numpy(), full)
            # the library's own row ownership (scenopt_shard_rows) is this mask
            counted = np.zeros(prob.dual_dim, np.uint8)
            so.api.check(so.lib().scenopt_shard_rows(prob._h, world, stage, rank,
                                                     counted.ctypes.data_as(C.POINTER(C.c_uint8))))
            assert np.array_equal(counted.astype(bool), rows)
            # the sweep's exchange also carries the shard-stage nodes' dual rows:
            # owners write theirs, the sum is every rank's copy of those rows
            lo_s, hi_s = so_[s], so_[s + 1]
            r0, r1 = doff[lo_s - 1], doff[hi_s - 1]
            ysec = np.where(rows[r0:r1], y[r0:r1], 0.0)
            t = torch.from_numpy(ysec.copy())
            dist.all_reduce(t)
            assert np.array_equal(t.numpy(), y[r0:r1])
            # a dual-kernel reduction: each rank's partial sums over its counted
            # rows (the FB step's conj / |z|^2 / <Hx,R> / |R|^2, and max |R|),
            # allgathered and combined in rank order -- the same bits on
            # every rank, equal to the full reduction
            g = orc.Nonsmooth.from_problem(po)
            st_ = orc.fb_step(fac, g, y, 0.37)
            z, R, T = st_["z"], st_["R"], st_["T"]
            conj_rows = np.array([g.conj(np.where(np.arange(len(T)) == i, T, 0.0)) for i in range(len(T))])
            terms = np.stack([conj_rows, z * z, st_["Hx"] * R, R * R])
            part = np.concatenate([np.where(rows, terms, 0.0).sum(axis=1), [np.abs(np.where(rows, R, 0.0)).max()]])
            gathered = [torch.zeros(5, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(part))
            tot = gathered[0].numpy().copy()
            for q in range(1, world):
                tot[:4] += gathered[q].numpy()[:4]
                tot[4] = max(tot[4], gathered[q].numpy()[4])
            every = [torch.zeros(5, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(every, torch.from_numpy(tot))
            assert all(np.array_equal(e.numpy(), tot) for e in every)
            full = np.concatenate([terms.sum(axis=1), [np.abs(R).max()]])
            assert np.allclose(tot, full, rtol=1e-12, atol=1e-12)
            assert tot[0] == pytest.approx(st_["conj_T"], rel=1e-12, abs=1e-12)
        out.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        out.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_plan_and_exchange_over_two_gloo_ranks(_built_libraries):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
