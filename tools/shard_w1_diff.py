"""Diagnostic: world-1 sharded handle (NCCL, phased dual kernels) against the
unsharded handle, operation by operation; prints the first mismatch."""
import numpy as np

import paper_2107_01745_b200 as so

prob = so.gen_random_instance(5, 6, 3, 8, [3, 3, 2])
full = so.factor(prob)
shard = so.factor(prob)
shard.shard(0, 1, so.nccl_unique_id(), 0, -1)
rng = np.random.default_rng(1)
y = rng.uniform(-1, 1, prob.dual_dim)


def cmp(name, a, b):
    a, b = np.asarray(a), np.asarray(b)
    eq = np.array_equal(a, b)
    print(f"{name:28s} {'bitwise' if eq else 'DIFF max %.3e' % np.abs(a - b).max()}")


L1 = so.estimate_dual_lipschitz(full, prob)
L2 = so.estimate_dual_lipschitz(shard, prob)
cmp("lipschitz", L1[0], L2[0])
pf, hf = so.sweep(full, [y], True)
ps, hs = so.sweep(shard, [y], True)
cmp("sweep Hx", hf[0], hs[0])
cmp("sweep x", pf[0].x, ps[0].x)
a = so.fb_step(full, prob, y, 0.1)
b = so.fb_step(shard, prob, y, 0.1)
for f in ("Hx", "z", "R", "T"):
    cmp("fb_step " + f, getattr(a, f), getattr(b, f))
cmp("fb_step scalars", [a.fhat, a.conj_T, a.znorm_sq, a.value], [b.fhat, b.conj_T, b.znorm_sq, b.value])
cmp("fbe_grad", so.fbe_grad(a, full, prob), so.fbe_grad(b, shard, prob))
cmp("fhat_value", so.fhat_value(full, prob, y), so.fhat_value(shard, prob, y))
for kind in ("minfbe", "nama"):
    for it in (1, 2, 3, 5, 8, 1000):
        cfg = so.SolverConfig(max_iters=it, lambda0=0.9 / L1[0], nama_parallel_linesearch=(kind == "nama"))
        ra = so.api._solve_direct(kind, prob, full, cfg)
        rb = so.api._solve_direct(kind, prob, shard, cfg)
        cmp(f"{kind} iters<={it} y", ra.y, rb.y)
        cmp(f"{kind} iters<={it} trace", ra.residual_trace, rb.residual_trace)
