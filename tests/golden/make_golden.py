"""Generates tests/golden/golden_v1.npz from the CPU oracle.

The reference cannot be compiled here (Eigen is absent), so the goldens are
produced by the oracle restatement and cross-checked on generation against
the reference's own ground truth (dense KKT solve, tests/support.py) before
being written. They pin (a) the oracle against regressions and (b) the CUDA
path on the GPU box, where neither /root/reference nor the oracle build is
needed to read them.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from tests import support as sup  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def add_case(store, name, po, y, r, lam):
    f = po.flat()
    fac = orc.Factor(po)
    x, u = fac.dual_grad(y)
    kx, ku = sup.kkt_dual_grad(f, y)
    assert sup.rel_gap(kx, ku, x, u) < 1e-8, name
    x0, u0 = fac.hessian_vec(r)
    Hx = orc.apply_H(po, x, u)
    g = orc.Nonsmooth.from_problem(po)
    st = orc.fb_step(fac, g, y, lam)
    for k, v in f.items():
        store[f"{name}/inst/{k}"] = np.asarray(v)
    store[f"{name}/y"] = y
    store[f"{name}/r"] = r
    store[f"{name}/lam"] = np.array(lam)
    store[f"{name}/x"], store[f"{name}/u"], store[f"{name}/Hx"] = x, u, Hx
    store[f"{name}/x0"], store[f"{name}/u0"] = x0, u0
    for k in ("z", "R", "T"):
        store[f"{name}/fb_{k}"] = st[k]
    store[f"{name}/fb_scalars"] = np.array([st["fhat"], st["conj_T"], st["znorm_sq"], st["value"]])
    for kind, label in ((0, "minfbe"), (1, "nama")):
        rep = orc.solve(po, orc.SolverConfig(), kind)
        store[f"{name}/{label}_iters"] = np.array(rep["iterations"])
        store[f"{name}/{label}_counts"] = np.array([rep["dual_grad_calls"], rep["hessian_vec_calls"],
                                                   rep["prox_calls"], rep["conj_calls"]])
        store[f"{name}/{label}_y"] = rep["y"]
        store[f"{name}/{label}_x"] = rep["x"]
        store[f"{name}/{label}_lipschitz"] = np.array(rep["lipschitz_estimate"])


def main():
    store = {}
    po = orc.gen_random(1, 10, 5, 10, [2, 2, 2])  # BASELINE C1/C2 shape
    rng = np.random.default_rng(2107)
    D = po.dual_dim
    add_case(store, "c1", po, rng.uniform(-1, 1, D), rng.uniform(-1, 1, D), 0.05)
    orng = orc.Rng(4101)
    for t in range(4):
        opt = orc.InstanceOptions(with_box=True, with_l1=True, with_none=t % 2 == 1,
                                  feasible_boxes=True)
        p = orng.random_instance(orng.integer(2, 4), 30, orng.integer(2, 4), orng.integer(1, 3), opt)
        add_case(store, f"rt{t}", p, orng.vector(p.dual_dim, 2.0), orng.vector(p.dual_dim, 2.0), 0.3)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {os.path.getsize(OUT) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
