"""Golden fixtures (tests/golden/golden_v1.npz, made by make_golden.py from
the oracle and cross-checked against the dense KKT ground truth): the CPU
oracle must reproduce them, and the CUDA path must match them on the GPU."""
import os

import numpy as np
import pytest

from tests import support as sup

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")
CASES = ["c1", "rt0", "rt1", "rt2", "rt3"]


def load():
    z = np.load(GOLD)
    out = {}
    for key in z.files:
        name, rest = key.split("/", 1)
        out.setdefault(name, {})[rest] = z[key]
    for name, d in out.items():
        inst = {k[5:]: d[k] for k in list(d) if k.startswith("inst/")}
        for k in ("nx", "nu", "num_stages", "num_nodes"):
            inst[k] = int(inst[k])
        d["flat"] = inst
    return out


G = load()


def close(a, b, tol):
    return np.abs(np.asarray(a) - np.asarray(b)).max(initial=0.0) <= tol * (1 + np.abs(b).max(initial=0.0))


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_golden(name):
    from oracle import oracle as orc

    d = G[name]
    po = orc.Problem.from_flat(d["flat"])
    fac = orc.Factor(po)
    x, u = fac.dual_grad(d["y"])
    assert close(x, d["x"], 1e-12) and close(u, d["u"], 1e-12)
    x0, u0 = fac.hessian_vec(d["r"])
    assert close(x0, d["x0"], 1e-12) and close(u0, d["u0"], 1e-12)
    kx, ku = sup.kkt_dual_grad(d["flat"], d["y"])
    assert sup.rel_gap(kx, ku, d["x"], d["u"]) < 1e-8
    rep = orc.solve(po, orc.SolverConfig(), 0)
    assert rep["iterations"] == int(d["minfbe_iters"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_cuda_path_matches_golden(gpu, name):
    import paper_2107_01745_b200 as so

    d = G[name]
    prob = so.ProblemInstance.from_flat(d["flat"])
    cache = so.factor(prob)
    pt = so.dual_grad(cache, prob, d["y"])
    assert sup.rel_gap(d["x"], d["u"], pt.x.ravel(order="F"), pt.u.ravel(order="F")) < 1e-9
    h = so.hessian_vec(cache, prob, d["r"])
    assert sup.rel_gap(d["x0"], d["u0"], h.x.ravel(order="F"), h.u.ravel(order="F")) < 1e-9
    st = so.fb_step(cache, prob, d["y"], float(d["lam"]))
    for k in ("z", "R", "T"):
        assert close(getattr(st, k), d[f"fb_{k}"], 1e-9), k
    sc = d["fb_scalars"]
    for v, ref in zip((st.fhat, st.conj_T, st.znorm_sq, st.value), sc):
        assert abs(v - ref) <= 1e-9 * (1 + abs(ref))
    for label in ("minfbe", "nama"):
        rep = so.solve(prob, so.SolverConfig(), label)
        assert abs(rep.iterations - int(d[f"{label}_iters"])) <= 1
        assert rep.lipschitz_estimate == pytest.approx(float(d[f"{label}_lipschitz"]), rel=1e-9)
        assert np.abs(rep.y - d[f"{label}_y"]).max() <= 10 * 5e-4 * (1 + np.abs(d[f"{label}_y"]).max())
