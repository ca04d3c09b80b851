"""Speculative next-iteration work in MINFBE / NAMA (solver.cpp, DESIGN.md
§5): the sweeps and L-BFGS launch enqueued behind fb_finish's skip word
change scheduling only. On instances where lambda is halved (both
backtracking rules, so speculative work is discarded and the L-BFGS buffer
cleared after a speculative push), solves with speculation on must equal
the same solves with SCENOPT_SPEC_HR=0 bitwise, and match the oracle."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"minfbe": 0, "nama": 1}
RULE = {"original": 0, "simple": 1}

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2107_01745_b200 as so
cases = json.load(open(sys.argv[2]))
out = []
for c in cases:
    z = np.load(c["npz"])
    prob = so.ProblemInstance.from_flat({k: (z[k].item() if z[k].ndim == 0 else z[k]) for k in z.files})
    cfg = so.SolverConfig(backtracking_rule=["original", "simple"][c["rule"]], lambda0=c["lambda0"], eps=1e-6)
    rep = so.solve_minfbe(prob, so.factor(prob), cfg) if c["kind"] == "minfbe" else \
        so.solve_nama(prob, so.factor(prob), cfg)
    np.save(c["npz"] + ".y.npy", rep.y)
    out.append([rep.iterations, rep.lambda_final, rep.stats.dual_grad_calls, rep.stats.hessian_vec_calls])
json.dump(out, open(sys.argv[3], "w"))
"""


def _cases(tmp_path):
    rng = orc.Rng(4242)
    cases = []
    for kind in ("minfbe", "nama"):
        for rule in ("simple", "original"):
            while True:  # active constraints, so lambda halvings matter
                po = rng.random_instance(3, 40, 3, 2, orc.InstanceOptions(with_box=True, with_l1=True,
                                                                          with_none=True, feasible_boxes=True))
                if orc.solve(po, orc.SolverConfig(), 0)["iterations"] > 2:
                    break
            lip = sup.dual_lipschitz_dense(orc.Factor(po))
            path = str(tmp_path / f"{kind}_{rule}.npz")
            np.savez(path, **po.flat())
            cases.append(dict(kind=kind, rule=RULE[rule], lambda0=10.0 / lip, npz=path, po=po))
    return cases


def test_speculation_is_bitwise_neutral_and_matches_oracle(gpu, tmp_path):
    cases = _cases(tmp_path)
    spec_file, res_file = tmp_path / "cases.json", tmp_path / "res.json"
    json.dump([{k: v for k, v in c.items() if k != "po"} for c in cases], open(spec_file, "w"))
    env = dict(os.environ, SCENOPT_SPEC_HR="0")
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(spec_file), str(res_file)], env=env, check=True,
                   timeout=600)
    ref = json.load(open(res_file))
    halved = 0
    for c, r in zip(cases, ref):
        prob = so.ProblemInstance.from_flat(c["po"].flat())
        cfg = so.SolverConfig(backtracking_rule=["original", "simple"][c["rule"]], lambda0=c["lambda0"], eps=1e-6)
        solve = so.solve_minfbe if c["kind"] == "minfbe" else so.solve_nama
        rep = solve(prob, so.factor(prob), cfg)
        y_off = np.load(c["npz"] + ".y.npy")
        assert [rep.iterations, rep.lambda_final, rep.stats.dual_grad_calls,
                rep.stats.hessian_vec_calls] == r, (c["kind"], c["rule"])
        assert np.array_equal(rep.y, y_off), (c["kind"], c["rule"])
        halved += rep.lambda_final < c["lambda0"]
        oc = orc.SolverConfig(backtracking_rule=c["rule"], lambda0=c["lambda0"], eps=1e-6)
        orep = orc.solve_direct(c["po"], orc.Factor(c["po"]), oc, KIND[c["kind"]])
        assert rep.lambda_final == orep["lambda_final"]
        assert abs(rep.iterations - orep["iterations"]) <= 1
    assert halved >= 2
