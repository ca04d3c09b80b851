"""Spring-mass benchmark (PAPER §IV-A; reference treebench `bench spring-mass`)
under the reference code and single-change variants, on the CPU oracle, to
locate what separates the code's numbers from the paper's (84 % of
MINFBE / NAMA runs within 50 oracle calls, GPAD median 188).

Variants (one change each against the reference code path):
  ref       generators.hpp:223-233 sampling (positions +-velocity_bound,
            velocities +-velocity_bound/2), precondition on
            (treebench.cpp:196-198), residual ||R / sqrt(pi)||_inf
            (solvers.hpp:117-120, 677-688)
  halfpos   positions +-velocity_bound/2 (the doc comment of
            sample_initial_state: every component within half the bound)
  scaledres precondition on, termination on the scaled problem's own
            residual ||R_scaled||_inf = ||sqrt(pi) R||_inf (no weight)
  both      halfpos + scaledres
usage: python tools/spring_mass_study.py [HORIZON] [SAMPLES] > profiles/spring_mass_study_r02.md"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S = int(sys.argv[2]) if len(sys.argv) > 2 else 50
M = 5
KIND = {"minfbe": 0, "nama": 1, "gpad": 2}


class Par:
    def __init__(self, horizon, root=None):
        self.horizon = horizon
        self.root_state = root


def states(half_positions):
    x = orc.sample_initial_states(M, Par(H), seed=1, count=S).reshape(S, 2 * M)
    if half_positions:  # the same draws, positions scaled from +-5 to +-2.5
        x = x.copy()
        x[:, :M] *= 0.5
    return x


def run(variant):
    half = variant in ("halfpos", "both")
    scaled = variant in ("scaledres", "both")
    rows = {k: [] for k in KIND}
    for x0 in states(half):
        prob = orc.gen_spring_mass(M, Par(H, x0))
        for kind, code in KIND.items():
            cfg = orc.SolverConfig(eps=5e-4, memory=5)
            if scaled:
                pre = prob.precondition()
                rep = orc.solve_direct(pre, orc.Factor(pre), cfg, code)
            else:
                cfg.precondition = True
                rep = orc.solve(prob, cfg, code)
            calls = rep["dual_grad_calls"] + rep["hessian_vec_calls"]
            rows[kind].append((rep["status"] == 0, calls))
    out = {}
    for kind, r in rows.items():
        calls = [c for ok, c in r if ok]
        out[kind] = dict(conv=sum(ok for ok, _ in r), median=statistics.median(calls) if calls else None,
                         within50=100.0 * sum(ok and c <= 50 for ok, c in r) / len(r))
    return out


print(f"# Spring-mass study: M = {M} masses, N = {H} ({2 ** (H + 1) - 1} nodes), {S} samples, eps 5e-4, "
      "memory 5, CPU oracle\n")
print("| variant | solver | converged | median calls | within 50 calls | GPAD median / NAMA median |")
print("|---|---|---|---|---|---|")
for v in ("ref", "halfpos", "scaledres", "both"):
    r = run(v)
    ratio = r["gpad"]["median"] / r["nama"]["median"] if r["gpad"]["median"] and r["nama"]["median"] else None
    for kind in KIND:
        q = r[kind]
        print(f"| {v} | {kind} | {q['conv']}/{S} | {q['median']} | {q['within50']:.0f}% | "
              f"{'' if kind != 'gpad' or ratio is None else f'{ratio:.2f}'} |", flush=True)
