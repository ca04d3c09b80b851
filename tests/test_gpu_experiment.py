"""Experiment harness (experiment.hpp:22-283), the spring-mass benchmark
(generators.hpp:119-234) and the treebench CLI on the device solvers, against
the reference's own tests (test_experiment.cpp:38-203) and the CPU oracle's
solvers (iteration counts within +-1)."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

KIND = {"minfbe": 0, "nama": 1, "pnama": 1, "gpad": 2}


def random_batch(count, seed0=1):
    return [so.BatchEntry(f"r{seed0 + k}", so.gen_random_instance(seed0 + k)) for k in range(count)]


def row_of(rep, iid, solver):
    for r in rep.rows:
        if r.instance_id == iid and r.solver == solver:
            return r
    raise KeyError((iid, solver))


def test_single_run_emits_one_row_under_the_pinned_header(gpu):
    rep = so.run_experiment(random_batch(1), ["nama"], include_timing=False)
    assert len(rep.rows) == 1 and rep.rows[0].converged and rep.rows[0].error == ""
    csv = rep.csv()
    assert csv.count("\n") == 2 and csv.endswith("\n")
    assert csv.split("\n")[0] == so.RESULTS_CSV_HEADER
    assert "\nr1,nama," in csv


def test_reports_are_byte_deterministic_without_timing(gpu):
    a = so.run_experiment(random_batch(3), include_timing=False)
    b = so.run_experiment(random_batch(3), include_timing=False)
    assert a.csv() == b.csv() and a.traces_csv() == b.traces_csv() and a.summary_json() == b.summary_json()


def test_rows_match_the_oracle_solvers(gpu):
    cfg = so.SolverConfig(eps=1e-6)
    rep = so.run_experiment(random_batch(3), ["minfbe", "nama", "pnama", "gpad"], cfg, include_timing=False)
    for r in rep.rows:
        seed = int(r.instance_id[1:])
        orep = orc.solve(orc.gen_random(seed, 3, 2, 3, [2, 2, 2]), orc.SolverConfig(eps=1e-6), KIND[r.solver])
        assert r.converged and orep["status"] == 0
        assert abs(r.iterations - orep["iterations"]) <= 1, (r.instance_id, r.solver)


def test_newton_type_solvers_beat_the_baseline_median(gpu):
    rep = so.run_experiment(random_batch(6), solver=so.SolverConfig(eps=1e-6), include_timing=False)
    med = {}
    for s in rep.summaries():
        assert s.count == 6 and s.converged == 6
        med[s.solver] = s.median_calls
    assert 0 < med["nama"] < med["gpad"]


def test_summary_numbers_recompute_from_the_rows(gpu):
    rep = so.run_experiment(random_batch(5), ["minfbe"], include_timing=False)
    calls = sorted(r.oracle_calls() for r in rep.rows if r.converged)
    assert len(calls) == 5
    (s,) = rep.summaries()
    assert s.median_calls == calls[(len(calls) - 1) // 2] and s.p95_calls == calls[-1]
    assert s.frac_within_50 == sum(c <= 50 for c in calls) / 5.0 and s.fbe_violations == 0
    rep.metadata = {"generator": "random", "eps": 5e-4, "nested": {"b": [1, 2.5], "a": True}}
    text = rep.summary_json()
    j = json.loads(text)
    assert j["schema"] == "scenopt-runreport-v1" and j["metadata"]["nested"]["b"] == [1, 2.5]
    assert j["solvers"]["minfbe"]["median_oracle_calls"] == s.median_calls
    assert j["solvers"]["minfbe"]["count"] == 5
    assert '"metadata": {\n    "eps": 0.0005,\n    "generator": "random",\n    "nested": {\n      "a": true,' in text


def test_per_instance_failures_are_recorded_not_fatal(gpu):
    batch = random_batch(2)
    f = batch[0].prob.flat()
    R = f["R"].copy().reshape(-1, 2, 2)
    R[1:] = -1000.0 * np.eye(2)
    f["R"] = R.ravel()
    batch[0] = so.BatchEntry(batch[0].id, so.ProblemInstance.from_flat(f))
    for reuse in (True, False):
        rep = so.run_experiment(batch, ["nama"], include_timing=False, reuse_factors=reuse)
        assert len(rep.rows) == 2
        bad, good = row_of(rep, "r1", "nama"), row_of(rep, "r2", "nama")
        assert bad.error and not bad.converged
        assert good.error == "" and good.converged


def test_factor_reuse_leaves_the_results_unchanged(gpu):
    batch = []
    for k in range(3):
        par = so.SpringMassParams(horizon=2, root_state=np.full(4, 0.05 * (k + 1)))
        batch.append(so.BatchEntry(f"s{k}", so.gen_spring_mass(2, par)))
    assert so.factor_hash(batch[0].prob) == so.factor_hash(batch[2].prob)
    a = so.run_experiment(batch, include_timing=False, reuse_factors=True)
    b = so.run_experiment(batch, include_timing=False, reuse_factors=False)
    assert a.csv() == b.csv() and a.traces_csv() == b.traces_csv()


def test_trace_rows_cover_every_visited_iterate(gpu):
    rep = so.run_experiment(random_batch(2), ["gpad"], include_timing=False)
    expected = 1
    for r in rep.rows:
        assert r.converged and len(r.residual_trace) == r.iterations + 1
        expected += len(r.residual_trace)
    assert rep.traces_csv().count("\n") == expected


def test_parallel_linesearch_column_reproduces_serial_nama(gpu):
    rep = so.run_experiment(random_batch(3), ["nama", "pnama"], include_timing=False)
    for k in range(3):
        s, p = row_of(rep, f"r{k + 1}", "nama"), row_of(rep, f"r{k + 1}", "pnama")
        assert s.iterations == p.iterations and s.oracle_calls() == p.oracle_calls()
        assert s.final_residual_inf == p.final_residual_inf


def test_envelope_monotonicity_holds_across_the_batch(gpu):
    rep = so.run_experiment(random_batch(4), ["minfbe", "nama"], include_timing=False)
    assert all(s.fbe_violations == 0 for s in rep.summaries())


@pytest.mark.parametrize("kind", ["minfbe", "nama", "gpad"])
def test_spring_mass_benchmark_matches_the_oracle(gpu, kind):
    """The paper's benchmark instance (5 masses, 4095 nodes) from sampled
    initial states, preconditioned as treebench runs it."""
    par = so.SpringMassParams()
    states = so.sample_initial_state(5, par, seed=1, count=3)
    for x0 in states:
        p = so.SpringMassParams(root_state=x0)
        prob = so.gen_spring_mass(5, p)
        po = orc.gen_spring_mass(5, p)
        cfg = so.SolverConfig(precondition=True)
        rep = so.solve(prob, cfg, kind)
        orep = orc.solve(po, orc.SolverConfig(precondition=True), KIND[kind])
        assert rep.status == ("converged" if orep["status"] == 0 else "max_iters_exceeded")
        assert rep.verified == bool(orep["verified"])
        assert abs(rep.iterations - orep["iterations"]) <= 1, (rep.iterations, orep["iterations"])
        scale = 1 + np.abs(orep["x"]).max()
        assert np.abs(rep.x.x.ravel(order="F") - orep["x"]).max() <= 10 * cfg.eps * scale


@pytest.mark.parametrize("kind", ["minfbe", "nama", "gpad"])
def test_spring_mass_study_variant_matches_the_oracle(gpu, kind):
    """The `both` variant of profiles/spring_mass_study_r02.md (positions in
    +-velocity_bound/2, termination on the preconditioned problem's own
    residual) through the device solvers: the oracle's iteration counts."""
    par = so.SpringMassParams(horizon=8)
    states = so.sample_initial_state(5, par, seed=1, count=3)
    for x0 in states:
        x0 = x0 * np.r_[np.full(5, 0.5), np.ones(5)]
        p = so.SpringMassParams(horizon=8, root_state=x0)
        scaled = so.precondition(so.gen_spring_mass(5, p))
        rep = so.api._solve_direct(kind, scaled, so.factor(scaled), so.SolverConfig())
        pre = orc.gen_spring_mass(5, p).precondition()
        orep = orc.solve_direct(pre, orc.Factor(pre), orc.SolverConfig(), KIND[kind])
        assert rep.status == "converged" and orep["status"] == 0
        assert abs(rep.iterations - orep["iterations"]) <= 1, (rep.iterations, orep["iterations"])


def _treebench():
    return os.path.join(os.path.dirname(so._native.LIB_PATH), "..", "bin", "treebench")


def test_treebench_solve_and_bench(gpu, tmp_path):
    exe = _treebench()
    assert subprocess.run([exe, "gen", "spring-mass", "--masses", "3", "--horizon", "4", "--sample-seed", "2",
                           "--out", str(tmp_path / "s.json")]).returncode == 0
    r = subprocess.run([exe, "solve", str(tmp_path / "s.json"), "--solver", "pnama", "--precondition",
                        "--out", str(tmp_path / "rep.json")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    j = json.loads((tmp_path / "rep.json").read_text())
    assert j["schema"] == "scenopt-solvereport-v1" and j["status"] == "converged" and j["verified"]
    assert j["solver"] == "pnama" and len(j["residual_trace"]) == j["iterations"] + 1
    assert len(j["root_control"]) == 2
    assert j["oracle_calls"]["total"] == j["oracle_calls"]["dual_grad"] + j["oracle_calls"]["hessian_vec"]
    out = tmp_path / "bench"
    r = subprocess.run([exe, "bench", "spring-mass", "--samples", "4", "--horizon", "4", "--masses", "3",
                        "--no-timing", "--out", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "minfbe: 4/4 converged" in r.stdout
    csv = (out / "results.csv").read_text().splitlines()
    assert csv[0] == so.RESULTS_CSV_HEADER and len(csv) == 1 + 4 * 3
    s = json.loads((out / "summary.json").read_text())
    assert s["metadata"]["generator"] == "spring-mass" and s["metadata"]["samples"] == 4
    assert set(s["solvers"]) == {"minfbe", "nama", "gpad"}
    # byte-stable without timing
    out2 = tmp_path / "bench2"
    subprocess.run([exe, "bench", "spring-mass", "--samples", "4", "--horizon", "4", "--masses", "3",
                    "--no-timing", "--out", str(out2)], capture_output=True, check=True)
    for name in ("results.csv", "traces.csv", "summary.json"):
        assert (out / name).read_bytes() == (out2 / name).read_bytes()
