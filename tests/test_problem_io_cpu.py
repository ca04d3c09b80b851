"""Problem files (problem_io.hpp:18-559) against the
reference's own tests (test_io.cpp:12-162): canonical round trips, the
shared / per-node field forms, markov tree specs, malformed documents,
validation messages, content / factor hashes and the filesystem round trip.
Host-only: the JSON reader / writer is native library code with no device
work."""
import json
import os

import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

# test_io.cpp:12-28
CHAIN_FILE = r'''{
  "schema": "scenopt-problem-v1",
  "dims": {"nx": 2, "nu": 1},
  "root_state": [0.25, -0.5],
  "tree": {"stage": [0, 1, 2], "ancestor": [-1, 0, 1],
           "probability": [1.0, 1.0, 1.0]},
  "dynamics": {"A": [[0.9, 0.1], [0.0, 0.8]], "B": [[0.5], [1.0]],
               "c": [0.0, 0.0]},
  "cost": {"Q": [[1.0, 0.0], [0.0, 1.0]], "R": [[1.0]], "S": [[0.0, 0.0]],
           "q": [0.0, 0.0], "r": [0.0]},
  "constraints": {"F": [[1.0, 0.0]], "G": [[1.0]], "kind": "box",
                  "zmin": [[-1.0], [-2.0]], "zmax": [[1.0], [2.0]],
                  "gamma": 0.0},
  "terminal_cost": {"P": [[1.0, 0.0], [0.0, 1.0]], "p": [0.0, 0.0]},
  "terminal_constraints": {"F": [[0.0, 1.0]], "kind": "box",
                           "zmin": [-1.0], "zmax": [1.0], "gamma": 0.0}
}'''


def test_serialization_is_canonical_and_round_trips_byte_identically():
    for prob in (so.gen_random_instance(7), so.gen_spring_mass(3, so.SpringMassParams(horizon=3))):
        first = so.serialize_problem(prob)
        again = so.parse_problem(first)
        assert so.serialize_problem(again) == first
        assert first.endswith("}\n") and json.loads(first)["schema"] == "scenopt-problem-v1"
        # the parsed copy is the same instance, bit for bit, modes included
        a, b = prob.flat(), again.flat()
        for k in a:
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
        assert np.array_equal(prob.mode(), again.mode())


def test_layout_matches_nlohmann_dump():
    """dump(2): sorted keys, 2-space indent, nlohmann's float placement."""
    doc = json.loads(CHAIN_FILE)
    doc["root_state"] = [1e-05, 1e15]
    text = so.serialize_problem(so.problem_from_json(doc))
    assert list(json.loads(text)) == sorted(json.loads(text))
    assert text.startswith('{\n  "constraints": {\n    "F": [\n      [\n        1.0,\n        0.0\n      ]\n    ],')
    assert '"root_state": [\n    1e-05,\n    1e+15\n  ],' in text
    assert '"dims": {\n    "nu": 1,\n    "nx": 2\n  },' in text
    assert '"stage": [\n      0,\n      1,\n      2\n    ]' in text
    # number placement rules (dtoa_impl::format_buffer, min_exp -4, max_exp 15)
    for v, tok in ((0.25, "0.25"), (-0.0, "-0.0"), (123.0, "123.0"), (0.0001, "0.0001"),
                   (1.5e300, "1.5e+300"), (123456789012345.6, "123456789012345.6"),
                   (1234567890123456.0, "1.234567890123456e+15"), (5e-324, "5e-324"),
                   (0.1, "0.1"), (-2.5e-7, "-2.5e-07")):
        doc["root_state"] = [v, 0.0]
        t = so.serialize_problem(so.problem_from_json(doc))
        assert f'"root_state": [\n    {tok},\n' in t, (v, tok)
        assert so.serialize_problem(so.parse_problem(t)) == t


def test_shared_fields_broadcast_to_every_node():
    prob = so.parse_problem(CHAIN_FILE)  # test_io.cpp:63-78
    f = prob.flat()
    assert f["num_nodes"] == 3 and f["num_nodes"] - f["stage_offsets"][2] == 1
    assert list(f["root_state"]) == [0.25, -0.5]
    A1, A2 = sup.node_mat(f, "A", 1, 2, 2), sup.node_mat(f, "A", 2, 2, 2)
    assert np.array_equal(A1, A2) and A1[0, 0] == 0.9
    lay = orc.layout(f)
    assert f["zmin"][lay["dual_offset"][1]] == -1.0 and f["zmin"][lay["dual_offset"][2]] == -2.0
    assert f["zmax"][lay["dual_offset"][2]] == 2.0
    assert f["tg_kind"][0] == 1
    assert prob.validate() == []
    assert len(prob.mode()) == 0  # arrays without "mode": none recorded


def test_markov_tree_spec_parses_to_the_built_tree():
    prob = so.gen_spring_mass(2, so.SpringMassParams(horizon=2))  # test_io.cpp:80-92
    doc = so.problem_to_json(prob)
    doc["tree"] = {"markov": {"transition": [[0.1, 0.9], [0.9, 0.1]], "initial": [0.5, 0.5], "horizon": 2}}
    assert so.serialize_problem(so.problem_from_json(doc)) == so.serialize_problem(prob)
    bad = dict(doc)
    bad["tree"] = {"markov": {"transition": [[0.5, 0.6], [0.5, 0.5]], "initial": [0.5, 0.5], "horizon": 2}}
    with pytest.raises(so.ParseError, match="tree.markov: build_from_markov: transition row 0"):
        so.problem_from_json(bad)


def test_malformed_documents_are_rejected_with_messages():
    with pytest.raises(so.ParseError, match="not valid JSON"):  # test_io.cpp:94-125
        so.parse_problem("not json at all")
    with pytest.raises(so.ParseError, match='missing key "schema"'):
        so.parse_problem("{}")
    base = json.loads(CHAIN_FILE)
    cases = [
        ("schema", "something-else", "schema must be"),
        ("dynamics", None, 'missing key "dynamics"'),
    ]
    for key, val, msg in cases:
        doc = json.loads(CHAIN_FILE)
        if val is None:
            del doc[key]
        else:
            doc[key] = val
        with pytest.raises(so.ParseError, match=msg):
            so.problem_from_json(doc)
    doc = json.loads(CHAIN_FILE)
    doc["dynamics"]["A"] = [[1.0, 0.0], [0.0]]
    with pytest.raises(so.ParseError, match="ragged matrix rows"):
        so.problem_from_json(doc)
    doc = json.loads(CHAIN_FILE)
    doc["dynamics"]["B"] = [[0.5]]  # B has too few rows: an invalid instance
    with pytest.raises(so.ParseError) as e:
        so.problem_from_json(doc)
    assert "node 1" in str(e.value) and "instance validation failed" in str(e.value)
    doc = json.loads(CHAIN_FILE)
    doc["constraints"]["zmax"] = [-3.0]  # shared box with zmin > zmax on node 1
    with pytest.raises(so.ParseError, match="node 1 stage block: box needs zmin <= zmax"):
        so.problem_from_json(doc)
    doc = json.loads(CHAIN_FILE)
    doc["tree"]["stage"] = [0, 1.0, 2]
    with pytest.raises(so.ParseError, match="tree.stage: entries must be integers"):
        so.problem_from_json(doc)
    doc = json.loads(CHAIN_FILE)
    doc["constraints"]["kind"] = "ellipse"
    with pytest.raises(so.ParseError, match='unknown kind "ellipse"'):
        so.problem_from_json(doc)
    doc = json.loads(CHAIN_FILE)
    doc["dynamics"]["c"] = [[0.0, 0.0]] * 3  # a per-node list of the wrong length
    with pytest.raises(so.ParseError, match="expected one shared value or a list of 2"):
        so.problem_from_json(doc)


def test_per_node_lists_and_mixed_kinds_round_trip():
    rng = orc.Rng(77)
    po = rng.random_instance(3, 14, 3, 2, orc.InstanceOptions(with_box=True, with_l1=True, with_none=True))
    prob = so.ProblemInstance.from_flat(po.flat())
    text = so.serialize_problem(prob)
    doc = json.loads(text)
    assert isinstance(doc["constraints"]["kind"], list) and isinstance(doc["dynamics"]["A"][0][0], list)
    back = so.parse_problem(text)
    assert so.serialize_problem(back) == text
    a, b = prob.flat(), back.flat()
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_document_validation_lists_violations_without_throwing():
    assert so.validate_problem_text(CHAIN_FILE) == []  # test_io.cpp:127-133
    assert so.validate_problem_text('{"schema": 3}')
    assert so.validate_problem_text("[1, 2")
    doc = json.loads(CHAIN_FILE)
    doc["tree"]["probability"] = [1.0, 0.5, 1.0]
    msgs = so.validate_problem_text(json.dumps(doc))
    assert msgs[0] == "instance validation failed" and any("node 1" in m for m in msgs[1:])


def test_content_and_factor_hashes_separate_what_the_cache_depends_on():
    base = so.gen_random_instance(5)  # test_io.cpp:135-151
    flat = base.flat()

    def variant(**kw):
        f = dict(flat)
        f.update(kw)
        p = so.ProblemInstance.from_flat(f)
        p.set_mode(base.mode())
        return p

    moved = variant(root_state=np.full(base.nx, 0.01))
    assert so.content_hash(moved) != so.content_hash(base)
    assert so.factor_hash(moved) == so.factor_hash(base)
    zmax = flat["zmax"].copy()
    zmax[0] += 1.0
    loosened = variant(zmax=zmax)
    assert so.content_hash(loosened) != so.content_hash(base)
    assert so.factor_hash(loosened) == so.factor_hash(base)
    A = flat["A"].copy()
    A[base.nx * base.nx] += 0.125  # node 1, A(0, 0)
    assert so.factor_hash(variant(A=A)) != so.factor_hash(base)
    assert so.content_hash(base) == so.content_hash(so.gen_random_instance(5))
    # the hash is FNV-1a of the canonical text (problem_io.hpp:527-541)
    h = 1469598103934665603
    for b in so.serialize_problem(base).encode():
        h = ((h ^ b) * 1099511628211) % (1 << 64)
    assert h == so.content_hash(base)


def test_problem_files_survive_the_filesystem_round_trip(tmp_path):
    prob = so.gen_random_instance(13)  # test_io.cpp:153-162
    path = tmp_path / "io_roundtrip.json"
    so.save_problem(prob, path)
    assert so.serialize_problem(so.load_problem(path)) == so.serialize_problem(prob)
    with pytest.raises(so.ParseError):
        so.load_problem(tmp_path / "definitely_missing_dir" / "x.json")


def test_treebench_cli_generates_and_validates(tmp_path):
    """tools/treebench.cpp: gen / validate without a GPU; exit codes 0 / 1 / 2."""
    import subprocess
    exe = os.path.join(os.path.dirname(so._native.LIB_PATH), "..", "bin", "treebench")
    r = subprocess.run([exe, "gen", "random", "--seed", "3", "--horizon", "2", "--out", str(tmp_path / "r.json")],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "dual dimension" in r.stdout
    assert so.serialize_problem(so.load_problem(tmp_path / "r.json")) == so.serialize_problem(
        so.gen_random_instance(3, horizon=2))
    r = subprocess.run([exe, "gen", "spring-mass", "--masses", "3", "--horizon", "3", "--sample-seed", "4",
                        "--out", str(tmp_path / "s.json")], capture_output=True, text=True)
    assert r.returncode == 0
    state = so.sample_initial_state(3, seed=4)[0]
    assert np.array_equal(so.load_problem(tmp_path / "s.json").flat()["root_state"], state)
    assert subprocess.run([exe, "validate", str(tmp_path / "s.json")]).returncode == 0
    (tmp_path / "bad.json").write_text('{"schema": 3}')
    r = subprocess.run([exe, "validate", str(tmp_path / "bad.json")], capture_output=True, text=True)
    assert r.returncode == 1 and "schema must be" in r.stderr
    assert subprocess.run([exe, "frobnicate"], capture_output=True).returncode == 2
    assert subprocess.run([exe, "gen", "random"], capture_output=True).returncode == 2  # --out required


def test_json_reader_edge_cases():
    """The in-house reader (csrc/host/json.cpp): escapes, number forms, whitespace,
    duplicate keys (the last wins, as std::map assignment), and malformed input."""
    base = json.loads(CHAIN_FILE)
    text = json.dumps(base)
    # whitespace and key order do not matter; unicode escapes in strings are decoded
    spaced = text.replace(":", " :\n\t").replace(",", " ,\r\n ")
    assert so.serialize_problem(so.parse_problem(spaced)) == so.serialize_problem(so.parse_problem(text))
    doc = dict(base)
    doc["constraints"] = dict(base["constraints"], kind="\\u0062ox")  # "box" spelled with an escape
    assert so.parse_problem(json.dumps(doc).replace("\\\\u0062", "\\u0062")).flat()["g_kind"][1] == 1
    # number forms: exponents, negative zero, integers where doubles are expected
    doc = json.loads(CHAIN_FILE)
    doc["root_state"] = [2.5e-1, -5E-1]
    doc["dims"] = {"nx": 2, "nu": 1.0}  # dims accept numbers
    t = json.dumps(doc).replace("0.25", "2.5e-1")
    assert list(so.parse_problem(t).flat()["root_state"]) == [0.25, -0.5]
    # duplicate keys: the last one is used
    dup = text[:-1] + ', "root_state": [1.0, 2.0]}'
    assert list(so.parse_problem(dup).flat()["root_state"]) == [1.0, 2.0]
    # malformed documents name a byte position
    for bad in ('{"schema": "scenopt-problem-v1",}', '{"a": [1, 2,]}', '{"a": 01}', '{"a": "x\\q"}',
                '{"a": .5}', '{"a": tru}', '["unterminated]', '{"a": 1} trailing', '', '   '):
        with pytest.raises(so.ParseError, match="not valid JSON"):
            so.parse_problem(bad)
    # deep nesting is bounded, not a stack overflow
    with pytest.raises(so.ParseError):
        so.parse_problem("[" * 100000)
