"""BASELINE's full-size tree (C4: nx=50, nu=20, N=20, branching [8,8,8,8,4];
266,825 nodes, 18.35 M primal, 550k dual) checked through size-independent
properties, where the CPU oracle would take minutes per sweep:
- linearity of the homogeneous sweep (x0 and H x0 are linear in r);
- the affine / homogeneous split: x(y) - x(0) = x0(y) (tree_oracles.hpp:96-114);
- symmetry of the dual Hessian: <r1, H x0(r2)> = <r2, H x0(r1)>, and its sign;
- bitwise determinism, and 2-RHS launches equal to two 1-RHS launches.
Together with the oracle parity at C1-C3 sizes these pin the C4 sweep."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4():
    prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 8, 4])
    cache = so.factor(prob)
    cache.device()
    return prob, cache


def _flat(pt):
    return np.concatenate([pt.x.ravel(order="F"), pt.u.ravel(order="F")])


def test_c4_homogeneous_sweep_is_linear(gpu, c4):
    prob, cache = c4
    assert prob.num_nodes() == 266825 and prob.primal_dim() == 18350020
    rng = np.random.default_rng(7)
    r1, r2 = rng.uniform(-1, 1, prob.dual_dim), rng.uniform(-1, 1, prob.dual_dim)
    a, b = 0.75, -1.25
    (p1, p2), (h1, h2) = so.sweep(cache, [r1, r2], False)
    (p3,), (h3,) = so.sweep(cache, [a * r1 + b * r2], False)
    lin = a * _flat(p1) + b * _flat(p2)
    assert np.abs(_flat(p3) - lin).max() <= 1e-11 * (1 + np.abs(lin).max())
    hl = a * h1 + b * h2
    assert np.abs(h3 - hl).max() <= 1e-11 * (1 + np.abs(hl).max())
    # dual Hessian symmetry and negative semi-definiteness (f* concave on the dual)
    s12, s21 = float(r1 @ h2), float(r2 @ h1)
    assert abs(s12 - s21) <= 1e-10 * (abs(s12) + abs(s21) + 1)
    for r, h in ((r1, h1), (r2, h2)):
        assert float(r @ h) <= 1e-9 * np.linalg.norm(r) * np.linalg.norm(h)


def test_c4_affine_sweep_is_homogeneous_plus_offset(gpu, c4):
    prob, cache = c4
    rng = np.random.default_rng(8)
    y = rng.uniform(-1, 1, prob.dual_dim)
    (pa,), (ha,) = so.sweep(cache, [y], True)
    (p0,), (h0,) = so.sweep(cache, [np.zeros(prob.dual_dim)], True)
    (ph,), (hh,) = so.sweep(cache, [y], False)
    diff = _flat(pa) - _flat(p0)
    assert np.abs(diff - _flat(ph)).max() <= 1e-11 * (1 + np.abs(_flat(pa)).max())
    assert np.abs((ha - h0) - hh).max() <= 1e-11 * (1 + np.abs(ha).max())


def test_c4_sweeps_are_deterministic_and_rhs_independent(gpu, c4):
    prob, cache = c4
    rng = np.random.default_rng(9)
    y, r = rng.uniform(-1, 1, prob.dual_dim), rng.uniform(-1, 1, prob.dual_dim)
    (a1,), (ah1,) = so.sweep(cache, [y], True)
    (a2,), (ah2,) = so.sweep(cache, [y], True)
    assert np.array_equal(_flat(a1), _flat(a2)) and np.array_equal(ah1, ah2)
    (q1, q2), (g1, g2) = so.sweep(cache, [y, r], False)
    (s1,), (k1,) = so.sweep(cache, [y], False)
    (s2,), (k2,) = so.sweep(cache, [r], False)
    assert np.array_equal(_flat(q1), _flat(s1)) and np.array_equal(_flat(q2), _flat(s2))
    assert np.array_equal(g1, k1) and np.array_equal(g2, k2)
