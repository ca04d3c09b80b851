"""GPU parity of the forward-backward machinery (fbe.hpp, prox.hpp,
lbfgs.hpp) against the CPU oracle, restating test_fbe.cpp / test_prox.cpp /
test_lbfgs.cpp properties through the CUDA path."""
import numpy as np
import pytest

import paper_2107_01745_b200 as so
from oracle import oracle as orc
from tests import support as sup

pytestmark = pytest.mark.gpu


def mixed():
    return orc.InstanceOptions(with_box=True, with_l1=True, with_none=True)


def fixture(rng, opt=None):
    po = rng.random_instance(rng.integer(2, 4), 25, rng.integer(2, 3), 2, opt or orc.InstanceOptions())
    prob = so.ProblemInstance.from_flat(po.flat())
    return po, prob, so.factor(prob), orc.Factor(po), orc.Nonsmooth.from_problem(po)


def close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max(initial=0.0) <= tol * (1 + np.abs(b).max(initial=0.0))


def test_fb_step_matches_oracle_and_is_consistent(gpu):
    rng = orc.Rng(61)  # test_fbe.cpp:44-79
    for trial in range(8):
        po, prob, cache, ofac, og = fixture(rng, mixed())
        y = rng.vector(prob.dual_dim)
        lam = rng.uniform(0.05, 2.0)
        st = so.OracleStats()
        s = so.fb_step(cache, prob, y, lam, st)
        assert (st.dual_grad_calls, st.prox_calls, st.hessian_vec_calls) == (1, 1, 0)
        o = orc.fb_step(ofac, og, y, lam)
        for k in ("Hx", "z", "R", "T"):
            assert close(getattr(s, k), o[k], 1e-9), k
        assert close(s.x.x.ravel(order="F"), o["x"], 1e-9)
        for k in ("fhat", "conj_T", "znorm_sq", "value"):
            assert abs(getattr(s, k) - o[k]) <= 1e-9 * (1 + abs(o[k])), k
        assert np.abs(s.R - (s.z - s.Hx)).max() < 1e-13
        assert np.abs(s.T - (s.y - lam * s.R)).max() < 1e-13
        other = s.fhat - 0.5 * lam * s.Hx @ s.Hx + s.conj_T + 0.5 * lam * s.znorm_sq
        assert abs(s.value - other) < 1e-10 * (1 + abs(s.value))
        assert np.isfinite(so.fbe_value(s))


def test_fb_step_rejects_nonpositive_step(gpu):
    rng = orc.Rng(62)
    po, prob, cache, _, _ = fixture(rng)
    y = rng.vector(prob.dual_dim)
    for lam in (0.0, -1.0):
        with pytest.raises(so.InvalidParams):
            so.fb_step(cache, prob, y, lam)


def test_unconstrained_blocks_make_T_zero(gpu):
    rng = orc.Rng(64)  # test_fbe.cpp:100-114
    po, prob, cache, _, _ = fixture(rng, orc.InstanceOptions(with_box=False, with_none=True))
    y = rng.vector(prob.dual_dim, 3.0)
    s = so.fb_step(cache, prob, y, 0.7)
    assert np.abs(s.T).max() < 1e-12 * (1 + np.abs(y).max())
    assert s.conj_T == 0.0


def test_fbe_grad_matches_oracle_and_finite_differences(gpu):
    rng = orc.Rng(66)  # test_fbe.cpp:135-165
    for trial in range(3):
        po, prob, cache, ofac, og = fixture(rng, mixed())
        lip = sup.dual_lipschitz_dense(ofac)
        lam = 0.7 / lip
        y = rng.vector(prob.dual_dim)
        s = so.fb_step(cache, prob, y, lam)
        g = so.fbe_grad(s, cache, prob)
        assert close(g, orc.fbe_grad(ofac, s.R, lam), 1e-9)
        fd = np.zeros(prob.dual_dim)
        for j in range(prob.dual_dim):
            h = 1e-5 * (1 + abs(y[j]))
            yp, ym = y.copy(), y.copy()
            yp[j] += h
            ym[j] -= h
            fd[j] = (so.fb_step(cache, prob, yp, lam).value - so.fb_step(cache, prob, ym, lam).value) / (2 * h)
        assert np.abs(g - fd).max() / (1 + np.abs(g).max()) < 1e-5


@pytest.mark.parametrize("shifted", [False, True])
def test_certificate_matches_oracle_and_direct_difference(gpu, shifted):
    rng = orc.Rng(68 if not shifted else 69)  # test_fbe.cpp:187-268
    taus = [1.0, 0.5, 0.25]
    for trial in range(6):
        po, prob, cache, ofac, og = fixture(rng, mixed())
        lip = sup.dual_lipschitz_dense(ofac)
        lam = (0.6 if trial % 2 == 0 else 2.0) / lip
        y = rng.vector(prob.dual_dim)
        d = rng.vector(prob.dual_dim)
        s = so.fb_step(cache, prob, y, lam)
        shift = None
        if shifted:
            shift = s.R.copy() if trial % 2 == 0 else rng.vector(prob.dual_dim)
        cert = so.linesearch_cert(cache, prob, s, d, taus, shift=shift)
        ostate = orc.fb_step(ofac, og, y, lam)
        ocert = orc.linesearch_cert(ofac, og, ostate, d, taus, shift=shift)
        assert close(cert["deltas"], ocert["deltas"], 1e-8)
        for k in ("alpha1", "alpha2", "conj_anchor", "znorm_sq_anchor", "value_anchor", "fhat_anchor"):
            assert abs(cert[k] - ocert[k]) <= 1e-8 * (1 + abs(ocert[k])), k
        anchor_value = s.value if shift is None else so.fb_step(cache, prob, y + shift, lam).value
        for t, delta in zip(taus, cert["deltas"]):
            w = y + t * d if shift is None else y + t * d + (1 - t) * shift
            direct = so.fb_step(cache, prob, w, lam)
            expected = direct.value - anchor_value
            assert abs(delta - expected) < 1e-8 * (1 + abs(expected))
        assert np.abs(cert["w"] - w).max() < 1e-12
        assert np.abs(cert["T"] - direct.T).max() < 1e-10
        assert np.abs(cert["cert_fhat"][-1] - direct.fhat) < 1e-9 * (1 + abs(direct.fhat))


def test_prox_conj_subdiff_match_oracle(gpu):
    rng = orc.Rng(24)  # test_prox.cpp
    po, prob, cache, ofac, og = fixture(rng, mixed())
    g = so.make_nonsmooth(prob, cache)
    for trial in range(10):
        v = rng.vector(prob.dual_dim, 3.0)
        s = rng.uniform(0.1, 3.0)
        z = g.prox(v, s)
        assert np.array_equal(z, og.prox(v, s)) or close(z, og.prox(v, s), 1e-15)
        w = v - z
        assert g.conj(w) == pytest.approx(og.conj(w), rel=1e-12, abs=1e-12)
        assert g.dist_subdiff_inf((v - z) / s, z) < 1e-12
        yy = rng.vector(prob.dual_dim)
        assert g.dist_subdiff_inf(yy, z) == pytest.approx(og.dist_subdiff_inf(yy, z), abs=1e-15)
    with pytest.raises(so.InvalidParams):
        g.prox(np.zeros(prob.dual_dim), 0.0)


def test_lbfgs_two_loop_matches_dense_bfgs(gpu):
    rng = orc.Rng(83)  # test_lbfgs.cpp:53-89
    prob = so.gen_random_instance(1, 3, 2, 2, 2)
    cache = so.factor(prob)
    for trial in range(6):
        dim = rng.integer(4, 12)
        memory = rng.integer(2, 6)
        buf = so.LbfgsBuffer(memory, 1e-12, cache)
        root = rng.matrix(dim, dim)
        spd = root @ root.T + 0.5 * np.eye(dim)
        accepted = []
        for k in range(memory + rng.integer(0, 3)):
            step = rng.vector(dim)
            change = spd @ step
            assert buf.push(step, change, 1.0)
            accepted.append((step, change))
            accepted = accepted[-memory:]
        assert buf.size() == len(accepted)
        s_, q_ = accepted[-1]
        gamma = s_ @ q_ / (q_ @ q_)
        assert buf.gamma0() == pytest.approx(gamma, abs=1e-14)
        inv = sup.dense_bfgs_inverse(accepted, dim, gamma)
        for probe in range(4):
            g = rng.vector(dim)
            expected = -(inv @ g)
            assert np.abs(buf.apply_direction(g) - expected).max() < 1e-11 * (1 + np.abs(expected).max())


@pytest.mark.parametrize("memory", [1, 6, 7, 9])
def test_lbfgs_direction_both_kernels_match_dense_bfgs(gpu, memory):
    """memory <= 6: compact-form kernel; above: the two-loop kernel. Both are
    the dense BFGS inverse of the stored pairs, with and without eviction."""
    rng = orc.Rng(84 + memory)
    prob = so.gen_random_instance(1, 3, 2, 2, 2)
    cache = so.factor(prob)
    dim = 14
    buf = so.LbfgsBuffer(memory, 1e-12, cache)
    root = rng.matrix(dim, dim)
    spd = root @ root.T + 0.5 * np.eye(dim)
    accepted = []
    for k in range(memory + 3):
        step = rng.vector(dim)
        change = spd @ step
        assert buf.push(step, change, 1.0)
        accepted = (accepted + [(step, change)])[-memory:]
        s_, q_ = accepted[-1]
        inv = sup.dense_bfgs_inverse(accepted, dim, s_ @ q_ / (q_ @ q_))
        g = rng.vector(dim)
        expected = -(inv @ g)
        assert np.abs(buf.apply_direction(g) - expected).max() < 1e-11 * (1 + np.abs(expected).max())


def test_lbfgs_gate_is_strict_and_clear_resets(gpu):
    prob = so.gen_random_instance(1, 3, 2, 2, 2)
    cache = so.factor(prob)
    step = np.zeros(5)
    step[0] = 1.0
    buf = so.LbfgsBuffer(4, 1e-12, cache)
    change = np.zeros(5)
    change[0] = 1e-12 * 3.0
    assert not buf.push(step, change, 3.0)  # borderline equality rejected
    assert buf.size() == 0 and buf.gamma0() == 1.0
    change[0] = 2e-12
    assert buf.push(step, change, 1.0)
    assert not buf.push(step, -step, 1.0)
    assert not buf.push(np.zeros(5), np.ones(5), 1.0)
    buf.clear()
    assert buf.size() == 0 and buf.gamma0() == 1.0
    g = np.arange(5.0)
    assert np.abs(buf.apply_direction(g) + g).max() < 1e-15
    with pytest.raises(so.InvalidParams):
        so.LbfgsBuffer(0, 1e-12, cache)
    with pytest.raises(so.InvalidParams):
        so.LbfgsBuffer(5, 0.0, cache)


def test_fhat_value_and_grad_match_oracle(gpu):
    rng = orc.Rng(45)
    po, prob, cache, ofac, og = fixture(rng, mixed())
    y = rng.vector(prob.dual_dim)
    assert so.fhat_value(cache, prob, y) == pytest.approx(ofac.fhat_value(y), rel=1e-10, abs=1e-10)
    gx, gu = ofac.dual_grad(y)
    assert close(so.grad_fhat(cache, prob, y), -orc.apply_H(po, gx, gu), 1e-9)
