"""Python mirror of the reference's scenopt C++ API for the hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/scenopt/{problem_data,riccati,tree_oracles,
prox,fbe,lbfgs,solvers}.hpp, so parity tests read like the reference's own
tests. Everything numeric runs in libscenopt_b200.so (sm_100a kernels);
this module only marshals numpy buffers through the C-ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import check, dptr, iptr

HOST = N.HOST_IO


# ---------------------------------------------------------------- data model
@dataclass
class PrimalPoint:
    """problem_data.hpp:64-77: x is nx x num_nodes, u is nu x first_leaf."""

    x: np.ndarray
    u: np.ndarray

    def flatten(self) -> np.ndarray:
        return np.concatenate([self.u.ravel(order="F"), self.x.ravel(order="F")])

    def dot(self, o: "PrimalPoint") -> float:
        return float(np.sum(self.u * o.u) + np.sum(self.x * o.x))


@dataclass
class OracleStats:
    """tree_oracles.hpp:14-21."""

    dual_grad_calls: int = 0
    hessian_vec_calls: int = 0
    prox_calls: int = 0
    conj_calls: int = 0

    def sweep_total(self) -> int:
        return self.dual_grad_calls + self.hessian_vec_calls


class ProblemInstance:
    """problem_data.hpp:95-141 (flat, node-indexed; see scenopt_problem_view)."""

    def __init__(self, handle):
        self._h = handle
        dims = np.zeros(8, np.int32)
        check(N.lib().scenopt_problem_dims(self._h, iptr(dims)))
        (self.nx, self.nu, self.num_stages, self._n, self.num_leaves, self.first_leaf,
         self.dual_dim, self._primal_dim) = (int(v) for v in dims)
        self._flat = None

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.scenopt_problem_destroy(self._h)
            self._h = None

    @classmethod
    def from_flat(cls, flat: dict) -> "ProblemInstance":
        v, keep = N.view_from_flat(flat)
        h = C.c_void_p()
        check(N.lib().scenopt_problem_create(C.byref(v), C.byref(h)))
        del keep
        return cls(h)

    def num_nodes(self) -> int:
        return self._n

    def primal_dim(self) -> int:
        return self._primal_dim

    def flat(self) -> dict:
        if self._flat is None:
            v = N.ProblemView()
            dd = C.c_int32()
            check(N.lib().scenopt_problem_get_view(self._h, C.byref(v), C.byref(dd)))
            n, nx, nu, Ns = v.num_nodes, v.nx, v.nu, v.num_stages
            L = self.num_leaves
            D = int(dd.value)
            rows = np.ctypeslib.as_array(v.stage_rows, shape=(n,)).copy()
            S = int(rows.sum())

            def arr(ptr, size, dtype=np.float64):
                if size == 0:
                    return np.zeros(0, dtype)
                return np.ctypeslib.as_array(ptr, shape=(size,)).copy().astype(dtype)

            self._flat = dict(
                nx=nx, nu=nu, num_stages=Ns, num_nodes=n,
                ancestor=arr(v.ancestor, n, np.int32), probability=arr(v.probability, n),
                stage_offsets=arr(v.stage_offsets, Ns + 2, np.int32),
                root_state=arr(v.root_state, nx), A=arr(v.A, n * nx * nx),
                B=arr(v.B, n * nx * nu), c=arr(v.c, n * nx), Q=arr(v.Q, n * nx * nx),
                R=arr(v.R, n * nu * nu), S=arr(v.S, n * nu * nx), q=arr(v.q, n * nx),
                r=arr(v.r, n * nu), stage_rows=rows.astype(np.int32), F=arr(v.F, S * nx),
                G=arr(v.G, S * nu), g_kind=arr(v.g_kind, n, np.int32),
                g_gamma=arr(v.g_gamma, n), P=arr(v.P, L * nx * nx), p=arr(v.p, L * nx),
                terminal_rows=arr(v.terminal_rows, L, np.int32), FN=arr(v.FN, (D - S) * nx),
                tg_kind=arr(v.tg_kind, L, np.int32), tg_gamma=arr(v.tg_gamma, L),
                zmin=arr(v.zmin, D), zmax=arr(v.zmax, D))
        return self._flat

    def validate(self) -> list:
        buf = C.create_string_buffer(1 << 16)
        check(N.lib().scenopt_problem_validate(self._h, buf, len(buf)))
        return [s for s in buf.value.decode().split("\n") if s]


def gen_random_instance(seed: int, nx: int = 3, nu: int = 2, horizon: int = 3,
                        branching=2) -> ProblemInstance:
    """generators.hpp:255-328; `branching` is an int (reference: full
    branching at every stage) or a per-stage list (1 after its end)."""
    if isinstance(branching, int):
        br = [branching] * horizon
    else:
        br = list(branching)
    b = np.asarray(br, np.int32)
    h = C.c_void_p()
    check(N.lib().scenopt_problem_gen_random(C.c_uint64(seed), nx, nu, horizon, iptr(b), len(b),
                                             C.byref(h)))
    return ProblemInstance(h)


def precondition(prob: ProblemInstance) -> ProblemInstance:
    """solvers.hpp:569-602."""
    h = C.c_void_p()
    check(N.lib().scenopt_problem_precondition(prob._h, C.byref(h)))
    return ProblemInstance(h)


# ---------------------------------------------------------------- factor
class FactorCache:
    """riccati.hpp:38-63. Owns the device-resident packed instance on first
    oracle use (the B200 counterpart of the reference's per-node Eigen
    matrices)."""

    def __init__(self, handle, prob: ProblemInstance):
        self._h = handle
        self._prob = prob
        self._dev = None
        self.nx, self.nu = prob.nx, prob.nu
        self.num_nodes = prob.num_nodes()
        self.first_leaf = prob.first_leaf
        self.dual_dim = prob.dual_dim

    def __del__(self):
        if getattr(self, "_dev", None) is not None and N._lib is not None:
            N._lib.scenopt_dev_destroy(self._dev)
            self._dev = None
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.scenopt_factor_destroy(self._h)
            self._h = None

    def device(self, device: int = 0):
        if self._dev is None:
            h = C.c_void_p()
            check(N.lib().scenopt_dev_create(self._prob._h, self._h, device, C.byref(h)))
            self._dev = h
        return self._dev

    def dev_info(self) -> dict:
        info = N.DevInfoC()
        check(N.lib().scenopt_dev_info_get(self.device(), C.byref(info)))
        return {k: getattr(info, k) for k, _ in N.DevInfoC._fields_}

    def export(self) -> dict:
        p = self._prob
        nx, nu, n, F, L, D = p.nx, p.nu, p.num_nodes(), p.first_leaf, p.num_leaves, p.dual_dim
        S = int(p.flat()["stage_rows"].sum())
        out = dict(gain=np.zeros(F * nu * nx), child_to_input=np.zeros(n * nu * nx),
                   closed_loop=np.zeros(n * nx * nx), dual_to_input=np.zeros(max(S, 1) * nu),
                   dual_to_costate=np.zeros(max(S, 1) * nx), input_affine=np.zeros(F * nu),
                   costate_affine=np.zeros(F * nx), value_quad=np.zeros(n * nx * nx),
                   leaf_costate_affine=np.zeros(L * nx))
        del D
        check(N.lib().scenopt_factor_export(self._h, *[dptr(out[k]) for k in (
            "gain", "child_to_input", "closed_loop", "dual_to_input", "dual_to_costate",
            "input_affine", "costate_affine", "value_quad", "leaf_costate_affine")]))
        return out


def factor(prob: ProblemInstance) -> FactorCache:
    """riccati.hpp:82-182."""
    h = C.c_void_p()
    check(N.lib().scenopt_factor_create(prob._h, C.byref(h)))
    return FactorCache(h, prob)


def refactor_affine(cache: FactorCache, prob: ProblemInstance) -> None:
    """riccati.hpp:187-216 (the device copy is re-packed on next use)."""
    check(N.lib().scenopt_refactor_affine(cache._h, prob._h))
    if cache._dev is not None:
        N.lib().scenopt_dev_destroy(cache._dev)
        cache._dev = None
    cache._prob = prob


def _check_shapes(cache: FactorCache, prob: ProblemInstance, who: str):
    # riccati.hpp:67-74
    if (cache.num_nodes != prob.num_nodes() or cache.nx != prob.nx or cache.nu != prob.nu
            or cache.dual_dim != prob.dual_dim or cache.first_leaf != prob.first_leaf):
        raise N.CacheMismatch(f"{who}: cache was built for a different problem shape")


def _dual(prob, v, who):
    a = np.ascontiguousarray(v, dtype=np.float64)
    if a.ndim != 1 or a.size != prob.dual_dim:
        raise N.DimensionMismatch(f"{who}: dual vector has wrong length")
    return a


def _primal_out(prob):
    return (np.zeros(prob.nx * prob.num_nodes()), np.zeros(prob.nu * prob.first_leaf))


def _pp(prob, x, u) -> PrimalPoint:
    return PrimalPoint(x.reshape((prob.nx, prob.num_nodes()), order="F"),
                       u.reshape((prob.nu, prob.first_leaf), order="F"))


# ---------------------------------------------------------------- oracles
def dual_grad(cache: FactorCache, prob: ProblemInstance, y, stats: OracleStats | None = None):
    """tree_oracles.hpp:96-102: x(y) = argmin <z, H'y> + f(z)."""
    _check_shapes(cache, prob, "dual_grad")
    yv = _dual(prob, y, "riccati_sweep")
    x, u = _primal_out(prob)
    check(N.lib().scenopt_dual_grad(cache.device(), dptr(yv), dptr(x), dptr(u), HOST))
    if stats is not None:
        stats.dual_grad_calls += 1
    return _pp(prob, x, u)


def hessian_vec(cache: FactorCache, prob: ProblemInstance, r, stats: OracleStats | None = None):
    """tree_oracles.hpp:107-114: homogeneous part x0(r)."""
    _check_shapes(cache, prob, "hessian_vec")
    rv = _dual(prob, r, "riccati_sweep")
    x, u = _primal_out(prob)
    check(N.lib().scenopt_hessian_vec(cache.device(), dptr(rv), dptr(x), dptr(u), HOST))
    if stats is not None:
        stats.hessian_vec_calls += 1
    return _pp(prob, x, u)


def sweep(cache: FactorCache, ys, affine: bool, want_primal: bool = True):
    """Fused multi-RHS sweep (1 or 2 right-hand sides) returning
    (PrimalPoint list, Hx list) — the p-NAMA building block."""
    prob = cache._prob
    nr = len(ys)
    yv = [_dual(prob, y, "sweep") for y in ys]
    xs = [np.zeros(prob.nx * prob.num_nodes()) for _ in range(nr)] if want_primal else None
    us = [np.zeros(prob.nu * prob.first_leaf) for _ in range(nr)] if want_primal else None
    hs = [np.zeros(prob.dual_dim) for _ in range(nr)]
    P = C.POINTER(C.c_double)
    Yarr = (P * 2)(*[dptr(a) for a in yv])
    Xarr = (P * 2)(*[dptr(a) for a in xs]) if xs else None
    Uarr = (P * 2)(*[dptr(a) for a in us]) if us else None
    Harr = (P * 2)(*[dptr(a) for a in hs])
    check(N.lib().scenopt_dev_sweep(cache.device(), nr, int(affine), Yarr, Xarr, Uarr, Harr, HOST))
    pts = [_pp(prob, xs[i], us[i]) for i in range(nr)] if want_primal else None
    return pts, hs
