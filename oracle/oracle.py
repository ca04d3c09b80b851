"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU parity oracle.

Imported only by tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs. The product package never imports
this module (it must fail loudly without its CUDA library instead).

Problems cross the boundary as a *flat dict* of numpy arrays whose keys are
the fields of ``orc_problem_view`` (oracle/oracle_capi.h), the same layout as
the product's ``scenopt_problem_view`` (include/scenopt_b200.h).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)


class ProblemView(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("nu", C.c_int32), ("num_stages", C.c_int32), ("num_nodes", C.c_int32),
        ("ancestor", I32P), ("probability", F64P), ("stage_offsets", I32P), ("root_state", F64P),
        ("A", F64P), ("B", F64P), ("c", F64P), ("Q", F64P), ("R", F64P), ("S", F64P),
        ("q", F64P), ("r", F64P), ("stage_rows", I32P), ("F", F64P), ("G", F64P),
        ("g_kind", I32P), ("g_gamma", F64P), ("P", F64P), ("p", F64P), ("terminal_rows", I32P),
        ("FN", F64P), ("tg_kind", I32P), ("tg_gamma", F64P), ("zmin", F64P), ("zmax", F64P),
    ]


INT_FIELDS = ("ancestor", "stage_offsets", "stage_rows", "g_kind", "terminal_rows", "tg_kind")
DBL_FIELDS = ("probability", "root_state", "A", "B", "c", "Q", "R", "S", "q", "r", "F", "G",
              "g_gamma", "P", "p", "FN", "tg_gamma", "zmin", "zmax")


class SolverConfigC(C.Structure):
    _fields_ = [
        ("lambda0", C.c_double), ("eps", C.c_double), ("eps_curv", C.c_double),
        ("eps_bt", C.c_double), ("beta_bt", C.c_double), ("memory", C.c_int32),
        ("max_iters", C.c_int32), ("backtracking_rule", C.c_int32), ("warm_start", C.c_int32),
        ("warm_start_iters", C.c_int32), ("precondition", C.c_int32),
        ("nama_parallel_linesearch", C.c_int32), ("nama_update_tlambda", C.c_int32),
    ]


class ReportSummaryC(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("iterations", C.c_int32), ("verified", C.c_int32),
        ("trace_len", C.c_int32), ("dual_grad_calls", C.c_uint64),
        ("hessian_vec_calls", C.c_uint64), ("prox_calls", C.c_uint64),
        ("conj_calls", C.c_uint64), ("lipschitz_calls", C.c_uint64),
        ("lipschitz_estimate", C.c_double), ("lambda_final", C.c_double), ("eps", C.c_double),
        ("residual_inf", C.c_double), ("wall_ms", C.c_double),
        ("verify_residual_inf", C.c_double), ("verify_subdiff_dist", C.c_double),
    ]


class InstanceOptionsC(C.Structure):
    _fields_ = [
        ("with_box", C.c_int32), ("with_l1", C.c_int32), ("with_none", C.c_int32),
        ("affine", C.c_int32), ("stage_rows_lo", C.c_int32), ("stage_rows_hi", C.c_int32),
        ("feasible_boxes", C.c_int32),
    ]


ERROR_NAMES = {
    -1: "Error", -2: "NonStochasticMatrix", -3: "StageOutOfRange", -4: "DimensionMismatch",
    -5: "UnsupportedSpec", -6: "NotStronglyConvex", -7: "ShapeChanged", -8: "CacheMismatch",
    -9: "LineSearchStalled", -10: "StepUnderflow", -11: "ZeroProbability", -12: "InvalidParams",
    -13: "InfiniteConjugate", -14: "ParseError",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERROR_NAMES.get(code, "Error")


def build() -> str:
    """Compile liboracle.so (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None
_NATIVE_PATH = os.path.join(_HERE, "_build", "native", "liboracle.so")


def use_native() -> bool:
    """Timed CPU baseline only (bench.py): build the oracle with -O3
    -march=native on THIS host (``make native``, ~15 s) and load it instead of
    the portable parity build. Must run before the first lib() call. Returns
    False (portable build kept) when the build fails."""
    global _LIB_PATH
    if _lib is not None:
        return _LIB_PATH == _NATIVE_PATH
    try:
        subprocess.run(["make", "-s", "-C", _HERE, "native"], check=True,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    except (OSError, subprocess.CalledProcessError):
        return False
    _LIB_PATH = _NATIVE_PATH
    return True


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_rng_uniform.restype = C.c_double
        L.orc_lbfgs_gamma0.restype = C.c_double
        _lib = L
    return _lib


def _check(rc: int):
    if rc < 0:
        raise OracleError(rc, lib().orc_last_error().decode())
    return rc


def _p(a: np.ndarray):
    if a is None:
        return None
    if a.dtype == np.int32:
        return a.ctypes.data_as(I32P)
    return a.ctypes.data_as(F64P)


def _buf(n):
    return np.zeros(int(n), dtype=np.float64)


# ------------------------------------------------------------------ problems
def layout(flat: dict) -> dict:
    """Derived layout numbers of a flat problem (problem_data.hpp:126-140)."""
    n = int(flat["num_nodes"])
    N = int(flat["num_stages"])
    so = flat["stage_offsets"]
    first_leaf = int(so[N])
    L = n - first_leaf
    rows = flat["stage_rows"]
    dual_offset = np.full(n, -1, dtype=np.int64)
    off = 0
    for i in range(1, n):
        dual_offset[i] = off
        off += int(rows[i])
    stage_total = off
    tdual_offset = np.zeros(L, dtype=np.int64)
    for l in range(L):
        tdual_offset[l] = off
        off += int(flat["terminal_rows"][l])
    return dict(n=n, N=N, first_leaf=first_leaf, L=L, dual_dim=off, stage_total=stage_total,
                dual_offset=dual_offset, tdual_offset=tdual_offset)


class Problem:
    """Owning handle to an oracle ProblemInstance."""

    def __init__(self, handle):
        self.h = handle
        self._flat = None

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_problem_free(self.h)
            self.h = None

    @classmethod
    def from_flat(cls, flat: dict) -> "Problem":
        v, keep = _view_from_flat(flat)
        h = C.c_void_p()
        _check(lib().orc_problem_from_view(C.byref(v), C.byref(h)))
        del keep
        return cls(h)

    def flat(self) -> dict:
        """Copy of the instance as a flat dict of numpy arrays."""
        if self._flat is None:
            v = ProblemView()
            dd = C.c_int32()
            _check(lib().orc_problem_view_get(self.h, C.byref(v), C.byref(dd)))
            self._flat = _flat_from_view(v, int(dd.value))
        return self._flat

    @property
    def dual_dim(self) -> int:
        return layout(self.flat())["dual_dim"]

    def validate(self) -> list:
        buf = C.create_string_buffer(1 << 16)
        rc = lib().orc_problem_validate(self.h, buf, len(buf))
        _check(rc)
        return [s for s in buf.value.decode().split("\n") if s]

    def precondition(self) -> "Problem":
        h = C.c_void_p()
        _check(lib().orc_precondition(self.h, C.byref(h)))
        return Problem(h)

    def probability_roots(self):
        out = _buf(self.dual_dim)
        _check(lib().orc_probability_roots(self.h, _p(out)))
        return out


def _view_from_flat(flat):
    keep = {}
    v = ProblemView()
    for k in ("nx", "nu", "num_stages", "num_nodes"):
        setattr(v, k, int(flat[k]))
    for k in INT_FIELDS:
        a = np.ascontiguousarray(flat[k], dtype=np.int32)
        keep[k] = a
        setattr(v, k, a.ctypes.data_as(I32P))
    for k in DBL_FIELDS:
        a = np.ascontiguousarray(flat[k], dtype=np.float64)
        if a.size == 0:
            a = np.zeros(1)
        keep[k] = a
        setattr(v, k, a.ctypes.data_as(F64P))
    return v, keep


def _flat_from_view(v: ProblemView, dual_dim: int) -> dict:
    n, nx, nu, N = v.num_nodes, v.nx, v.nu, v.num_stages
    so = np.ctypeslib.as_array(v.stage_offsets, shape=(N + 2,)).copy()
    L = n - int(so[N])
    rows = np.ctypeslib.as_array(v.stage_rows, shape=(n,)).copy()
    trows = np.ctypeslib.as_array(v.terminal_rows, shape=(L,)).copy() if L else np.zeros(0, np.int32)
    S_tot = int(rows.sum())

    def arr(ptr, size, dtype=np.float64):
        if size == 0:
            return np.zeros(0, dtype)
        return np.ctypeslib.as_array(ptr, shape=(size,)).copy().astype(dtype)

    return dict(
        nx=nx, nu=nu, num_stages=N, num_nodes=n,
        ancestor=arr(v.ancestor, n, np.int32), probability=arr(v.probability, n),
        stage_offsets=so.astype(np.int32), root_state=arr(v.root_state, nx),
        A=arr(v.A, n * nx * nx), B=arr(v.B, n * nx * nu), c=arr(v.c, n * nx),
        Q=arr(v.Q, n * nx * nx), R=arr(v.R, n * nu * nu), S=arr(v.S, n * nu * nx),
        q=arr(v.q, n * nx), r=arr(v.r, n * nu), stage_rows=rows.astype(np.int32),
        F=arr(v.F, S_tot * nx), G=arr(v.G, S_tot * nu), g_kind=arr(v.g_kind, n, np.int32),
        g_gamma=arr(v.g_gamma, n), P=arr(v.P, L * nx * nx), p=arr(v.p, L * nx),
        terminal_rows=trows.astype(np.int32), FN=arr(v.FN, (dual_dim - S_tot) * nx),
        tg_kind=arr(v.tg_kind, L, np.int32), tg_gamma=arr(v.tg_gamma, L),
        zmin=arr(v.zmin, dual_dim), zmax=arr(v.zmax, dual_dim),
    )


def gen_random(seed: int, nx: int, nu: int, horizon: int, branching) -> Problem:
    br = np.asarray(list(branching), dtype=np.int32)
    h = C.c_void_p()
    _check(lib().orc_gen_random(C.c_uint64(seed), nx, nu, horizon, _p(br), len(br), C.byref(h)))
    return Problem(h)


class SpringMassC(C.Structure):
    _fields_ = [
        ("mass_kg", C.c_double), ("stiffness", C.c_double), ("damping", C.c_double),
        ("input_bound", C.c_double), ("velocity_bound", C.c_double), ("horizon", C.c_int32),
        ("sampling", C.c_double), ("state_weight", C.c_double), ("input_weight", C.c_double),
        ("terminal_weight", C.c_double), ("initial_len", C.c_int32), ("transition_rows", C.c_int32),
        ("transition_cols", C.c_int32), ("mode_values_len", C.c_int32), ("root_state_len", C.c_int32),
        ("initial_probs", F64P), ("transition", F64P), ("mode_values", F64P), ("root_state", F64P),
    ]


_SM_DEFAULTS = dict(mass_kg=5.0, stiffness=1.0, damping=0.1, input_bound=2.0, velocity_bound=5.0,
                    horizon=11, sampling=0.5, state_weight=5.0, input_weight=2.0, terminal_weight=100.0)


def _spring_params(par):
    """generators.hpp:49-64 from any object carrying the SpringMassParams
    attribute names (None / missing -> defaults)."""
    st = SpringMassC()
    for k, v in _SM_DEFAULTS.items():
        setattr(st, k, getattr(par, k, v) if par is not None else v)
    keep = []
    for name, ln in (("initial_probs", "initial_len"), ("mode_values", "mode_values_len"),
                     ("root_state", "root_state_len")):
        v = getattr(par, name, None) if par is not None else None
        if v is not None:
            a = np.ascontiguousarray(v, np.float64).ravel()
            keep.append(a)
            setattr(st, ln, a.size)
            setattr(st, name, a.ctypes.data_as(F64P))
    T = getattr(par, "transition", None) if par is not None else None
    if T is not None:
        T = np.ascontiguousarray(np.atleast_2d(T), np.float64)
        keep.append(T)
        st.transition_rows, st.transition_cols = T.shape
        st.transition = T.ctypes.data_as(F64P)
    return st, keep


def gen_spring_mass(masses: int, par=None) -> Problem:
    """generators.hpp:119-218 (series exponential for the ZOH)."""
    st, keep = _spring_params(par)
    h = C.c_void_p()
    _check(lib().orc_gen_spring_mass(int(masses), C.byref(st), C.byref(h)))
    return Problem(h)


def spring_mass_continuous(masses: int, par=None):
    st, keep = _spring_params(par)
    nx, nu = 2 * masses, masses - 1
    A, B = _buf(nx * nx), _buf(max(nx * nu, 1))
    _check(lib().orc_spring_mass_continuous(int(masses), C.byref(st), _p(A), _p(B)))
    return A.reshape((nx, nx), order="F"), B[:nx * nu].reshape((nx, nu), order="F")


def expm_series(X) -> np.ndarray:
    """test_generators.cpp:23-38."""
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    src = np.ascontiguousarray(X.ravel(order="F"))
    out = _buf(n * n)
    _check(lib().orc_expm_series(_p(src), n, _p(out)))
    return out.reshape((n, n), order="F")


def sample_initial_states(masses: int, par=None, seed: int = 0, count: int = 1) -> np.ndarray:
    st, keep = _spring_params(par)
    out = _buf(count * 2 * masses)
    _check(lib().orc_sample_initial_states(int(masses), C.byref(st), C.c_uint64(seed), int(count), _p(out)))
    return out.reshape(count, 2 * masses)


@dataclass
class InstanceOptions:
    with_box: bool = True
    with_l1: bool = False
    with_none: bool = False
    affine: bool = True
    stage_rows_lo: int = 1
    stage_rows_hi: int = 3
    feasible_boxes: bool = False

    def c(self):
        return InstanceOptionsC(int(self.with_box), int(self.with_l1), int(self.with_none),
                                int(self.affine), self.stage_rows_lo, self.stage_rows_hi,
                                int(self.feasible_boxes))


class Rng:
    """tests/support.hpp:24-44 (mt19937_64, top-53-bit doubles, column-major)."""

    def __init__(self, seed: int):
        self.h = C.c_void_p()
        lib().orc_rng_new(C.c_uint64(seed), C.byref(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_rng_free(self.h)
            self.h = None

    def uniform(self, lo=0.0, hi=1.0) -> float:
        return float(lib().orc_rng_uniform(self.h, C.c_double(lo), C.c_double(hi)))

    def integer(self, lo: int, hi: int) -> int:
        return int(lib().orc_rng_integer(self.h, lo, hi))

    def vector(self, n: int, scale: float = 1.0):
        out = _buf(n)
        lib().orc_rng_vector(self.h, n, C.c_double(scale), _p(out))
        return out

    def matrix(self, rows: int, cols: int, scale: float = 1.0):
        out = _buf(rows * cols)
        lib().orc_rng_matrix(self.h, rows, cols, C.c_double(scale), _p(out))
        return out.reshape((rows, cols), order="F")

    def random_instance(self, stages: int, max_nodes: int, nx: int, nu: int,
                        opt: InstanceOptions | None = None) -> Problem:
        o = (opt or InstanceOptions()).c()
        h = C.c_void_p()
        _check(lib().orc_random_instance(self.h, stages, max_nodes, nx, nu, C.byref(o), C.byref(h)))
        return Problem(h)

    def markov_instance(self, transition, initial, horizon, nx, nu,
                        opt: InstanceOptions | None = None) -> Problem:
        T = np.ascontiguousarray(transition, dtype=np.float64)
        p0 = np.ascontiguousarray(initial, dtype=np.float64)
        o = (opt or InstanceOptions()).c()
        h = C.c_void_p()
        _check(lib().orc_markov_instance(self.h, _p(T), _p(p0), len(p0), horizon, nx, nu,
                                         C.byref(o), C.byref(h)))
        return Problem(h)


def tree_from_markov(transition, initial, horizon):
    T = np.ascontiguousarray(transition, dtype=np.float64)
    p0 = np.ascontiguousarray(initial, dtype=np.float64)
    cap = 1 << 16
    n = C.c_int32()
    anc = np.zeros(cap, np.int32)
    prob = np.zeros(cap)
    so = np.zeros(horizon + 2, np.int32)
    mode = np.zeros(cap, np.int32)
    _check(lib().orc_tree_from_markov(_p(T), _p(p0), len(p0), horizon, C.byref(n), _p(anc),
                                      _p(prob), _p(so), _p(mode), cap))
    k = n.value
    return dict(num_nodes=k, ancestor=anc[:k], probability=prob[:k], stage_offsets=so,
                mode=mode[:k])


# ------------------------------------------------------------------ factor
class Factor:
    def __init__(self, prob: Problem):
        self.prob = prob
        self.h = C.c_void_p()
        _check(lib().orc_factor_create(prob.h, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_factor_free(self.h)
            self.h = None

    def refactor_affine(self, prob: Problem):
        _check(lib().orc_refactor_affine(self.h, prob.h))

    def export(self) -> dict:
        f = self.prob.flat()
        lay = layout(f)
        nx, nu, n, F, L = f["nx"], f["nu"], lay["n"], lay["first_leaf"], lay["L"]
        D = lay["dual_dim"]
        out = dict(gain=_buf(F * nu * nx), child_to_input=_buf(n * nu * nx),
                   closed_loop=_buf(n * nx * nx), dual_to_input=_buf(D * nu),
                   dual_to_costate=_buf(D * nx), input_affine=_buf(F * nu),
                   costate_affine=_buf(F * nx), value_quad=_buf(n * nx * nx),
                   leaf_costate_affine=_buf(L * nx))
        _check(lib().orc_factor_export(self.h, *[_p(out[k]) for k in (
            "gain", "child_to_input", "closed_loop", "dual_to_input", "dual_to_costate",
            "input_affine", "costate_affine", "value_quad", "leaf_costate_affine")]))
        return out

    # oracles ---------------------------------------------------------
    def _primal_bufs(self):
        f = self.prob.flat()
        lay = layout(f)
        return _buf(f["nx"] * lay["n"]), _buf(f["nu"] * lay["first_leaf"])

    def sweep(self, y, affine: bool):
        y = np.ascontiguousarray(y, dtype=np.float64)
        x, u = self._primal_bufs()
        _check(lib().orc_sweep(self.h, self.prob.h, _p(y), int(affine), _p(x), _p(u)))
        return x, u

    def dual_grad(self, y):
        return self.sweep(y, True)

    def hessian_vec(self, r):
        return self.sweep(r, False)

    def fhat_value(self, y):
        out = C.c_double()
        _check(lib().orc_fhat_value(self.h, self.prob.h, _p(np.ascontiguousarray(y, np.float64)),
                                    C.byref(out)))
        return out.value

    def estimate_lipschitz(self, rel_tol: float = 1e-6, max_rounds: int = 100):
        calls = C.c_uint64()
        out = C.c_double()
        _check(lib().orc_estimate_lipschitz_ex(self.h, self.prob.h, C.c_double(rel_tol), int(max_rounds),
                                               C.byref(calls), C.byref(out)))
        return out.value, int(calls.value)

    def time_sweeps(self, nsweeps: int, affine: bool = True) -> float:
        out = C.c_double()
        _check(lib().orc_time_sweeps(self.h, self.prob.h, nsweeps, int(affine), C.byref(out)))
        return out.value


def apply_H(prob: Problem, x, u):
    z = _buf(prob.dual_dim)
    _check(lib().orc_apply_H(prob.h, _p(np.ascontiguousarray(x, np.float64)),
                             _p(np.ascontiguousarray(u, np.float64)), _p(z)))
    return z


def apply_H_adjoint(prob: Problem, y):
    f = prob.flat()
    lay = layout(f)
    x, u = _buf(f["nx"] * lay["n"]), _buf(f["nu"] * lay["first_leaf"])
    _check(lib().orc_apply_H_adjoint(prob.h, _p(np.ascontiguousarray(y, np.float64)), _p(x), _p(u)))
    return x, u


def eval_f(prob: Problem, x, u) -> float:
    out = C.c_double()
    _check(lib().orc_eval_f(prob.h, _p(np.ascontiguousarray(x, np.float64)),
                            _p(np.ascontiguousarray(u, np.float64)), C.byref(out)))
    return out.value


# ------------------------------------------------------------------ nonsmooth
class Nonsmooth:
    def __init__(self, handle, dim):
        self.h = handle
        self.dim = dim

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_g_free(self.h)
            self.h = None

    @classmethod
    def from_problem(cls, prob: Problem):
        h = C.c_void_p()
        _check(lib().orc_g_from_problem(prob.h, C.byref(h)))
        return cls(h, prob.dual_dim)

    @classmethod
    def from_blocks(cls, dim, blocks):
        """blocks: list of dicts(offset,size,weight,kind,gamma,zmin,zmax)."""
        nb = len(blocks)
        off = np.array([b["offset"] for b in blocks], np.int32)
        size = np.array([b["size"] for b in blocks], np.int32)
        w = np.array([b["weight"] for b in blocks], np.float64)
        kind = np.array([b["kind"] for b in blocks], np.int32)
        gam = np.array([b.get("gamma", 0.0) for b in blocks], np.float64)
        zmin = np.zeros(dim)
        zmax = np.zeros(dim)
        for b in blocks:
            if b["kind"] == 1:
                zmin[b["offset"]:b["offset"] + b["size"]] = b["zmin"]
                zmax[b["offset"]:b["offset"] + b["size"]] = b["zmax"]
        h = C.c_void_p()
        _check(lib().orc_g_create(dim, nb, _p(off), _p(size), _p(w), _p(kind), _p(gam), _p(zmin),
                                  _p(zmax), C.byref(h)))
        return cls(h, dim)

    def prox(self, v, gamma_prox):
        out = _buf(self.dim)
        _check(lib().orc_prox_g(self.h, _p(np.ascontiguousarray(v, np.float64)),
                                C.c_double(gamma_prox), _p(out)))
        return out

    def conj(self, w):
        out = C.c_double()
        _check(lib().orc_conj_value_g(self.h, _p(np.ascontiguousarray(w, np.float64)), C.byref(out)))
        return out.value

    def prox_conj(self, v, lam):
        out = _buf(self.dim)
        _check(lib().orc_prox_g_conj(self.h, _p(np.ascontiguousarray(v, np.float64)),
                                     C.c_double(lam), _p(out)))
        return out

    def dist_subdiff_inf(self, y, z):
        out = C.c_double()
        _check(lib().orc_dist_subdiff_inf(self.h, _p(np.ascontiguousarray(y, np.float64)),
                                          _p(np.ascontiguousarray(z, np.float64)), C.byref(out)))
        return out.value


# ------------------------------------------------------------------ fbe
def fb_step(fac: Factor, g: Nonsmooth, y, lam: float) -> dict:
    prob = fac.prob
    D = prob.dual_dim
    x, u = fac._primal_bufs()
    Hx, z, R, T = _buf(D), _buf(D), _buf(D), _buf(D)
    sc = _buf(4)
    _check(lib().orc_fb_step(fac.h, prob.h, g.h, _p(np.ascontiguousarray(y, np.float64)),
                             C.c_double(lam), _p(x), _p(u), _p(Hx), _p(z), _p(R), _p(T), _p(sc)))
    return dict(y=np.array(y, dtype=np.float64), lam=lam, x=x, u=u, Hx=Hx, z=z, R=R, T=T,
                fhat=sc[0], conj_T=sc[1], znorm_sq=sc[2], value=sc[3])


def fbe_grad(fac: Factor, R, lam: float):
    out = _buf(fac.prob.dual_dim)
    _check(lib().orc_fbe_grad(fac.h, fac.prob.h, _p(np.ascontiguousarray(R, np.float64)),
                              C.c_double(lam), _p(out)))
    return out


def linesearch_cert(fac: Factor, g: Nonsmooth, state: dict, direction, taus, shift=None) -> dict:
    D = fac.prob.dual_dim
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    deltas = _buf(len(taus))
    cfh = _buf(len(taus))
    cs = _buf(6)
    w, Hxw, z, R, T = _buf(D), _buf(D), _buf(D), _buf(D), _buf(D)
    ss = np.array([state["fhat"], state["conj_T"], state["znorm_sq"], state["value"]])
    sh = None if shift is None else np.ascontiguousarray(shift, np.float64)
    _check(lib().orc_linesearch_cert(
        fac.h, fac.prob.h, g.h, _p(state["y"]), _p(state["Hx"]), C.c_double(state["lam"]), _p(ss),
        _p(sh), _p(np.ascontiguousarray(direction, np.float64)), len(taus), _p(taus), _p(deltas),
        _p(cs), _p(cfh), _p(w), _p(Hxw), _p(z), _p(R), _p(T)))
    return dict(deltas=deltas, alpha1=cs[0], alpha2=cs[1], conj_anchor=cs[2], znorm_sq_anchor=cs[3],
                value_anchor=cs[4], fhat_anchor=cs[5], cert_fhat=cfh, w=w, Hx_w=Hxw, z=z, R=R, T=T)


class Lbfgs:
    def __init__(self, memory: int, eps_curv: float):
        self.h = C.c_void_p()
        _check(lib().orc_lbfgs_new(memory, C.c_double(eps_curv), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_lbfgs_free(self.h)
            self.h = None

    def push(self, step, change, scale_ref) -> bool:
        s = np.ascontiguousarray(step, np.float64)
        q = np.ascontiguousarray(change, np.float64)
        return bool(lib().orc_lbfgs_push(self.h, len(s), _p(s), _p(q), C.c_double(scale_ref)))

    def apply_direction(self, grad):
        g = np.ascontiguousarray(grad, np.float64)
        out = _buf(len(g))
        _check(lib().orc_lbfgs_apply(self.h, len(g), _p(g), _p(out)))
        return out

    def clear(self):
        lib().orc_lbfgs_clear(self.h)

    def size(self):
        return lib().orc_lbfgs_size(self.h)

    def gamma0(self):
        return lib().orc_lbfgs_gamma0(self.h)


# ------------------------------------------------------------------ solvers
@dataclass
class SolverConfig:
    lambda0: float = 0.0
    eps: float = 5e-4
    eps_curv: float = 1e-12
    eps_bt: float = 0.25
    beta_bt: float = 0.05
    memory: int = 5
    max_iters: int = 20000
    backtracking_rule: int = 1  # 0 Original, 1 Simple, 2 None
    warm_start: bool = False
    warm_start_iters: int = 5
    precondition: bool = False
    nama_parallel_linesearch: bool = False
    nama_update_tlambda: bool = True

    def c(self):
        return SolverConfigC(self.lambda0, self.eps, self.eps_curv, self.eps_bt, self.beta_bt,
                             self.memory, self.max_iters, self.backtracking_rule,
                             int(self.warm_start), self.warm_start_iters, int(self.precondition),
                             int(self.nama_parallel_linesearch), int(self.nama_update_tlambda))


def _report(prob: Problem, h) -> dict:
    s = ReportSummaryC()
    lib().orc_report_summary_get(h, C.byref(s))
    f = prob.flat()
    lay = layout(f)
    D = lay["dual_dim"]
    x, u = _buf(f["nx"] * lay["n"]), _buf(f["nu"] * lay["first_leaf"])
    y, z = _buf(D), _buf(D)
    rt, ft = _buf(s.trace_len), _buf(s.trace_len)
    lib().orc_report_arrays(h, _p(x), _p(u), _p(y), _p(z), _p(rt), _p(ft))
    out = {k: getattr(s, k) for k, _ in ReportSummaryC._fields_}
    out.update(x=x, u=u, y=y, z=z, residual_trace=rt, fbe_trace=ft, _h=h)
    return out


def solve(prob: Problem, cfg: SolverConfig, kind: int, shared: Factor | None = None) -> dict:
    h = C.c_void_p()
    c = cfg.c()
    _check(lib().orc_solve(prob.h, C.byref(c), kind, shared.h if shared else None, C.byref(h)))
    try:
        return _report(prob, h)
    finally:
        pass


def solve_direct(prob: Problem, fac: Factor, cfg: SolverConfig, kind: int, y0=None, weight=None):
    D = prob.dual_dim
    y0 = np.zeros(D) if y0 is None else np.ascontiguousarray(y0, np.float64)
    w = None if weight is None else np.ascontiguousarray(weight, np.float64)
    h = C.c_void_p()
    c = cfg.c()
    _check(lib().orc_solve_direct(prob.h, fac.h, C.byref(c), kind, _p(y0), _p(w), C.byref(h)))
    return _report(prob, h)


def warm_start(prob: Problem, fac: Factor, cfg: SolverConfig, lam: float):
    y = _buf(prob.dual_dim)
    dg = C.c_uint64()
    c = cfg.c()
    _check(lib().orc_warm_start(prob.h, fac.h, C.byref(c), C.c_double(lam), _p(y), C.byref(dg)))
    return y, int(dg.value)


def verify_report(prob: Problem, rep: dict, z_override=None) -> dict:
    zo = None if z_override is None else np.ascontiguousarray(z_override, np.float64)
    _check(lib().orc_verify_report(prob.h, rep["_h"], _p(zo)))
    return _report(prob, rep["_h"])
