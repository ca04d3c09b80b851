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

__all__ = [
    # problem_data.hpp / generators.hpp / solvers.hpp:569-623
    "PrimalPoint", "ProblemInstance", "gen_random_instance", "gen_random_instance_shard", "precondition",
    "serialize_problem", "parse_problem", "save_problem", "load_problem", "validate_problem_text",
    "problem_to_json", "problem_from_json", "content_hash", "factor_hash", "PROBLEM_SCHEMA",
    "SpringMassParams", "gen_spring_mass", "spring_mass_continuous", "discretize_zoh", "expm",
    "sample_initial_state",
    # riccati.hpp (+ device factor, subtree sharding)
    "FactorCache", "DeviceFactorCache", "factor", "factor_device", "refactor_affine", "nccl_unique_id",
    "ShardGroup",
    # tree_oracles.hpp
    "OracleStats", "dual_grad", "hessian_vec", "sweep", "grad_fhat", "fhat_value", "apply_H",
    # prox.hpp / fbe.hpp / lbfgs.hpp
    "Nonsmooth", "make_nonsmooth", "FbState", "fb_step", "fbe_value", "fbe_grad", "linesearch_cert",
    "LbfgsBuffer",
    # solvers.hpp
    "SolverConfig", "SolverReport", "estimate_dual_lipschitz", "solve_minfbe", "solve_nama", "solve_gpad",
    "warm_start", "solve", "verify_report",
    # experiment.hpp
    "SolverSpec", "solver_spec_from_name", "default_solver_set", "BatchEntry", "ExperimentRow",
    "SolverSummary", "RunReport", "run_experiment", "RESULTS_CSV_HEADER",
]
from ._native import InvalidParams, check, dptr, iptr

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

    def mode(self) -> np.ndarray:
        """ScenarioTree::mode (scenario_tree.hpp:41); empty when unknown."""
        out = np.zeros(self._n, np.int32)
        k = check(N.lib().scenopt_problem_get_mode(self._h, iptr(out), self._n))
        return out[:k]

    def set_mode(self, mode) -> None:
        m = np.ascontiguousarray(mode, np.int32)
        check(N.lib().scenopt_problem_set_mode(self._h, iptr(m) if m.size else None, m.size))

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


def gen_random_instance_shard(seed: int, nx: int, nu: int, horizon: int, branching, rank: int, world: int,
                              stage: int = -1) -> ProblemInstance:
    """One rank's part of gen_random_instance(seed, ...) for a subtree-sharded
    run (scenopt_problem_gen_random_shard): only the nodes the rank holds are
    built, bit-identical to the full instance; use it with
    DeviceFactorCache.sharded(...) on that rank."""
    br = [branching] * horizon if isinstance(branching, int) else list(branching)
    b = np.asarray(br, np.int32)
    h = C.c_void_p()
    check(N.lib().scenopt_problem_gen_random_shard(C.c_uint64(seed), nx, nu, horizon, iptr(b), len(b), world,
                                                   rank, stage, C.byref(h)))
    return ProblemInstance(h)


# ---------------------------------------------------------------- problem files
PROBLEM_SCHEMA = "scenopt-problem-v1"  # problem_io.hpp:27


def serialize_problem(prob: ProblemInstance) -> str:
    """problem_io.hpp:480: canonical JSON text (sorted keys, 2-space indent)."""
    n = C.c_size_t()
    check(N.lib().scenopt_problem_serialize(prob._h, None, C.c_size_t(0), C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(N.lib().scenopt_problem_serialize(prob._h, buf, C.c_size_t(n.value + 1), C.byref(n)))
    return buf.raw[:n.value].decode()


def parse_problem(text: str) -> ProblemInstance:
    """problem_io.hpp:484 (ParseError on malformed or invalid documents)."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    check(N.lib().scenopt_problem_parse(raw, C.c_size_t(len(raw)), C.byref(h)))
    return ProblemInstance(h)


def save_problem(prob: ProblemInstance, path: str) -> None:
    check(N.lib().scenopt_problem_save(prob._h, str(path).encode()))


def load_problem(path: str) -> ProblemInstance:
    h = C.c_void_p()
    check(N.lib().scenopt_problem_load(str(path).encode(), C.byref(h)))
    return ProblemInstance(h)


def validate_problem_text(text: str) -> list:
    """problem_io.hpp:512-524: violation lines; empty when the document parses and validates."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    buf = C.create_string_buffer(1 << 16)
    k = check(N.lib().scenopt_problem_validate_text(raw, C.c_size_t(len(raw)), buf, len(buf)))
    return [ln for ln in buf.value.decode().split("\n") if ln][:k] if k else []


def problem_to_json(prob: ProblemInstance) -> dict:
    """problem_io.hpp:220 as a Python dict (the parsed canonical text)."""
    import json
    return json.loads(serialize_problem(prob))


def problem_from_json(doc: dict) -> ProblemInstance:
    """problem_io.hpp:323 from a Python dict."""
    import json
    return parse_problem(json.dumps(doc))


def content_hash(prob: ProblemInstance) -> int:
    """problem_io.hpp:539: FNV-1a of the canonical serialization."""
    h = C.c_uint64()
    check(N.lib().scenopt_problem_hashes(prob._h, C.byref(h), None))
    return h.value


def factor_hash(prob: ProblemInstance) -> int:
    """problem_io.hpp:546: FNV-1a of the factor-determining content (no root
    state, modes or nonsmooth specs)."""
    h = C.c_uint64()
    check(N.lib().scenopt_problem_hashes(prob._h, None, C.byref(h)))
    return h.value


@dataclass
class SpringMassParams:
    """generators.hpp:49-64; None arrays take the reference defaults
    (initial (0.5, 0.5), transition [[0.1, 0.9], [0.9, 0.1]], mode values
    (0, 0.1), zero root state)."""
    mass_kg: float = 5.0
    stiffness: float = 1.0
    damping: float = 0.1
    input_bound: float = 2.0
    velocity_bound: float = 5.0
    horizon: int = 11
    sampling: float = 0.5
    state_weight: float = 5.0
    input_weight: float = 2.0
    terminal_weight: float = 100.0
    initial_probs: np.ndarray | None = None
    transition: np.ndarray | None = None
    mode_values: np.ndarray | None = None
    root_state: np.ndarray | None = None

    def c(self, cls=None):
        """(struct, keep-alive arrays) for the C-ABI (or an identical layout `cls`)."""
        cls = cls or N.SpringMassC
        st = cls()
        for k in ("mass_kg", "stiffness", "damping", "input_bound", "velocity_bound", "horizon",
                  "sampling", "state_weight", "input_weight", "terminal_weight"):
            setattr(st, k, getattr(self, k))
        keep = []
        for name, ln in (("initial_probs", "initial_len"), ("mode_values", "mode_values_len"),
                         ("root_state", "root_state_len")):
            v = getattr(self, name)
            if v is not None:
                a = np.ascontiguousarray(v, np.float64).ravel()
                keep.append(a)
                setattr(st, ln, a.size)
                setattr(st, name, a.ctypes.data_as(N.F64P))
        if self.transition is not None:
            T = np.ascontiguousarray(np.atleast_2d(self.transition), np.float64)  # row-major
            keep.append(T)
            st.transition_rows, st.transition_cols = T.shape
            st.transition = T.ctypes.data_as(N.F64P)
        return st, keep


def gen_spring_mass(masses: int, params: SpringMassParams | None = None) -> ProblemInstance:
    """generators.hpp:119-218: ZOH-discretized spring-mass-damper array
    (nx = 2M, nu = M-1) on the Markov mode tree, box constraints on every
    velocity and input."""
    st, keep = (params or SpringMassParams()).c()
    h = C.c_void_p()
    check(N.lib().scenopt_problem_gen_spring_mass(int(masses), C.byref(st), C.byref(h)))
    return ProblemInstance(h)


def _colmajor(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))


def spring_mass_continuous(masses: int, params: SpringMassParams | None = None):
    """detail::spring_mass_continuous, generators.hpp:70-91 -> (A, B)."""
    st, keep = (params or SpringMassParams()).c()
    nx, nu = 2 * masses, max(masses - 1, 0)
    A, B = np.zeros(nx * nx), np.zeros(max(nx * nu, 1))
    check(N.lib().scenopt_spring_mass_continuous(int(masses), C.byref(st), dptr(A), dptr(B)))
    return A.reshape((nx, nx), order="F"), B[:nx * nu].reshape((nx, nu), order="F")


def expm(X) -> np.ndarray:
    """Matrix exponential (Pade scaling and squaring, the method of Eigen's exp())."""
    X = np.asarray(X, np.float64)
    if X.ndim != 2 or X.shape[0] != X.shape[1]:
        raise N.DimensionMismatch("expm: matrix must be square")
    n = X.shape[0]
    out = np.zeros(n * n)
    check(N.lib().scenopt_expm(dptr(_colmajor(X)), n, dptr(out)))
    return out.reshape((n, n), order="F")


def discretize_zoh(A, B, period: float):
    """generators.hpp:97-112 -> (Ad, Bd)."""
    A = np.atleast_2d(np.asarray(A, np.float64))
    B = np.asarray(B, np.float64)
    if B.ndim == 1:
        B = B.reshape(-1, 1)
    if A.shape[0] != A.shape[1] or B.shape[0] != A.shape[0]:
        raise N.DimensionMismatch("discretize_zoh: A must be square and match B")
    n, m = A.shape[0], B.shape[1]
    Ad, Bd = np.zeros(n * n), np.zeros(max(n * m, 1))
    check(N.lib().scenopt_discretize_zoh(dptr(_colmajor(A)), dptr(_colmajor(B) if m else np.zeros(1)), n, m,
                                         C.c_double(period), dptr(Ad), dptr(Bd)))
    return Ad.reshape((n, n), order="F"), Bd[:n * m].reshape((n, m), order="F")


def sample_initial_state(masses: int, params: SpringMassParams | None = None, seed: int = 0,
                         count: int = 1) -> np.ndarray:
    """generators.hpp:223-234: `count` consecutive draws from
    std::mt19937_64(seed); shape (count, 2M)."""
    st, keep = (params or SpringMassParams()).c()
    out = np.zeros((count, 2 * masses))
    check(N.lib().scenopt_sample_initial_states(int(masses), C.byref(st), C.c_uint64(seed), int(count),
                                                dptr(out)))
    return out


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

    def shard(self, rank: int, world: int, nccl_id: bytes | None, device: int = 0, stage: int = -1):
        """Attach a subtree-sharded device handle: every
        rank of `world` (one process per GPU) calls this concurrently with the
        same instance, factor and nccl_id (nccl_unique_id() on one rank,
        shared). All oracle and solver calls on this cache then run sharded."""
        if self._dev is not None:
            raise InvalidParams("shard(): the cache already has a device handle")
        if nccl_id is not None and len(nccl_id) != 128:
            raise InvalidParams("shard(): nccl_id must be 128 bytes")
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        check(N.lib().scenopt_dev_create_sharded(self._prob._h, self._h, device, rank, world, stage, buf,
                                                 C.byref(h)))
        self._dev = h
        return h

    def shard_emulated(self, rank: int, group: "ShardGroup", device: int = 0, stage: int = -1):
        """As shard(), for a rank of an emulated group (one process, one host
        thread per rank; exchanges through host memory, no NCCL): tests of
        the sharded solver with several ranks on one GPU."""
        if self._dev is not None:
            raise InvalidParams("shard_emulated(): the cache already has a device handle")
        h = C.c_void_p()
        check(N.lib().scenopt_dev_create_sharded_group(self._prob._h, self._h, device, rank, group._h, stage,
                                                       C.byref(h)))
        self._dev = h
        return h

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


class ShardGroup:
    """Emulated shard group of `world` ranks in this process
    (scenopt_shard_group_create); see FactorCache.shard_emulated."""

    def __init__(self, world: int):
        self._h = C.c_void_p()
        check(N.lib().scenopt_shard_group_create(world, C.byref(self._h)))
        self.world = world

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.scenopt_shard_group_destroy(self._h)
            self._h = None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) for FactorCache.shard()."""
    buf = C.create_string_buffer(128)
    check(N.lib().scenopt_nccl_unique_id(buf))
    return buf.raw


class DeviceFactorCache(FactorCache):
    """factor() computed on the device (K9): the handle
    is packed from problem data and the Riccati factor is written into the
    sweep layout by a per-stage GPU kernel; export() reads it back in the
    FactorCache layout."""

    def __init__(self, prob: ProblemInstance, device: int = 0, _handle=None):
        super().__init__(None, prob)
        h = _handle
        if h is None:
            h = C.c_void_p()
            check(N.lib().scenopt_dev_create_device_factor(prob._h, device, C.byref(h)))
        self._dev = h

    @classmethod
    def sharded(cls, prob: ProblemInstance, rank: int, world: int = 1, nccl_id: bytes | None = None,
                group: "ShardGroup | None" = None, device: int = 0, stage: int = -1) -> "DeviceFactorCache":
        """A subtree-sharded handle whose factor is computed on the device
        (each rank factors its own subtrees and the replicated top; no host
        factor): one rank of an NCCL group (nccl_id) or of an emulated
        ShardGroup (group)."""
        h = C.c_void_p()
        if group is not None:
            check(N.lib().scenopt_dev_create_sharded_group(prob._h, None, device, rank, group._h, stage,
                                                           C.byref(h)))
        else:
            if nccl_id is not None and len(nccl_id) != 128:
                raise InvalidParams("sharded(): nccl_id must be 128 bytes")
            buf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
            check(N.lib().scenopt_dev_create_sharded(prob._h, None, device, rank, world, stage, buf, C.byref(h)))
        return cls(prob, device, _handle=h)

    def device(self, device: int = 0):
        return self._dev

    def shard(self, *a, **k):
        raise InvalidParams("shard(): a device factor cannot be sharded (use factor())")

    def export(self) -> dict:
        p = self._prob
        nx, nu, n, F, L = p.nx, p.nu, p.num_nodes(), p.first_leaf, p.num_leaves
        S = int(p.flat()["stage_rows"].sum())
        out = dict(gain=np.zeros(F * nu * nx), child_to_input=np.zeros(n * nu * nx),
                   closed_loop=np.zeros(n * nx * nx), dual_to_input=np.zeros(max(S, 1) * nu),
                   dual_to_costate=np.zeros(max(S, 1) * nx), input_affine=np.zeros(F * nu),
                   costate_affine=np.zeros(F * nx), value_quad=np.zeros(n * nx * nx),
                   leaf_costate_affine=np.zeros(L * nx))
        check(N.lib().scenopt_dev_factor_export(self._dev, p._h, *[dptr(out[k]) for k in (
            "gain", "child_to_input", "closed_loop", "dual_to_input", "dual_to_costate",
            "input_affine", "costate_affine", "value_quad", "leaf_costate_affine")]))
        return out


def factor_device(prob: ProblemInstance, device: int = 0) -> DeviceFactorCache:
    """riccati.hpp:82-182 on the GPU (no host factor, no factor upload)."""
    return DeviceFactorCache(prob, device)


def factor(prob: ProblemInstance) -> FactorCache:
    """riccati.hpp:82-182."""
    h = C.c_void_p()
    check(N.lib().scenopt_factor_create(prob._h, C.byref(h)))
    return FactorCache(h, prob)


def refactor_affine(cache: FactorCache, prob: ProblemInstance) -> None:
    """riccati.hpp:187-216: new linear terms (q, r, c, p_N) with the same
    matrices. A device-factored cache recomputes them on the GPU and moves
    only the vectors (scenopt_dev_refactor_affine)."""
    if isinstance(cache, DeviceFactorCache):
        _check_shapes(cache, prob, "refactor_affine")
        check(N.lib().scenopt_dev_refactor_affine(cache._dev, prob._h))
        return
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


def grad_fhat(cache: FactorCache, prob: ProblemInstance, y, stats: OracleStats | None = None):
    """tree_oracles.hpp:117-121: -H x(y)."""
    return -apply_H(prob, dual_grad(cache, prob, y, stats), cache)


def fhat_value(cache: FactorCache, prob: ProblemInstance, y, stats: OracleStats | None = None):
    """tree_oracles.hpp:125-129."""
    _check_shapes(cache, prob, "fhat_value")
    yv = _dual(prob, y, "fhat_value")
    out = C.c_double()
    check(N.lib().scenopt_fhat_value(cache.device(), dptr(yv), C.byref(out), HOST))
    if stats is not None:
        stats.dual_grad_calls += 1
    return out.value


def apply_H(prob: ProblemInstance, pt: PrimalPoint, cache: FactorCache | None = None):
    """problem_data.hpp:144-162 (on the device of `cache`, or of a
    factor-less handle of `prob`)."""
    dev = cache.device() if cache is not None else _lite(prob)
    x = np.ascontiguousarray(pt.x, dtype=np.float64).ravel(order="F")
    u = np.ascontiguousarray(pt.u, dtype=np.float64).ravel(order="F")
    if x.size != prob.nx * prob.num_nodes() or u.size != prob.nu * prob.first_leaf:
        raise N.DimensionMismatch("apply_H: point does not match the instance")
    z = np.zeros(prob.dual_dim)
    check(N.lib().scenopt_apply_H(dev, dptr(np.ascontiguousarray(x)), dptr(np.ascontiguousarray(u)),
                                  dptr(z), HOST))
    return z


_LITE = {}


def _lite(prob: ProblemInstance):
    """Factor-less device handle (apply_H / prox / verification)."""
    key = id(prob)
    h = _LITE.get(key)
    if h is None or h[0] is not prob:
        dev = C.c_void_p()
        check(N.lib().scenopt_dev_create(prob._h, None, 0, C.byref(dev)))
        _LITE[key] = (prob, dev)
        return dev
    return h[1]


# ---------------------------------------------------------------- nonsmooth
class Nonsmooth:
    """SeparableNonsmooth bound to a problem (prox.hpp:24-52)."""

    def __init__(self, prob: ProblemInstance, cache: FactorCache | None = None):
        self.prob = prob
        self.dim = prob.dual_dim
        self._dev = cache.device() if cache is not None else _lite(prob)

    def prox(self, v, gamma_prox):
        out = np.zeros(self.dim)
        check(N.lib().scenopt_prox_g(self._dev, dptr(_dual(self.prob, v, "prox_g")),
                                     C.c_double(gamma_prox), dptr(out), HOST))
        return out

    def conj(self, w):
        out = C.c_double()
        check(N.lib().scenopt_conj_value_g(self._dev, dptr(_dual(self.prob, w, "conj_value_g")),
                                           C.byref(out), HOST))
        return out.value

    def dist_subdiff_inf(self, y, z):
        out = C.c_double()
        check(N.lib().scenopt_dist_subdiff_inf(self._dev, dptr(_dual(self.prob, y, "dist")),
                                               dptr(_dual(self.prob, z, "dist")), C.byref(out), HOST))
        return out.value


def make_nonsmooth(prob: ProblemInstance, cache: FactorCache | None = None) -> Nonsmooth:
    return Nonsmooth(prob, cache)


# ---------------------------------------------------------------- FBE
@dataclass
class FbState:
    """fbe.hpp:22-34."""

    y: np.ndarray
    lam: float
    x: PrimalPoint
    Hx: np.ndarray
    z: np.ndarray
    T: np.ndarray
    R: np.ndarray
    fhat: float
    conj_T: float
    znorm_sq: float
    value: float


def fb_step(cache: FactorCache, prob: ProblemInstance, y, lam: float,
            stats: OracleStats | None = None) -> FbState:
    """fbe.hpp:55-67 (one dual_grad sweep + fused prox / conjugate / FBE)."""
    _check_shapes(cache, prob, "fb_step")
    yv = _dual(prob, y, "fb_step")
    x, u = _primal_out(prob)
    D = prob.dual_dim
    Hx, z, R, T = np.zeros(D), np.zeros(D), np.zeros(D), np.zeros(D)
    sc = np.zeros(4)
    check(N.lib().scenopt_fb_step(cache.device(), dptr(yv), C.c_double(lam), dptr(x), dptr(u),
                                  dptr(Hx), dptr(z), dptr(R), dptr(T), dptr(sc), HOST))
    if stats is not None:
        stats.dual_grad_calls += 1
        stats.prox_calls += 1
        stats.conj_calls += 1
    return FbState(yv.copy(), lam, _pp(prob, x, u), Hx, z, T, R, sc[0], sc[1], sc[2], sc[3])


def fbe_value(state: FbState) -> float:
    """fbe.hpp:82-86."""
    if not np.isfinite(state.value):
        raise N.InfiniteConjugate("fbe_value: g*(T) is infinite")
    return state.value


def fbe_grad(state: FbState, cache: FactorCache, prob: ProblemInstance,
             stats: OracleStats | None = None):
    """fbe.hpp:89-94: R + lam H x0(R)."""
    out = np.zeros(prob.dual_dim)
    check(N.lib().scenopt_fbe_grad(cache.device(), dptr(_dual(prob, state.R, "fbe_grad")),
                                   C.c_double(state.lam), dptr(out), HOST))
    if stats is not None:
        stats.hessian_vec_calls += 1
    return out


def linesearch_cert(cache: FactorCache, prob: ProblemInstance, state: FbState, direction, taus,
                    shift=None) -> dict:
    """linesearch_cert / linesearch_cert_shifted + evaluate_cert at `taus`
    (fbe.hpp:136-231). Returns deltas, the certificate scalars, cert_fhat(tau)
    and w / Hx_w / z / R / T of the last tau."""
    D = prob.dual_dim
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    deltas, cfh, cs = np.zeros(len(taus)), np.zeros(len(taus)), np.zeros(6)
    w, Hxw, z, R, T = (np.zeros(D) for _ in range(5))
    ss = np.array([state.fhat, state.conj_T, state.znorm_sq, state.value])
    sh = None if shift is None else _dual(prob, shift, "shift")
    check(N.lib().scenopt_linesearch_cert(
        cache.device(), dptr(_dual(prob, state.y, "y")), dptr(_dual(prob, state.Hx, "Hx")),
        C.c_double(state.lam), dptr(ss), dptr(sh), dptr(_dual(prob, direction, "dir")),
        len(taus), dptr(taus), dptr(deltas), dptr(cs), dptr(cfh), dptr(w), dptr(Hxw), dptr(z),
        dptr(R), dptr(T), HOST))
    return dict(deltas=deltas, alpha1=cs[0], alpha2=cs[1], conj_anchor=cs[2],
                znorm_sq_anchor=cs[3], value_anchor=cs[4], fhat_anchor=cs[5], cert_fhat=cfh,
                w=w, Hx_w=Hxw, z=z, R=R, T=T)


# ---------------------------------------------------------------- L-BFGS
class LbfgsBuffer:
    """lbfgs.hpp:22-84 with device-resident pairs (on `cache`'s device)."""

    def __init__(self, memory: int, eps_curv: float, cache: FactorCache):
        self._h = C.c_void_p()
        check(N.lib().scenopt_lbfgs_create(cache.device(), memory, C.c_double(eps_curv),
                                           C.byref(self._h)))
        self._cache = cache
        self._memory = memory

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.scenopt_lbfgs_destroy(self._h)
            self._h = None

    def push(self, step, change, scale_ref) -> bool:
        s = np.ascontiguousarray(step, np.float64)
        q = np.ascontiguousarray(change, np.float64)
        return bool(check(N.lib().scenopt_lbfgs_push(self._h, len(s), dptr(s), dptr(q),
                                                     C.c_double(scale_ref))))

    def apply_direction(self, grad):
        g = np.ascontiguousarray(grad, np.float64)
        out = np.zeros(len(g))
        check(N.lib().scenopt_lbfgs_apply(self._h, len(g), dptr(g), dptr(out)))
        return out

    def clear(self):
        check(N.lib().scenopt_lbfgs_clear(self._h))

    def size(self) -> int:
        return check(N.lib().scenopt_lbfgs_size(self._h))

    def memory(self) -> int:
        return self._memory

    def gamma0(self) -> float:
        return float(N.lib().scenopt_lbfgs_gamma0(self._h))


# ---------------------------------------------------------------- solvers
BACKTRACKING = {"original": 0, "simple": 1, "none": 2}
KINDS = {"minfbe": 0, "nama": 1, "gpad": 2}


@dataclass
class SolverConfig:
    """solvers.hpp:28-46."""

    lambda0: float = 0.0
    eps: float = 5e-4
    eps_curv: float = 1e-12
    eps_bt: float = 0.25
    beta_bt: float = 0.05
    memory: int = 5
    max_iters: int = 20000
    backtracking_rule: str = "simple"
    warm_start: bool = False
    warm_start_iters: int = 5
    precondition: bool = False
    nama_parallel_linesearch: bool = False
    nama_update_tlambda: bool = True

    def c(self):
        return N.SolverConfigC(self.lambda0, self.eps, self.eps_curv, self.eps_bt, self.beta_bt,
                               self.memory, self.max_iters,
                               BACKTRACKING[self.backtracking_rule], int(self.warm_start),
                               self.warm_start_iters, int(self.precondition),
                               int(self.nama_parallel_linesearch), int(self.nama_update_tlambda))


@dataclass
class SolverReport:
    """solvers.hpp:66-84."""

    status: str
    x: PrimalPoint
    y: np.ndarray
    z: np.ndarray
    residual_inf: float
    iterations: int
    stats: OracleStats
    lipschitz_calls: int
    lipschitz_estimate: float
    lambda_final: float
    eps: float
    residual_trace: np.ndarray
    fbe_trace: np.ndarray
    wall_ms: float
    verified: bool
    verify_residual_inf: float
    verify_subdiff_dist: float
    _h: object = field(default=None, repr=False)

    def __del__(self):
        if getattr(self, "_h", None) is not None and N._lib is not None:
            N._lib.scenopt_report_destroy(self._h)
            self._h = None


def _report(prob: ProblemInstance, h) -> SolverReport:
    s = N.ReportSummaryC()
    check(N.lib().scenopt_report_summary_get(h, C.byref(s)))
    x, u = _primal_out(prob)
    D = prob.dual_dim
    y, z = np.zeros(D), np.zeros(D)
    rt, ft = np.zeros(s.trace_len), np.zeros(s.trace_len)
    check(N.lib().scenopt_report_arrays(h, dptr(x), dptr(u), dptr(y), dptr(z), dptr(rt), dptr(ft)))
    return SolverReport(
        status="converged" if s.status == 0 else "max_iters_exceeded", x=_pp(prob, x, u), y=y, z=z,
        residual_inf=s.residual_inf, iterations=s.iterations,
        stats=OracleStats(s.dual_grad_calls, s.hessian_vec_calls, s.prox_calls, s.conj_calls),
        lipschitz_calls=s.lipschitz_calls, lipschitz_estimate=s.lipschitz_estimate,
        lambda_final=s.lambda_final, eps=s.eps, residual_trace=rt, fbe_trace=ft,
        wall_ms=s.wall_ms, verified=bool(s.verified), verify_residual_inf=s.verify_residual_inf,
        verify_subdiff_dist=s.verify_subdiff_dist, _h=h)


def estimate_dual_lipschitz(cache: FactorCache, prob: ProblemInstance, rel_tol: float = 1e-6,
                            max_rounds: int = 100):
    """solvers.hpp:89-113 -> (estimate, sweeps)."""
    _check_shapes(cache, prob, "estimate_dual_lipschitz")
    calls = C.c_uint64()
    out = C.c_double()
    check(N.lib().scenopt_estimate_lipschitz_ex(cache.device(), C.c_double(rel_tol), int(max_rounds),
                                                C.byref(calls), C.byref(out)))
    return out.value, int(calls.value)


def _solve_direct(kind, prob, cache, cfg, y0=None, residual_weight=None):
    _check_shapes(cache, prob, "solve")
    y0v = None if y0 is None else _dual(prob, y0, "y0")
    wv = None if residual_weight is None else _dual(prob, residual_weight, "weight")
    h = C.c_void_p()
    c = cfg.c()
    check(N.lib().scenopt_dev_solve(cache.device(), C.byref(c), KINDS[kind], dptr(y0v), dptr(wv),
                                    C.byref(h)))
    return _report(prob, h)


def solve_minfbe(prob, cache, cfg: SolverConfig, y0=None, residual_weight=None) -> SolverReport:
    """solvers.hpp:234-356."""
    return _solve_direct("minfbe", prob, cache, cfg, y0, residual_weight)


def solve_nama(prob, cache, cfg: SolverConfig, y0=None, residual_weight=None) -> SolverReport:
    """solvers.hpp:362-492."""
    return _solve_direct("nama", prob, cache, cfg, y0, residual_weight)


def solve_gpad(prob, cache, cfg: SolverConfig, y0=None, residual_weight=None) -> SolverReport:
    """solvers.hpp:498-540."""
    return _solve_direct("gpad", prob, cache, cfg, y0, residual_weight)


def warm_start(prob, cache, cfg: SolverConfig, lam: float):
    """solvers.hpp:545-564 -> (y, dual_grad_calls)."""
    y = np.zeros(prob.dual_dim)
    dg = C.c_uint64()
    c = cfg.c()
    check(N.lib().scenopt_warm_start(cache.device(), C.byref(c), C.c_double(lam), dptr(y),
                                     C.byref(dg)))
    return y, int(dg.value)


def solve(prob: ProblemInstance, cfg: SolverConfig, kind: str = "nama",
          shared_cache: FactorCache | None = None, device: int = 0) -> SolverReport:
    """solvers.hpp:645-720: precondition, factor, Lipschitz estimate, warm
    start, solver run and independent verification."""
    h = C.c_void_p()
    c = cfg.c()
    check(N.lib().scenopt_solve(prob._h, C.byref(c), KINDS[kind],
                                shared_cache._h if shared_cache is not None else None, device,
                                C.byref(h)))
    return _report(prob, h)


def verify_report(prob: ProblemInstance, rep: SolverReport, z_override=None, device: int = 0):
    """solvers.hpp:630-639 (recomputes the verify_* fields in place)."""
    zo = None if z_override is None else _dual(prob, z_override, "z")
    check(N.lib().scenopt_verify_report(prob._h, rep._h, dptr(zo), device))
    new = _report(prob, rep._h)
    rep.verified, rep.verify_residual_inf, rep.verify_subdiff_dist = (
        new.verified, new.verify_residual_inf, new.verify_subdiff_dist)
    new._h = None
    if zo is not None:
        rep.z = zo.copy()
    return rep


# ---------------------------------------------------------------- experiment.hpp
RESULTS_CSV_HEADER = ("instance_id,solver,iterations,dual_grad_calls,hessian_vec_calls,"
                      "prox_calls,final_residual_inf,wall_ms,converged")  # experiment.hpp:133-135


@dataclass
class SolverSpec:
    """experiment.hpp:26-30; p-NAMA is NAMA with the parallel line search."""
    name: str
    kind: str = "nama"
    parallel_linesearch: bool = False


def solver_spec_from_name(name: str) -> SolverSpec:
    """experiment.hpp:32-40."""
    table = {"minfbe": SolverSpec("minfbe", "minfbe"), "nama": SolverSpec("nama", "nama"),
             "pnama": SolverSpec("pnama", "nama", True), "gpad": SolverSpec("gpad", "gpad")}
    if name not in table:
        raise InvalidParams(f'unknown solver "{name}"; expected minfbe, nama, pnama, or gpad')
    return table[name]


def default_solver_set() -> list:
    return [solver_spec_from_name(n) for n in ("minfbe", "nama", "gpad")]


@dataclass
class BatchEntry:
    id: str
    prob: ProblemInstance


@dataclass
class ExperimentRow:
    """experiment.hpp:63-80."""
    instance_id: str
    solver: str
    iterations: int
    dual_grad_calls: int
    hessian_vec_calls: int
    prox_calls: int
    final_residual_inf: float
    wall_ms: float
    converged: bool
    fbe_monotone: bool
    error: str
    residual_trace: np.ndarray

    def oracle_calls(self) -> int:
        return self.dual_grad_calls + self.hessian_vec_calls


@dataclass
class SolverSummary:
    """experiment.hpp:86-96."""
    solver: str
    count: int
    converged: int
    median_calls: float
    p84_calls: float
    p95_calls: float
    frac_within_50: float
    fbe_violations: int
    total_wall_ms: float


class RunReport:
    """experiment.hpp:136-214 (rendered by the native library)."""

    def __init__(self, handle):
        self._h = handle
        self.metadata: dict = {}
        self.rows = []
        k = N.lib().scenopt_experiment_row_count(handle)
        r = N.ExperimentRowC()
        for i in range(k):
            check(N.lib().scenopt_experiment_row_get(handle, i, C.byref(r)))
            tr = (np.ctypeslib.as_array(r.residual_trace, shape=(r.trace_len,)).copy()
                  if r.trace_len else np.zeros(0))
            self.rows.append(ExperimentRow(r.instance_id.decode(), r.solver.decode(), r.iterations,
                                           r.dual_grad_calls, r.hessian_vec_calls, r.prox_calls,
                                           r.final_residual_inf, r.wall_ms, bool(r.converged),
                                           bool(r.fbe_monotone), r.error.decode(), tr))

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.scenopt_experiment_destroy(self._h)
            self._h = None

    def _text(self, which: int, meta=None) -> str:
        import json
        m = json.dumps(meta).encode() if meta is not None else None
        n = C.c_size_t()
        check(N.lib().scenopt_experiment_text(self._h, which, m, None, C.c_size_t(0), C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(N.lib().scenopt_experiment_text(self._h, which, m, buf, C.c_size_t(n.value + 1), C.byref(n)))
        return buf.raw[:n.value].decode()

    def csv(self) -> str:
        return self._text(0)

    def traces_csv(self) -> str:
        return self._text(1)

    def summary_json(self) -> str:
        """summary_json().dump(2) + "\\n" (the report file's text)."""
        return self._text(2, self.metadata)

    def summaries(self) -> list:
        out = (N.SolverSummaryC * 16)()
        k = check(N.lib().scenopt_experiment_summaries(self._h, out, 16))
        return [SolverSummary(s.solver.decode(), s.count, s.converged, s.median_calls, s.p84_calls,
                              s.p95_calls, s.frac_within_50, s.fbe_violations, s.total_wall_ms)
                for s in out[:k]]


def run_experiment(instances, solvers=None, solver: SolverConfig | None = None,
                   include_timing: bool = True, reuse_factors: bool = True, device: int = 0) -> RunReport:
    """experiment.hpp:222-283: every solver on every instance, in order.
    `instances` are BatchEntry or (id, ProblemInstance) pairs; `solvers` are
    SolverSpec or names (default: minfbe, nama, gpad)."""
    entries = [e if isinstance(e, BatchEntry) else BatchEntry(*e) for e in instances]
    specs = default_solver_set() if solvers is None else [
        s if isinstance(s, SolverSpec) else solver_spec_from_name(s) for s in solvers]
    probs = (C.c_void_p * max(len(entries), 1))(*[e.prob._h for e in entries])
    ids = (C.c_char_p * max(len(entries), 1))(*[e.id.encode() for e in entries])
    names = (C.c_char_p * max(len(specs), 1))(*[s.name.encode() for s in specs])
    c = (solver or SolverConfig()).c()
    h = C.c_void_p()
    check(N.lib().scenopt_run_experiment(probs, ids, len(entries), names, len(specs), C.byref(c),
                                         int(include_timing), int(reuse_factors), device, C.byref(h)))
    return RunReport(h)
