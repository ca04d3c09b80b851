"""ctypes binding of libscenopt_b200.so (include/scenopt_b200.h).

The library is built in-tree (``make -C paper_2107_01745_b200``, or
``__graft_entry__.build()``); importing a device entry point without it
raises immediately — there is no Python or CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCENOPT_LIBRARY") or os.path.join(_HERE, "lib", "libscenopt_b200.so")

I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)
HOST_IO = 1


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


class DevInfoC(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("sm_count", C.c_int32), ("grid_ctas", C.c_int32),
        ("ctas_per_sm", C.c_int32), ("slots", C.c_int32), ("items_bw", C.c_int32),
        ("items_fw", C.c_int32), ("nodes_per_item_max", C.c_int32),
        ("slot_bytes", C.c_int64), ("matrix_bytes_bw", C.c_int64),
        ("matrix_bytes_fw", C.c_int64), ("device_bytes", C.c_int64),
        ("sweep_bytes_hom", C.c_int64), ("sweep_bytes_aff", C.c_int64),
        ("sweep_bytes_hom2", C.c_int64), ("cut_stage", C.c_int32), ("shard_stage", C.c_int32),
        ("rank", C.c_int32), ("world", C.c_int32), ("shard_first", C.c_int32), ("shard_past", C.c_int32),
        ("items_global", C.c_int32), ("consumer_stage", C.c_int32),
        ("flat_top", C.c_int32), ("device_factor", C.c_int32), ("producer_warps", C.c_int32),
        ("exchange_doubles", C.c_int64),
    ]


class ExperimentRowC(C.Structure):
    _fields_ = [
        ("instance_id", C.c_char_p), ("solver", C.c_char_p), ("error", C.c_char_p),
        ("iterations", C.c_int32), ("dual_grad_calls", C.c_uint64), ("hessian_vec_calls", C.c_uint64),
        ("prox_calls", C.c_uint64), ("final_residual_inf", C.c_double), ("wall_ms", C.c_double),
        ("converged", C.c_int32), ("fbe_monotone", C.c_int32), ("trace_len", C.c_int32),
        ("residual_trace", F64P),
    ]


class SolverSummaryC(C.Structure):
    _fields_ = [
        ("solver", C.c_char * 16), ("count", C.c_int32), ("converged", C.c_int32),
        ("fbe_violations", C.c_int32), ("median_calls", C.c_double), ("p84_calls", C.c_double),
        ("p95_calls", C.c_double), ("frac_within_50", C.c_double), ("total_wall_ms", C.c_double),
    ]


class SpringMassC(C.Structure):
    """scenopt_spring_mass_params (generators.hpp:49-64)."""
    _fields_ = [
        ("mass_kg", C.c_double), ("stiffness", C.c_double), ("damping", C.c_double),
        ("input_bound", C.c_double), ("velocity_bound", C.c_double), ("horizon", C.c_int32),
        ("sampling", C.c_double), ("state_weight", C.c_double), ("input_weight", C.c_double),
        ("terminal_weight", C.c_double), ("initial_len", C.c_int32), ("transition_rows", C.c_int32),
        ("transition_cols", C.c_int32), ("mode_values_len", C.c_int32), ("root_state_len", C.c_int32),
        ("initial_probs", F64P), ("transition", F64P), ("mode_values", F64P), ("root_state", F64P),
    ]


# errors.hpp:9-80 -> Python exception types with the reference's names.
class Error(RuntimeError):
    code = -1


def _mk(name, code):
    return type(name, (Error,), {"code": code})


NonStochasticMatrix = _mk("NonStochasticMatrix", -2)
StageOutOfRange = _mk("StageOutOfRange", -3)
DimensionMismatch = _mk("DimensionMismatch", -4)
UnsupportedSpec = _mk("UnsupportedSpec", -5)
NotStronglyConvex = _mk("NotStronglyConvex", -6)
ShapeChanged = _mk("ShapeChanged", -7)
CacheMismatch = _mk("CacheMismatch", -8)
LineSearchStalled = _mk("LineSearchStalled", -9)
StepUnderflow = _mk("StepUnderflow", -10)
ZeroProbability = _mk("ZeroProbability", -11)
InvalidParams = _mk("InvalidParams", -12)
InfiniteConjugate = _mk("InfiniteConjugate", -13)
ParseError = _mk("ParseError", -14)
CudaError = _mk("CudaError", -20)
NcclError = _mk("NcclError", -21)
OutOfMemory = _mk("OutOfMemory", -22)
NoDevice = _mk("NoDevice", -23)

_BY_CODE = {cls.code: cls for cls in (
    NonStochasticMatrix, StageOutOfRange, DimensionMismatch, UnsupportedSpec, NotStronglyConvex,
    ShapeChanged, CacheMismatch, LineSearchStalled, StepUnderflow, ZeroProbability, InvalidParams,
    InfiniteConjugate, ParseError, CudaError, NcclError, OutOfMemory, NoDevice)}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA/C++ library for sm_100a in-tree (nvcc cross-compiles)."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-j8", "-C", _HERE], check=True, stdout=out)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                "(the scenopt_b200 hot path has no fallback implementation)")
        if not os.environ.get("SCENOPT_NCCL_LIBRARY"):
            # NCCL is loaded by the library on first use (sharded handles);
            # point it at the framework's own build when one is installed, so
            # a later `import torch` finds the libnccl.so.2 it was built against
            import importlib.util
            spec = importlib.util.find_spec("nvidia.nccl")
            for loc in (spec.submodule_search_locations or []) if spec else []:
                cand = os.path.join(loc, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["SCENOPT_NCCL_LIBRARY"] = cand
                    break
        L = C.CDLL(LIB_PATH)
        L.scenopt_last_error.restype = C.c_char_p
        if hasattr(L, "scenopt_lbfgs_gamma0"):
            L.scenopt_lbfgs_gamma0.restype = C.c_double
        _lib = L
    return _lib


def check(rc: int) -> int:
    if rc < 0:
        msg = lib().scenopt_last_error().decode()
        raise _BY_CODE.get(rc, Error)(msg)
    return rc


def dptr(a):
    """double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(F64P)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(I32P)


def view_from_flat(flat: dict):
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
