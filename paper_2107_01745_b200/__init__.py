"""scenopt_b200 — B200-native MINFBE / NAMA hot path (arXiv 2107.01745).

The public surface mirrors the reference's ``scenopt`` C++ API
(/root/reference/proj/include/scenopt/); the numerics run in the in-tree
CUDA library ``lib/libscenopt_b200.so`` (include/scenopt_b200.h).
"""
from ._native import (  # noqa: F401
    CacheMismatch, CudaError, DimensionMismatch, Error, InfiniteConjugate, InvalidParams,
    LineSearchStalled, NoDevice, NonStochasticMatrix, NotStronglyConvex, ParseError, ShapeChanged,
    StageOutOfRange, StepUnderflow, UnsupportedSpec,
    ZeroProbability, build, lib,
)
from .api import *  # noqa: F401,F403
from .api import (  # noqa: F401
    FactorCache, OracleStats, PrimalPoint, ProblemInstance, dual_grad, factor,
    gen_random_instance, hessian_vec, precondition, refactor_affine, sweep,
)


def device_count() -> int:
    """Number of visible sm_100 devices (0 on a GPU-less host)."""
    return int(lib().scenopt_device_count())
