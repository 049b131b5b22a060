"""B200-native FFT block-Toeplitz matvec (arXiv 2407.13066) — the hot path of
the reference ``btoep`` library, behind its own operator API.

Compute runs only in ``libbtg.so`` (hand-written sm_100a CUDA, C ABI in
``include/btg.h``); this package is the host-side mirror of the reference's
Python surface (operator, solver, files) plus the multi-GPU grid
(``distributed``).
"""

from ._lib import DimensionError, Error, FormatError, GridError, OrderingError, SolverError  # noqa: F401
from .distributed import Partition, distributed_adjoint, distributed_forward, partition_operator  # noqa: F401
from .io import (load_operator, peek_operator, read_operator, read_vector, save_operator,  # noqa: F401
                 write_operator, write_vector)
from .operator import (HessianOperator, SpectralOperator, create, fill_uniform, naive_apply_adjoint,  # noqa: F401
                       naive_apply_forward, setup)
from .planner import (apply_arithmetic_intensity, comm_cost, conventional_cost_estimate, modified_cost,  # noqa: F401
                      parse_grid, plan_grid, select_grid, weak_scaling_shape)
from .solver import cg_solve, cg_solve_op, objective_eval  # noqa: F401

__all__ = [
    "DimensionError",
    "Error",
    "FormatError",
    "GridError",
    "OrderingError",
    "Partition",
    "SolverError",
    "HessianOperator",
    "SpectralOperator",
    "apply_arithmetic_intensity",
    "cg_solve",
    "conventional_cost_estimate",
    "distributed_adjoint",
    "distributed_forward",
    "comm_cost",
    "modified_cost",
    "parse_grid",
    "plan_grid",
    "select_grid",
    "weak_scaling_shape",
    "cg_solve_op",
    "create",
    "fill_uniform",
    "load_operator",
    "naive_apply_adjoint",
    "naive_apply_forward",
    "objective_eval",
    "partition_operator",
    "peek_operator",
    "read_operator",
    "read_vector",
    "save_operator",
    "setup",
    "write_operator",
    "write_vector",
]
