"""B200-native inexact policy iteration (iPI) hot path.

Drop-in for the reference ``mdpsolve`` / ``mdpsolve_frontend`` API on the path
named by the north star: Bellman backup (fused sm_100a kernel), policy
compaction, GMRES/Richardson policy evaluation (persistent cooperative
kernel) and the outer iPI loop, all in ``libipi_b200.so`` (C ABI in
``include/ipi_b200.h``).  There is no CPU fallback: compute entry points raise
when the CUDA library or a GPU is missing.
"""

from .errors import DimensionError, ResourceLimitError, ValidationError
from .model import (MdpInstance, Mode, Partition, ROW_SUM_TOL, flatten_index, make_partition,
                    require_valid, validate)
from .sparse import (CsrMatrix, DeviceOperator, PolicyOperator, dot, gather_policy_cost, gather_policy_matrix,
                     norm, spmv)
from .bellman import GreedyResult, bellman_residual, greedy_policy, policy_residual
from .inner import (GMRES_RESTART, TARGET_FLOOR_SCALE, InnerSolver, InnerSolveReport,
                    Preconditioner, build_preconditioner, inner_solve)
from .driver import STALL_WINDOW, SolveOptions, SolveResult, SolveStatus, preset, solve
from .fileio import FileFormatError, read_matrix, write_matrix

__version__ = "0.1.0"

__all__ = [
    "CsrMatrix", "DeviceOperator", "DimensionError", "FileFormatError", "GMRES_RESTART", "GreedyResult",
    "InnerSolveReport", "InnerSolver", "MdpInstance", "Mode", "Partition", "PolicyOperator",
    "Preconditioner", "ROW_SUM_TOL", "ResourceLimitError", "STALL_WINDOW", "SolveOptions",
    "SolveResult", "SolveStatus", "TARGET_FLOOR_SCALE", "ValidationError", "bellman_residual",
    "build_preconditioner", "dot", "flatten_index", "gather_policy_cost", "gather_policy_matrix",
    "greedy_policy", "inner_solve", "make_partition", "norm", "policy_residual", "preset",
    "read_matrix", "require_valid", "solve", "spmv", "validate", "write_matrix",
]
