"""B200-native horizon-partitioned Riccati solve (arXiv 1809.06360).

Drop-in for the hot path of the reference package ``parlqr``:
``solve_parallel`` keeps ``parlqr.solve_parallel``'s signature, partition
rules, error contract and result types (the reference's own classes when
``parlqr`` is importable, see ``compat.py``), and runs on hand-written sm_100a
CUDA kernels (``libparlqr_b200.so``, C ABI in ``include/parlqr_b200.h``).
"""

from .errors import (CholeskyFailure, FactorizationFailure, Infeasible, LinkSingular,
                     SingularKkt, SolverError, UnsupportedPartition)
from .problem import (DEFAULT_TOLERANCES, USING_REFERENCE_TYPES, AffinePolicy, LqrProblem, LqrSolution,
                      StageCost, StageDynamics, TerminalCost, ToleranceSet, problem_from_arrays)
from .parallel import (BatchSolver, HostSolver, ParallelDetails, Partition, default_workers,
                       make_partition, smooth, solve_parallel, solve_parallel_batch, solve_parallel_host,
                       stack_problem)

from .endpoint import (EndpointAffineSolution, EndpointBatch, solve_endpoint, solve_endpoint_affine,
                       solve_endpoint_batch)

__version__ = "0.1.0"

__all__ = [
    "AffinePolicy", "BatchSolver", "CholeskyFailure", "DEFAULT_TOLERANCES", "FactorizationFailure",
    "HostSolver", "Infeasible", "LinkSingular", "LqrProblem", "LqrSolution", "ParallelDetails",
    "Partition", "SingularKkt", "SolverError", "StageCost", "StageDynamics", "TerminalCost",
    "ToleranceSet", "UnsupportedPartition", "default_workers", "make_partition", "solve_parallel",
    "problem_from_arrays", "USING_REFERENCE_TYPES",
    "smooth", "solve_parallel_batch", "solve_parallel_host", "stack_problem",
    "EndpointAffineSolution", "EndpointBatch", "solve_endpoint", "solve_endpoint_affine", "solve_endpoint_batch",
]
