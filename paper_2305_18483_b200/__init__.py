"""B200-native RDROT (regularized Douglas-Rachford optimal transport) hot path.

Drop-in for the reference otdr solver API (proj/include/otdr): the DR
iteration, its stopping logic, the objective and the duality certificate run in
hand-written sm_100a kernels (csrc/) behind the C-ABI in include/otdr_dev.h.
"""
from .otdr import (  # noqa: F401
    BatchEngine, DeviceError, DimensionMismatch, DualCertificate, Engine, GroupLassoReg, GroupPartition,
    InvalidArgument, MarginalSumOutOfRange, NegativeEntry, NonFiniteIterate, OtdrError, Problem,
    QuadraticReg, Regularizer, Shard, SolveReport, SolverOptions, SolverState, Termination,
    TraceRow, Unsupported, WarmStart, ZeroIterations, ZeroReg, column_class_blocks,
    compute_skip_count, default_init, default_stepsize, duality_gap, link_local, make_partition, make_state,
    normalize_cost, ot_cost_gradient, primal_objective, recover_duals, solve, solve_batch, step,
    to_string,
    validate_problem,
)

__version__ = "0.1.0"
