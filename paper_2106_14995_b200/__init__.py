"""B200-native batched trust-region Newton (TRON) solver — drop-in for the
reference tronbatch::solve_batch path."""
from .tron import (  # noqa: F401
    BatchResult,
    EvaluationError,
    Family,
    FactorizationError,
    KernelForm,
    LaunchOrder,
    ImbalanceStats,
    ProblemBatch,
    SingularFactorError,
    SolveReport,
    SolveStatus,
    Solver,
    SolverError,
    TronConfig,
    family_nparams,
    imbalance,
    solve_batch,
)
