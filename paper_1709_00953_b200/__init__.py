"""B200-native randomized block row/column gradient solver (CSGD / GCSGD,
arXiv 1709.00953), a drop-in for the reference package ``blockct``'s solver
path: hand-written sm_100a kernels behind a C ABI (include/blockct.h), with
the reference's Python solver API on the host.  No CPU fallback."""

from .baselines import BaselineParams, run_column_action, run_row_action
from .errors import (BlockCTError, BudgetExceededError, ConfigurationError, DivergenceError,
                     ExecutorError, GeometryError, NativeLibraryError, ScheduleError)
from .executor import EpochExecutor, EpochStats, TaskDescriptor
from .geometry import CONFIGS, ParallelBeamSpec, ProblemConfig, add_noise, random_ellipses
from .metrics import ConvergenceTrace, TraceRow, observation_gap_db, snr_db
from .sampling import (BlockScheduler, ProbabilityTable, SamplingConfig, ScriptedScheduler,
                       dump_schedule, mixed_weights, parse_schedule, select_column_blocks,
                       select_row_blocks)
from .solvers import (SolverParams, SolverState, audit_state, basic_iteration, run_csgd,
                      run_gcsgd)
from .system import DeviceBlockSystem, PanelArrays

__version__ = "0.1.0"

__all__ = [
    "BlockCTError", "BudgetExceededError", "ConfigurationError", "DivergenceError",
    "ExecutorError", "GeometryError", "NativeLibraryError", "ScheduleError",
    "EpochExecutor", "EpochStats", "TaskDescriptor",
    "CONFIGS", "ParallelBeamSpec", "ProblemConfig", "add_noise", "random_ellipses",
    "ConvergenceTrace", "TraceRow", "observation_gap_db", "snr_db",
    "BlockScheduler", "ProbabilityTable", "SamplingConfig", "ScriptedScheduler",
    "dump_schedule", "mixed_weights", "parse_schedule", "select_column_blocks",
    "select_row_blocks",
    "SolverParams", "SolverState", "audit_state", "basic_iteration", "run_csgd", "run_gcsgd",
    "DeviceBlockSystem", "PanelArrays",
    "BaselineParams", "run_row_action", "run_column_action",
]
