"""Whole-system cyclic baselines on the device: the reference's
``BaselineParams``, ``run_row_action`` and ``run_column_action``
(src/blockct/solvers.py:283-379) with the same signatures, running on the
context's own system matrix through ``bct_baseline_*`` (csrc/baseline.cu).

The reference builds A with ``BlockSystem.to_scipy`` (projector.py:779-793)
and sweeps it with scipy; the device assembles the same CSR/CSC from its
panels and reproduces scipy's operation order, so x is bitwise equal to the
reference's on the same A.  Like the rest of the product there is no CPU
path: a missing library raises NativeLibraryError.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .metrics import ConvergenceTrace, TraceRow, snr_from_sq
from .validation import as_vector, check_choice, check_count, check_positive

M_RULES = ("identity", "sum_inverse", "norm_inverse")   # solvers.py:43


@dataclass(frozen=True)
class BaselineParams:
    """Cyclic baseline knobs (solvers.py:287-300): relaxation omega and the
    diagonal scaling rule (identity, sum_inverse or norm_inverse)."""

    epochs: int
    omega: float = 1.0
    m_rule: str = "norm_inverse"

    def __post_init__(self):
        check_count("epochs", self.epochs, minimum=0)
        check_positive("omega", self.omega)
        check_choice("m_rule", self.m_rule, M_RULES)


def _run(system, y, params, x_true, kind, mode):
    y = as_vector("y", y, length=system.n_measurements)
    L = N.load()
    system.set_y(y)
    if x_true is not None:
        x_true = as_vector("x_true", x_true, length=system.n_voxels)
    system.set_x_true(x_true)
    N.check(L.bct_baseline_init(system._ctx, kind, N.M_RULE_CODES[params.m_rule]), system._ctx)
    trace = ConvergenceTrace()
    started = time.perf_counter()
    norms = np.zeros(4)
    for epoch in range(1, params.epochs + 1):
        N.check(L.bct_baseline_epoch(system._ctx, float(params.omega), N.ptr(norms)), system._ctx)
        # solvers.py:309-314 (_baseline_trace_row): SNR of x, gap of y_est
        snr = snr_from_sq(math.sqrt(norms[2]), norms[3]) if x_true is not None else math.nan
        gap = snr_from_sq(math.sqrt(norms[0]), norms[1]) if norms[0] > 0.0 else math.nan
        trace.append(TraceRow(epoch=epoch, effective_epoch=float(epoch), snr_db=snr,
                              obs_gap_db=gap, wall_seconds=time.perf_counter() - started,
                              mode=mode, theta=math.nan))
    x = np.empty(system.n_voxels)
    N.check(L.bct_baseline_get_x(system._ctx, N.ptr(x)), system._ctx)
    return x, trace


def run_row_action(system, y, params, x_true=None):
    """Cyclic row-action sweeps (solvers.py:317-346): per measurement block I
    in partition order, x += omega * A_I^T M (y_I - A_I x).  Returns (x, trace);
    effective_epoch counts full data passes."""
    return _run(system, y, params, x_true, N.BCT_ROW_ACTION, "row_action")


def run_column_action(system, y, params, x_true=None):
    """Cyclic column-action sweeps (solvers.py:349-379): per volume block J,
    x_J += omega * D (A^J)^T r with r = y - A x maintained incrementally.
    Returns (x, trace)."""
    return _run(system, y, params, x_true, N.BCT_COLUMN_ACTION, "column_action")


__all__ = ["BaselineParams", "M_RULES", "run_row_action", "run_column_action"]
