"""The CSGD / GCSGD driver with the reference's API (``solvers.py:50-279``).

``run_gcsgd(system, y, params, x_true=None, x0=None, callback=None,
schedule=None, plan_record=None) -> (x, trace)`` is a drop-in for the
reference's runner on a ``DeviceBlockSystem``.  Each epoch is one fused device
launch (tasks + z commit + refresh + _commit_epoch + metric norms); the host
draws the selection variates with numpy's PCG64 exactly like the reference
and reads back four scalars per epoch for the trace and the divergence test.
Without a callback the host draws epoch e+1 while the device runs epoch e.
"""

from __future__ import annotations

import functools
import gc
import logging
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ConfigurationError, DivergenceError
from .executor import (EXECUTION_MODES, EpochExecutor, SampledPlan, pack_loops, submit,
                       submit_sampled, wait)
from .metrics import ConvergenceTrace, TraceRow, snr_from_sq
from .sampling import BlockScheduler, SamplingConfig, ScriptedScheduler, group_beta
from .validation import as_vector, check_choice, check_count, check_positive

logger = logging.getLogger(__name__)


@dataclass(frozen=True)
class SolverParams:
    """Run knobs, validated like the reference (solvers.py:89-116)."""

    epochs: int
    b: float = 100.0
    sampling: SamplingConfig = field(default_factory=SamplingConfig)
    group_size: int = 1
    execution_mode: str = "serial_faithful"
    worker_count: int = 1
    audit_interval: int = 0
    divergence_factor: float = 1e6
    seed: int | None = None

    def __post_init__(self):
        check_count("epochs", self.epochs, minimum=0)
        check_positive("b", self.b)
        check_count("group_size", self.group_size, minimum=1)
        check_choice("execution_mode", self.execution_mode, EXECUTION_MODES)
        check_count("worker_count", self.worker_count, minimum=1)
        check_count("audit_interval", self.audit_interval, minimum=0)
        check_positive("divergence_factor", self.divergence_factor)


class SolverState:
    """View of the device-resident state of one system (solvers.py:50-82).

    ``x``, ``r``, ``z``, ``xhat``, ``counts`` copy from the device on access.
    A system holds one live state: initializing a new state resets it.
    """

    def __init__(self, system, y):
        self.system = system
        self.y = y
        self.epoch = 0

    @classmethod
    def begin(cls, system, y, x_true=None):
        """Cold start (x0 = 0) and the reference image in one asynchronous
        device call (bct_begin_solve): y and x_true are uploaded and r = y
        without a host wait when they are page-locked; the caller keeps both
        arrays alive and unchanged until its next synchronising call."""
        y = as_vector("y", y, length=system.n_measurements)
        xt = None if x_true is None else as_vector("x_true", x_true, length=system.n_voxels)
        N.check(N.load().bct_begin_solve(system.ctx, N.ptr(y),
                                         None if xt is None else N.ptr(xt)), system.ctx)
        return cls(system, y), xt

    @classmethod
    def initialize(cls, system, y, x0=None):
        # float64 and contiguous (no copy when it already is: the device holds
        # the solver's copy, the host keeps it for the trace's |y| only)
        y = as_vector("y", y, length=system.n_measurements)
        system.set_y(y)
        system.reset_accumulators()
        if x0 is None:
            system.clear_state()        # x = 0, z = 0 on the device
            system.reset_residual()     # r = y - 0 = y, exactly
        else:
            x0 = as_vector("x0", x0, length=system.n_voxels)
            system.set_x(x0)
            if np.any(x0 != 0.0):
                system.fill_z_from_image()
            else:
                system.set_z([np.zeros(system.n_local_rows(j)) if system.owns(j) else None
                              for j in range(system.n_col_blocks)])
            system.reset_residual()
        return cls(system, y)

    def load(self, x, r, z):
        """Teacher forcing: overwrite x, r and the z store (accumulators reset)."""
        self.system.set_x(x)
        self.system.set_r(r)
        self.system.set_z(z)
        self.system.reset_accumulators()

    @property
    def x(self):
        return self.system.get_x()

    @property
    def r(self):
        return self.system.get_r()

    @property
    def z(self):
        return self.system.get_z()

    @property
    def xhat(self):
        return self.system.get_xhat()

    @property
    def counts(self):
        return self.system.get_counts()


def basic_iteration(system, i, j, r_i, x_j, beta):
    """One relaxed steepest-descent step on block pair (I_i, J_j), on the device
    (the reference's single-step reference, solvers.py:123-147, here on a
    block of a DeviceBlockSystem instead of a SubmatrixHandle).

    Returns (x_j_new, z_i, mu): z_i = A_I^J x_j_new over the full row block
    (rows the panel does not hit are 0).  A zero gradient or a gradient in the
    block null space gives mu = 0 and an unchanged image.  Uses (and
    overwrites) the system's device state.
    """
    check_positive("beta", beta)
    rows = system.measurement_rows([i])
    x_j = as_vector("x_j", x_j, length=int(system.col_sizes[j]))
    r_i = as_vector("r_i", r_i, length=rows.size)
    x = np.zeros(system.n_voxels)
    x[system.voxel_indices(j)] = x_j
    r = np.zeros(system.n_measurements)
    r[rows] = r_i
    system.set_x(x)
    system.set_r(r)
    system.reset_accumulators()
    ex = EpochExecutor("parallel")
    ex.run_epoch(1, [(j, [(np.array([i], dtype=np.int64), float(beta))])], None, system)
    x_new = system.get_xhat()[system.voxel_indices(j)]
    # z of the block's rows: panel-local rows rbp[i]..rbp[i+1] -> their measurements
    pan = system.panel(j)
    zj = system.get_z()[j]
    z_i = np.zeros(rows.size)
    lo, hi = int(pan.rbp[i]), int(pan.rbp[i + 1])
    order = np.argsort(rows, kind="stable")
    pos = order[np.searchsorted(rows[order], pan.l2g[lo:hi])]
    z_i[pos] = zj[lo:hi]
    return x_new, z_i, float(ex.last_mus[0])


def audit_state(state, system):
    """max |r - (y - sum_j z^j)| / max |y| on the device (solvers.py:154-166)."""
    return {"epoch": state.epoch, "r_drift": system.audit_drift()}


def _commit_epoch(state, system):
    system.commit_epoch()


def _loops(plan, table, b):
    return [(j, [(ids, group_beta(table, b, j, ids)) for ids in groups]) for j, groups in plan]


def _without_gc_pauses(fn):
    """Run fn with Python's cyclic garbage collector paused (restored after):
    the pipelined epoch loop submits epoch e+1 before it waits on epoch e, and
    a collection pause in between leaves the device idle."""
    @functools.wraps(fn)
    def run(*args, **kwargs):
        was = gc.isenabled()
        gc.disable()
        try:
            return fn(*args, **kwargs)
        finally:
            if was:
                gc.enable()
    return run


@_without_gc_pauses
def run_gcsgd(system, y, params, x_true=None, x0=None, callback=None, schedule=None,
              plan_record=None, device_sampling=False):
    """Grouped solver for ``params.epochs`` epochs (solvers.py:188-269).

    Returns (x, ConvergenceTrace); raises DivergenceError with
    last_good_epoch and the partial trace when |x| is non-finite or exceeds
    divergence_factor times its first-epoch value.  ``device_sampling``
    draws the plan on the device from the same numpy variates
    (bct_sample_epoch); the trajectory is identical.
    """
    if schedule is not None:
        scheduler = ScriptedScheduler(schedule, group_size=params.group_size)
    else:
        scheduler = BlockScheduler(system.table, params.sampling, group_size=params.group_size)
    if x0 is None:
        # one asynchronous call: the uploads overlap planning epoch 1
        state, x_true = SolverState.begin(system, y, x_true)
    else:
        state = SolverState.initialize(system, y, x0=x0)
        if x_true is not None:
            x_true = as_vector("x_true", x_true, length=system.n_voxels)
            system.set_x_true(x_true)
        else:
            system.set_x_true(None)
    rng = np.random.default_rng(params.seed)
    trace = ConvergenceTrace()
    flags = N.BCT_COMMIT | N.BCT_METRICS
    # divergence guard on the device: epoch 1 records the reference norm, and
    # an epoch submitted before the host saw its predecessor diverge is a
    # no-op, so the state on raise is the diverged epoch's (solvers.py:251-258)
    N.check(N.load().bct_set_divergence_factor(system.ctx, float(params.divergence_factor)),
            system.ctx)
    mode = params.execution_mode
    started = time.perf_counter()
    ref_norm = None
    pipelined = callback is None and params.audit_interval == 0

    sampled = device_sampling and schedule is None

    def prepare(epoch):
        theta_now = scheduler.theta
        try:
            if sampled:
                packed = SampledPlan(system, scheduler.epoch_variates(epoch, rng),
                                     params.group_size)
            else:
                plan = scheduler.epoch_plan(epoch, rng)
                packed = pack_loops(_loops(plan, system.table, params.b), system)
                if plan_record is not None:
                    plan_record[epoch] = plan
        except Exception as exc:  # surfaced when the loop reaches this epoch
            return exc, theta_now
        scheduler.advance_epoch()
        return packed, theta_now

    def launch(prep, epoch):
        if isinstance(prep[0], Exception):
            return
        fl = flags | (N.BCT_GUARD_REF if epoch == 1 else N.BCT_GUARD)
        if sampled:
            submit_sampled(system, mode, prep[0], params.b, params.sampling.strategy, fl)
        else:
            submit(system, mode, prep[0], fl)

    pending = None
    if params.epochs >= 1:
        pending = prepare(1)
        launch(pending, 1)
    # host-side norms for the trace while the device runs epoch 1
    y_norm = float(np.linalg.norm(state.y))
    xt_norm = float(np.linalg.norm(x_true)) if x_true is not None else math.nan
    for epoch in range(1, params.epochs + 1):
        packed, theta_now = pending
        if isinstance(packed, Exception):
            raise packed
        nxt = None
        if pipelined and epoch < params.epochs:
            nxt = prepare(epoch + 1)
            launch(nxt, epoch + 1)
        res, _, _ = wait(system, packed.task_j.size)
        if sampled:
            plan = packed.finalize()
            if plan_record is not None:
                plan_record[epoch] = plan
        state.epoch = epoch
        if x_true is not None and xt_norm == 0.0:
            # the reference's snr_db raises at the first epoch's metrics
            # (metrics.py:25-27, solvers.py:239)
            if nxt is not None and not isinstance(nxt[0], Exception):
                wait(system, nxt[0].task_j.size)
            raise ConfigurationError("reference signal is identically zero")
        snr = snr_from_sq(xt_norm, res.err_sq) if x_true is not None else math.nan
        gap = snr_from_sq(y_norm, res.resid_sq) if y_norm > 0.0 else math.nan
        row = TraceRow(epoch=epoch, effective_epoch=epoch * params.sampling.alpha, snr_db=snr,
                       obs_gap_db=gap, wall_seconds=time.perf_counter() - started, mode=mode,
                       theta=theta_now, bytes_moved=packed.bytes_moved,
                       n_tasks=int(res.n_tasks), kernel_ms=res.kernel_ms)
        trace.append(row)
        norm_x = math.sqrt(res.x_sq) if res.x_sq >= 0 else math.nan
        if ref_norm is None:
            ref_norm = max(norm_x, 1e-12)
        if not math.isfinite(norm_x) or norm_x > params.divergence_factor * ref_norm:
            if nxt is not None and not isinstance(nxt[0], Exception):
                wait(system, nxt[0].task_j.size)
                if plan_record is not None:
                    plan_record.pop(epoch + 1, None)
            raise DivergenceError(
                f"image norm {norm_x:.3e} left the stable region at epoch {epoch}",
                last_good_epoch=epoch - 1, trace=trace)
        if params.audit_interval and epoch % params.audit_interval == 0:
            rec = audit_state(state, system)
            trace.audits.append(rec)
            if rec["r_drift"] > 1e-8:
                logger.warning("residual bookkeeping drift %.3e at epoch %d", rec["r_drift"],
                               epoch)
        if callback is not None:
            callback(epoch, state, row)
        if not pipelined and epoch < params.epochs:
            nxt = prepare(epoch + 1)
            launch(nxt, epoch + 1)
        pending = nxt
    return system.get_x(), trace


def run_csgd(system, y, params, **kwargs):
    """Ungrouped runner; requires group_size 1 (solvers.py:272-279)."""
    if params.group_size != 1:
        raise ConfigurationError("run_csgd requires group_size 1")
    return run_gcsgd(system, y, params, **kwargs)


__all__ = ["SolverParams", "SolverState", "audit_state", "run_gcsgd", "run_csgd",
           "EpochExecutor", "_commit_epoch"]
