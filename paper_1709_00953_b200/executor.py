"""Epoch execution on the device (the reference's ``executor.py:1-253``).

``EpochExecutor(mode, worker_count).run_epoch(epoch, loops, state, system)``
keeps the reference contract -- it mutates z, r, xhat and counts and leaves
the image commit to the caller -- but one call is one cooperative kernel
launch: every task of the plan, its z commit and the refresh run on the
device (csrc/epoch.cu).  ``worker_count`` is accepted for API compatibility;
the device result does not depend on it (the reference's own invariant,
tests/test_executor.py:113-128).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ExecutorError
from .validation import check_choice, check_count

EXECUTION_MODES = ("serial_faithful", "parallel")


@dataclass
class TaskDescriptor:
    index: int
    j: int
    i_ids: np.ndarray
    beta: float


@dataclass
class EpochStats:
    """Task and visit counts, the reference's bytes_moved accounting
    (16 bytes per drawn measurement row and per block voxel per task,
    executor.py:210-213), degenerate tasks, and the device epoch time."""

    n_tasks: int = 0
    n_loops: int = 0
    bytes_moved: int = 0
    n_degenerate: int = 0
    kernel_ms: float = 0.0
    resid_sq: float = float("nan")
    x_sq: float = float("nan")
    err_sq: float = float("nan")


@dataclass
class PackedPlan:
    task_j: np.ndarray
    task_visit: np.ndarray
    task_gptr: np.ndarray
    sel: np.ndarray
    betas: np.ndarray
    groups: list              # [(j, ids)] per task, for error reporting
    n_loops: int
    bytes_moved: int


def pack_loops(loops, system):
    """Flatten ``[(j, [(ids, beta), ...]), ...]`` into the C plan arrays."""
    tj, tv, sizes, sel, betas, groups = [], [], [], [], [], []
    bytes_moved = 0
    for v, (j, tasks) in enumerate(loops):
        j = int(j)
        pix = 0
        for ids, beta in tasks:
            ids = np.asarray(ids, dtype=np.int64).ravel()
            tj.append(j)
            tv.append(v)
            sizes.append(ids.size)
            sel.append(ids)
            betas.append(float(beta))
            groups.append((j, ids))
            if ids.size and (ids.min() < 0 or ids.max() >= system.n_row_blocks):
                raise ExecutorError(
                    f"tasks on volume block {j} failed to assemble: measurement block out "
                    f"of range", task=TaskDescriptor(len(tj) - 1, j, ids, float(beta)))
            pix += int(system.row_sizes[ids].sum()) if ids.size else 0
        if not (0 <= j < system.n_col_blocks):
            raise ExecutorError(f"volume block {j} out of range",
                                task=TaskDescriptor(len(tj) - 1, j, np.empty(0, np.int64), 0.0))
        bytes_moved += 16 * (pix + len(tasks) * int(system.col_sizes[j]))
    gptr = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=gptr[1:])
    return PackedPlan(N.i32(tj), N.i32(tv), gptr,
                      N.i64(np.concatenate(sel) if sel else np.empty(0, np.int64)),
                      N.f64(betas), groups, len(loops), bytes_moved)


def submit(system, mode, plan, flags):
    """Queue one epoch on the device (asynchronous)."""
    rc = N.load().bct_run_epoch(system.ctx, N.MODES[mode], plan.task_j.size,
                                N.ptr(plan.task_j), N.ptr(plan.task_visit),
                                N.ptr(plan.task_gptr), N.ptr(plan.sel), N.ptr(plan.betas),
                                flags)
    if rc != 0:
        j, ids = plan.groups[0] if plan.groups else (-1, np.empty(0, np.int64))
        N.check(rc, system.ctx, "epoch plan rejected",
                task=TaskDescriptor(0, j, ids, float(plan.betas[0]) if plan.betas.size else 0.0))


class SampledPlan:
    """An epoch whose plan the device draws (bct_sample_epoch) from the host's
    variates (sampling.BlockScheduler.epoch_variates).  The task structure is
    known up front; the drawn ids arrive with the epoch result
    (``finalize`` after ``wait``), giving the plan and bytes_moved."""

    def __init__(self, system, variates, group_size):
        self.variates = variates
        self.group_size = int(group_size)
        gs = self.group_size
        owned = [system.owns(int(j)) for j in variates.visit_j]
        self.task_j = np.array([int(j) for j, d, o in zip(variates.visit_j, variates.draws, owned)
                                if o for _ in range(-(-int(d) // gs))], dtype=np.int32)
        self.plan_ids = np.zeros(max(int(variates.draws.sum()), 1), dtype=np.int64)
        self.plan = None
        self.bytes_moved = 0
        self.n_loops = int(variates.visit_j.size)
        self._system = system

    def finalize(self):
        """Plan [(j, [ids chunks])] in visit order, and the reference's
        bytes_moved (executor.py:210-213), from the device-drawn ids."""
        plan, off, moved = [], 0, 0
        gs = self.group_size
        for j, d in zip(self.variates.visit_j, self.variates.draws):
            ids = self.plan_ids[off:off + int(d)].copy()
            off += int(d)
            groups = [ids[p:p + gs] for p in range(0, ids.size, gs)]
            plan.append((int(j), groups))
            pix = int(self._system.row_sizes[ids].sum()) if ids.size else 0
            moved += 16 * (pix + len(groups) * int(self._system.col_sizes[int(j)]))
        self.plan = plan
        self.bytes_moved = moved
        return plan


def submit_sampled(system, mode, sampled, b, strategy, flags):
    """Queue one epoch whose plan the device samples (asynchronous)."""
    v = sampled.variates
    rc = N.load().bct_sample_epoch(system.ctx, N.MODES[mode], int(v.visit_j.size),
                                   N.ptr(N.i32(v.visit_j)), N.ptr(N.f64(v.exp)), int(v.exp.size),
                                   N.ptr(N.i32(v.draws)), sampled.group_size, float(b),
                                   N.STRATEGY_CODES[strategy], float(v.theta), flags,
                                   N.ptr(sampled.plan_ids))
    if rc != 0:
        N.check(rc, system.ctx, "sampled epoch rejected")


def wait(system, n_tasks, want_status=False):
    """Block on the oldest queued epoch; returns (EpochResult, mus, statuses)."""
    res = N.EpochResult()
    mus = np.empty(max(n_tasks, 1)) if want_status else None
    st = np.empty(max(n_tasks, 1), dtype=np.int32) if want_status else None
    N.check(N.load().bct_wait_epoch(system.ctx, res, N.ptr(mus), N.ptr(st)), system.ctx,
            "epoch")
    return res, mus, st


class EpochExecutor:
    def __init__(self, mode="serial_faithful", worker_count=1):
        check_choice("execution_mode", mode, EXECUTION_MODES)
        check_count("worker_count", worker_count, minimum=1)
        self.mode = mode
        self.worker_count = int(worker_count)
        self.last_mus = None
        self.last_statuses = None

    def run_epoch(self, epoch, loops, state, system, flags=0):
        """Execute one epoch of ``loops``; returns EpochStats.  ``flags`` may add
        BCT_COMMIT / BCT_METRICS (the fused fast path used by run_gcsgd)."""
        plan = pack_loops(loops, system)
        submit(system, self.mode, plan, flags)
        res, mus, st = wait(system, plan.task_j.size, want_status=True)
        n = plan.task_j.size
        self.last_mus = mus[:n]
        self.last_statuses = st[:n]
        return EpochStats(n_tasks=int(res.n_tasks), n_loops=plan.n_loops,
                          bytes_moved=plan.bytes_moved, n_degenerate=int(res.n_degenerate),
                          kernel_ms=res.kernel_ms, resid_sq=res.resid_sq, x_sq=res.x_sq,
                          err_sq=res.err_sq)
