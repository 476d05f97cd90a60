"""Column-block sharding over ranks: one process per GPU.

Rank p owns the contiguous column blocks ``owned_range(n, world, p)``: their
forward panels, panel CSCs, z^j, x_J and xhat_J.  y and r are replicated and
every rank draws the same plan from the same seed, so the plan needs no
broadcast.  Per epoch (parallel execution only -- serial_faithful visits are
ordered through the residual and do not shard):

1. each rank runs the plan's tasks on its own column blocks against the
   epoch-start r (the device skips other ranks' tasks; BCT_SHARDED);
2. the epoch kernel writes the rank's partial projection sums
   S_p[g] = sum_{j owned} z^j[g] for every measurement, plus the partial
   squared norms of x and x_true - x, into the context's exchange buffer;
3. one all-reduce (NCCL over NVLink on the device path) sums the buffer in
   place;
4. ``bct_finish_sharded`` sets r = y - S on the rows of the drawn blocks
   (executor.py:249-252) and reduces |y - S|^2 for the trace.

The runner is written against a small backend interface so the same host
logic runs on the device (``DeviceShard``) and, in the multi-process CPU tests,
on a test-side oracle backend over the gloo backend.
"""

from __future__ import annotations

import ctypes
import math
import time

import numpy as np

from . import _native as N
from .errors import ConfigurationError, DivergenceError
from .executor import pack_loops, submit, wait
from .metrics import ConvergenceTrace, TraceRow, snr_from_sq
from .sampling import BlockScheduler, ScriptedScheduler
from .solvers import SolverState, _loops, _without_gc_pauses


def owned_range(n_panels, world, rank):
    """Contiguous column-block range of ``rank`` (balanced to within one block)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigurationError(f"bad rank {rank} of {world}")
    if n_panels < world:
        raise ConfigurationError(f"{n_panels} column blocks cannot shard over {world} ranks")
    return rank * n_panels // world, (rank + 1) * n_panels // world


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper of a device pointer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class DeviceShard:
    """Backend of ShardedRunner on a DeviceBlockSystem (the product path)."""

    def __init__(self, system):
        import torch
        self.system = system
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        N.check(N.load().bct_exchange_buffer(system.ctx, ctypes.byref(p), ctypes.byref(n)),
                system.ctx)
        self.n_meas = system.n_measurements
        self.buf = torch.as_tensor(_CudaArray(p.value, n.value), device=f"cuda:{system.device}")
        self.stream = torch.cuda.ExternalStream(system.stream(), device=system.device)

    def run_partial(self, packed, flags):
        # asynchronous: the all-reduce and the finish kernels follow on the
        # same stream; the host waits only in ``result``
        submit(self.system, "parallel", packed, flags | N.BCT_SHARDED)
        return packed.task_j.size

    def exchange(self):
        return self.buf

    def comm_stream(self):
        import torch
        return torch.cuda.stream(self.stream)

    def finish(self, flags):
        N.check(N.load().bct_finish_sharded(self.system.ctx, flags, None), self.system.ctx)
        return None

    def result(self, n_tasks):
        return wait(self.system, n_tasks)[0]


class ShardedRunner:
    """One sharded epoch = partial epoch, all-reduce of the exchange buffer,
    finish.  ``allreduce`` defaults to torch.distributed.all_reduce."""

    def __init__(self, system, backend=None, allreduce=None):
        self.system = system
        self.backend = backend if backend is not None else DeviceShard(system)
        if allreduce is None:
            import torch.distributed as dist
            allreduce = dist.all_reduce
        self.allreduce = allreduce
        self._pending = []

    def submit(self, packed, flags):
        """Enqueue one sharded epoch: partial epoch, all-reduce, finish."""
        token = self.backend.run_partial(packed, flags)
        ctx = getattr(self.backend, "comm_stream", None)
        if ctx is not None:
            with ctx():
                self.allreduce(self.backend.exchange())
        else:
            self.allreduce(self.backend.exchange())
        norms = self.backend.finish(flags)
        self._pending.append((packed, token, norms))

    def collect(self):
        """Result of the oldest submitted epoch (EpochResult with global norms)."""
        packed, token, norms = self._pending.pop(0)
        res = self.backend.result(token) if hasattr(self.backend, "result") else token
        if norms is not None:
            res.resid_sq, res.x_sq, res.err_sq = norms
        res.n_tasks = packed.task_j.size
        return res

    def epoch(self, packed, flags):
        self.submit(packed, flags)
        return self.collect()


def sharded_forward(system, x, allreduce=None):
    """y = A x with every rank contributing its panels (one all-reduce)."""
    import torch
    import torch.distributed as dist
    part = system.forward(x)  # owned panels only
    t = torch.as_tensor(part, device=f"cuda:{system.device}")
    (allreduce or dist.all_reduce)(t)
    return t.cpu().numpy()


@_without_gc_pauses
def run_gcsgd_sharded(system, y, params, x_true=None, schedule=None, plan_record=None,
                      runner=None, allreduce=None, callback=None):
    """run_gcsgd with the column blocks sharded over the process group
    (parallel execution).  Returns the full x on every rank and the trace.

    Pipelined like run_gcsgd: epoch e+1 is planned, packed and enqueued
    (partial epoch, all-reduce, finish -- all on the context's stream) before
    the host reads epoch e's norms; the device divergence guard makes an epoch
    submitted after a diverged one a no-op on every rank (the guard reads the
    all-reduced |x|), so the state on DivergenceError is the diverged epoch's.
    ``allreduce`` (default torch.distributed.all_reduce) sums a device tensor
    in place across ranks.  A callback disables the pipelining, as in
    run_gcsgd.  Audits are rank-local and not offered here."""
    import torch
    import torch.distributed as dist
    if params.execution_mode != "parallel":
        raise ConfigurationError("sharded execution requires execution_mode='parallel'")
    if params.audit_interval:
        raise ConfigurationError("audit_interval is not supported by sharded runs")
    allreduce = allreduce or dist.all_reduce
    runner = runner or ShardedRunner(system, allreduce=allreduce)
    if schedule is not None:
        scheduler = ScriptedScheduler(schedule, group_size=params.group_size)
    else:
        scheduler = BlockScheduler(system.table, params.sampling, group_size=params.group_size)
    # cold start and x_true in one asynchronous call (uploads overlap planning
    # epoch 1); the host norms for the trace are taken while epoch 1 runs
    state, x_true = SolverState.begin(system, y, x_true)
    rng = np.random.default_rng(params.seed)
    N.check(N.load().bct_set_divergence_factor(system.ctx, float(params.divergence_factor)),
            system.ctx)
    flags = N.BCT_COMMIT | N.BCT_METRICS
    trace = ConvergenceTrace()
    started = time.perf_counter()
    ref_norm = None
    pipelined = callback is None

    def prepare(epoch):
        theta_now = scheduler.theta
        try:
            plan = scheduler.epoch_plan(epoch, rng)
            packed = pack_loops(_loops(plan, system.table, params.b), system)
        except Exception as exc:  # surfaced when the loop reaches this epoch
            return exc, None, theta_now
        if plan_record is not None:
            plan_record[epoch] = plan
        scheduler.advance_epoch()
        return packed, plan, theta_now

    def launch(prep, epoch):
        if not isinstance(prep[0], Exception):
            runner.submit(prep[0], flags | (N.BCT_GUARD_REF if epoch == 1 else N.BCT_GUARD))

    pending = None
    if params.epochs >= 1:
        pending = prepare(1)
        launch(pending, 1)
    y_norm = float(np.linalg.norm(state.y))
    xt_norm = float(np.linalg.norm(x_true)) if x_true is not None else None
    for epoch in range(1, params.epochs + 1):
        packed, _, theta_now = pending
        if isinstance(packed, Exception):
            raise packed
        nxt = None
        if pipelined and epoch < params.epochs:
            nxt = prepare(epoch + 1)
            launch(nxt, epoch + 1)
        res = runner.collect()
        state.epoch = epoch
        snr = snr_from_sq(xt_norm, res.err_sq) if x_true is not None else math.nan
        gap = snr_from_sq(y_norm, res.resid_sq) if y_norm > 0 else math.nan
        row = TraceRow(epoch, epoch * params.sampling.alpha, snr, gap,
                       time.perf_counter() - started, params.execution_mode, theta_now,
                       packed.bytes_moved, packed.task_j.size, res.kernel_ms)
        trace.append(row)
        norm_x = math.sqrt(res.x_sq) if res.x_sq >= 0 else math.nan
        if ref_norm is None:
            ref_norm = max(norm_x, 1e-12)
        if not math.isfinite(norm_x) or norm_x > params.divergence_factor * ref_norm:
            if nxt is not None and not isinstance(nxt[0], Exception):
                runner.collect()          # the guarded no-op epoch
                if plan_record is not None:
                    plan_record.pop(epoch + 1, None)
            raise DivergenceError(f"image norm {norm_x:.3e} left the stable region at epoch "
                                  f"{epoch}", last_good_epoch=epoch - 1, trace=trace)
        if callback is not None:
            callback(epoch, state, row)
        if not pipelined and epoch < params.epochs:
            nxt = prepare(epoch + 1)
            launch(nxt, epoch + 1)
        pending = nxt
    # assemble the full image: owned entries from every rank
    x_local = system.get_x()
    mine = np.zeros(system.n_voxels)
    for j in range(system.panel_begin, system.panel_end):
        v = system.voxel_indices(j)
        mine[v] = x_local[v]
    t = torch.as_tensor(mine, device=f"cuda:{system.device}")
    allreduce(t)
    return t.cpu().numpy(), trace
