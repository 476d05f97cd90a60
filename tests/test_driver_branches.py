"""run_gcsgd's non-default branches on the device (solvers.py:188-269): the
divergence exit (DivergenceError with last_good_epoch and the diverged
epoch's state), audits and callbacks (the non-pipelined loop), and scripted
schedules (ScriptedScheduler, dump_schedule / parse_schedule)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

bct = pytest.importorskip("paper_1709_00953_b200")
from conftest import golden  # noqa: E402
from oracle.oracle import OracleSystem, oracle_run_gcsgd  # noqa: E402
from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, DivergenceError,  # noqa: E402
                                   SamplingConfig, SolverParams, dump_schedule, parse_schedule,
                                   run_gcsgd)


@pytest.fixture(scope="module")
def cfg1():
    g = golden("pb_cfg1_runs.npz")
    dev = DeviceBlockSystem.parallel_beam(CONFIGS[1].spec, dtype="f64")
    return dev, g["y"], g["x_true"]


def p1(**kw):
    base = dict(epochs=500, b=0.5, group_size=1, seed=1234, execution_mode="serial_faithful",
                sampling=SamplingConfig(alpha=0.25))
    base.update(kw)
    return SolverParams(**base)


@pytest.mark.parametrize("case", [0, 1])
def test_divergence_exit_matches_reference(cfg1, case):
    """config 1 with b=4 diverges.  The reference raises
    DivergenceError(last_good_epoch=E-1) at epoch E (tests/golden/divergence.json,
    made by running the reference); the oracle and the device raise at the
    same epoch with E trace rows.  The pipelined driver had already submitted
    epoch E+1; the device guard makes it a no-op, so the state on raise is
    epoch E's, bit for bit that of a run stopped there."""
    import json
    import os

    from conftest import GOLDEN
    want = json.load(open(os.path.join(GOLDEN, "divergence.json")))[case]
    b, seed, last = want["b"], want["seed"], want["last_good_epoch"]
    dev, y, xt = cfg1
    s = CONFIGS[1].spec
    ora = OracleSystem.parallel_beam(s.n, s.views, s.bins, s.m, s.nc)
    with pytest.raises(RuntimeError) as info:
        oracle_run_gcsgd(ora, y, 2000, b, alpha=0.25, seed=seed, x_true=xt)
    assert info.value.args == ("diverged", last)
    with pytest.raises(DivergenceError) as exc:
        run_gcsgd(dev, y, p1(epochs=2000, b=b, seed=seed), x_true=xt)
    assert exc.value.last_good_epoch == last
    assert len(exc.value.trace.rows) == want["trace_rows"]
    x_raise = dev.get_x()
    x_e, tr = run_gcsgd(dev, y, p1(epochs=last + 1, b=b, seed=seed, divergence_factor=1e300),
                        x_true=xt)
    assert np.array_equal(x_raise, x_e)
    # the non-pipelined loop (a callback) stops at the same epoch and state
    seen = []
    with pytest.raises(DivergenceError) as exc2:
        run_gcsgd(dev, y, p1(epochs=2000, b=b, seed=seed), x_true=xt,
                  callback=lambda e, st, row: seen.append(e))
    assert exc2.value.last_good_epoch == last and seen[-1] == last
    assert np.array_equal(dev.get_x(), x_e)


def test_audits_and_callback_branch(cfg1):
    """audit_interval and callback switch run_gcsgd to the non-pipelined loop:
    same trajectory bit for bit, one audit per interval (drift <= 1e-12:
    solvers.py:260-265), the callback sees every epoch's committed state."""
    dev, y, xt = cfg1
    x_pipe, tr_pipe = run_gcsgd(dev, y, p1(epochs=120), x_true=xt)
    seen = {}

    def cb(epoch, state, row):
        seen[epoch] = (state.x.copy(), row.snr_db)

    x_cb, tr_cb = run_gcsgd(dev, y, p1(epochs=120, audit_interval=25), x_true=xt, callback=cb)
    assert np.array_equal(x_pipe, x_cb)
    assert [r.snr_db for r in tr_pipe.rows] == [r.snr_db for r in tr_cb.rows]
    assert [a["epoch"] for a in tr_cb.audits] == [25, 50, 75, 100]
    assert max(a["r_drift"] for a in tr_cb.audits) <= 1e-12
    assert sorted(seen) == list(range(1, 121))
    assert np.array_equal(seen[120][0], x_cb)
    assert [seen[e][1] for e in range(1, 121)] == [r.snr_db for r in tr_cb.rows]


@pytest.mark.parametrize("mode,gs", [("serial_faithful", 2), ("parallel", 3)])
def test_schedule_replay_reproduces_recorded_run(cfg1, tmp_path, mode, gs):
    """plan_record -> dump_schedule -> parse_schedule -> run_gcsgd(schedule=)
    reproduces the recorded run bit for bit (solvers.py:213-217,
    sampling.py:160-225)."""
    dev, y, xt = cfg1
    p = SolverParams(epochs=15, b=0.4, group_size=gs, seed=31, execution_mode=mode,
                     sampling=SamplingConfig(alpha=0.75))
    rec = {}
    x0, tr0 = run_gcsgd(dev, y, p, x_true=xt, plan_record=rec)
    path = tmp_path / "plan.txt"
    dump_schedule(rec, str(path))
    sched = parse_schedule(str(path), n_row_blocks=dev.n_row_blocks,
                           n_col_blocks=dev.n_col_blocks)
    rec2 = {}
    x1, tr1 = run_gcsgd(dev, y, p, x_true=xt, schedule=sched, plan_record=rec2)
    assert np.array_equal(x0, x1)
    assert [r.obs_gap_db for r in tr0.rows] == [r.obs_gap_db for r in tr1.rows]
    for e in rec:
        assert [(j, [g.tolist() for g in gs_]) for j, gs_ in rec[e]] == \
               [(j, [g.tolist() for g in gs_]) for j, gs_ in rec2[e]]


def test_solver_start_inputs_pinned_or_pageable_and_state(cfg1):
    """bct_begin_solve (run_gcsgd's x0 = 0 start): the same run from
    page-locked inputs (asynchronous uploads) and from ordinary numpy arrays
    (staged uploads) is bit for bit the same, and equals the classic start
    (SolverState.initialize + set_x_true, the x0 path with x0 = 0)."""
    import torch

    dev, y, xt = cfg1
    params = p1(epochs=6)
    x_np, tr_np = run_gcsgd(dev, y.copy(), params, x_true=xt.copy())
    y_pin = torch.empty(y.size, dtype=torch.float64).pin_memory().numpy()
    xt_pin = torch.empty(xt.size, dtype=torch.float64).pin_memory().numpy()
    y_pin[:] = y
    xt_pin[:] = xt
    x_pin, tr_pin = run_gcsgd(dev, y_pin, params, x_true=xt_pin)
    assert np.array_equal(x_np, x_pin)
    assert [r.snr_db for r in tr_np.rows] == [r.snr_db for r in tr_pin.rows]
    r_pin = dev.get_r()
    x_cl, tr_cl = run_gcsgd(dev, y, params, x_true=xt, x0=np.zeros(dev.n_voxels))
    assert np.array_equal(x_np, x_cl)
    assert np.array_equal(r_pin, dev.get_r())
    assert [r.snr_db for r in tr_np.rows] == [r.snr_db for r in tr_cl.rows]


def test_zero_reference_raises_at_first_metrics(cfg1):
    """The reference's snr_db raises 'reference signal is identically zero'
    at the first epoch's metrics (src/metrics.py:25-27, src/solvers.py:239):
    a zero x_true raises with epochs >= 1 and not with epochs = 0."""
    from paper_1709_00953_b200 import ConfigurationError
    dev, y, xt = cfg1
    with pytest.raises(ConfigurationError, match="identically zero"):
        run_gcsgd(dev, y, p1(epochs=3), x_true=np.zeros_like(xt))
    x0, tr = run_gcsgd(dev, y, p1(epochs=0), x_true=np.zeros_like(xt))
    assert len(tr.rows) == 0 and not np.any(x0)
