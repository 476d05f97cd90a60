"""The reference's own acceptance runs on the device (tests/test_acceptance.py
A02, A10, A11): the standard 2D fan-beam asset (720 row blocks) and the 3D
random-sphere smoke run (360 row blocks), traced on the device and solved
through ``run_gcsgd``.  The expected images come from the CPU oracle, whose
runs are pinned bit for bit to the reference's (test_acceptance_pins.py
re-checks the hashes here too)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

bct = pytest.importorskip("paper_1709_00953_b200")
from _acceptance import (a11_geometry, fixtures, panels_match, params, sha,  # noqa: E402
                         standard_geometry, unflatten)
from oracle.oracle import (OracleState, OracleSystem, OracleTable,  # noqa: E402
                           oracle_commit_epoch, oracle_forward_project, oracle_group_beta,
                           oracle_run_epoch, oracle_run_gcsgd)
from paper_1709_00953_b200 import (DeviceBlockSystem, DivergenceError,  # noqa: E402
                                   EpochExecutor, SolverState, dump_schedule, parse_schedule,
                                   run_gcsgd)

WORKERS = max(1, min(16, os.cpu_count() or 1))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_from_device(dev):
    pans = [dev.panel(j) for j in range(dev.n_col_blocks)]
    vals = np.array(dev.table.values)
    return OracleSystem([p.data for p in pans], [p.cols for p in pans],
                        [p.indptr for p in pans], [p.rbp for p in pans], [p.l2g for p in pans],
                        [dev.measurement_rows([i]) for i in range(dev.n_row_blocks)],
                        [dev.voxel_indices(j) for j in range(dev.n_col_blocks)],
                        OracleTable(vals, vals.sum(axis=0)), dev.n_measurements, dev.n_voxels)


@pytest.fixture(scope="module")
def fx():
    return fixtures()


@pytest.fixture(scope="module")
def std(fx):
    f, H = fx
    geo, part = standard_geometry()
    dev = DeviceBlockSystem.scan(geo, partition=part, dtype="f64")
    assert panels_match(lambda j: (lambda p: (p.data, p.cols, p.indptr, p.rbp, p.l2g))(
        dev.panel(j)), H["std_panels"])
    np.testing.assert_array_equal(dev.table.values, f["std_table"])
    y = oracle_forward_project(geo, f["std_x_true"])
    assert sha(y) == H["std_y"]
    return dev, oracle_from_device(dev), y, f["std_x_true"]


# A02 runs converge to ~90 dB on noise-free data with over-relaxation (b=2);
# two FP64 implementations that sum in different orders drift apart
# geometrically there (SURVEY §0 finding 5): measured on B200, the device's x
# is within 6e-15 of the reference's through epoch 20 and first passes 1e-10
# at epoch 40 (serial) / 42 (parallel), growing ~10x per 2 epochs.  The
# free-running check is held to 30 epochs; epoch 101 is checked
# teacher-forced at 1e-12 below (protocol P3).
A02_FREE_EPOCHS = 30


@pytest.mark.parametrize("mode,tag", [("serial_faithful", "ser"), ("parallel", "par")])
def test_a02_residual_audits_and_trajectory(fx, std, mode, tag):
    """A02 on the device: 20 audits per mode (every 10 of 200 epochs) within
    1e-8; x within 1e-10 of the reference's (hash-pinned oracle replay) over
    the free-running window, and the plans equal the reference's."""
    f, H = fx
    dev, ora, y, xt = std
    xs, rec = [], {}
    x, tr = run_gcsgd(dev, y, params(200, 2.0, 100, 0, mode, 0.5, audit=10), x_true=xt,
                      plan_record=rec, callback=lambda e, s, r: xs.append(s.x.copy()))
    drifts = [a["r_drift"] for a in tr.audits]
    assert len(drifts) == 20
    print(f"A02 {mode}: worst device drift {max(drifts):.2e}")
    assert max(drifts) <= 1e-8
    xs_o, rec_o = [], {}
    x_o, rows = oracle_run_gcsgd(ora, y, 200, 2.0, alpha=0.5, group_size=100, mode=mode,
                                 seed=0, x_true=xt, workers=WORKERS, plan_record=rec_o,
                                 callback=lambda e, s, r: xs_o.append(s.x.copy()))
    assert sha(x_o) == H[f"a02_{tag}_x"]
    drift = np.array([rel(a, b) for a, b in zip(xs, xs_o)])
    first = int(np.argmax(drift > 1e-10)) + 1 if np.any(drift > 1e-10) else None
    snr = np.array([r.snr_db for r in tr.rows])
    dsnr = np.abs(snr - f[f"a02_{tag}_snr"]) / np.abs(f[f"a02_{tag}_snr"])
    print(f"A02 {mode}: x drift vs reference at epochs 10/20/50/100/200 "
          f"{drift[[9, 19, 49, 99, 199]]}, first > 1e-10 at {first}; "
          f"SNR rel dev epochs 1-20 {dsnr[:20].max():.2e}, all {dsnr.max():.2e}")
    assert drift[:A02_FREE_EPOCHS].max() <= 1e-10
    assert dsnr[:A02_FREE_EPOCHS].max() <= 1e-9
    for e in range(1, A02_FREE_EPOCHS + 1):
        assert [(j, [g.tolist() for g in gs]) for j, gs in rec[e]] == \
               [(j, [g.tolist() for g in gs]) for j, gs in rec_o[e]]


@pytest.mark.parametrize("mode,tag", [("serial_faithful", "ser"), ("parallel", "par")])
def test_a02_teacher_forced_epoch_101(fx, std, mode, tag):
    """The reference's epoch-100 state (oracle replay, hash-pinned), one epoch
    of its epoch-101 plan on the device: x, r, z at 1e-12."""
    f, H = fx
    dev, ora, y, xt = std
    snaps, rec = {}, {}

    def cb(epoch, state, row):
        if epoch in (100, 101):
            snaps[epoch] = state.copy()

    oracle_run_gcsgd(ora, y, 101, 2.0, alpha=0.5, group_size=100, mode=mode, seed=0,
                     callback=cb, plan_record=rec, workers=WORKERS)
    assert sha(snaps[100].x) == H[f"a02_{tag}_x100"]
    assert sha(snaps[101].x) == H[f"a02_{tag}_x101"]
    loops = [(j, [(ids, oracle_group_beta(ora.table, 2.0, j, ids)) for ids in groups])
             for j, groups in rec[101]]
    s100 = snaps[100]
    st = SolverState.initialize(dev, y)
    st.load(s100.x, s100.r, s100.z)
    EpochExecutor(mode).run_epoch(101, loops, st, dev)
    dev.commit_epoch()
    want = snaps[101]
    assert rel(st.x, want.x) <= 1e-12
    assert rel(st.r, want.r) <= 1e-12
    assert rel(np.concatenate(st.z), np.concatenate(want.z)) <= 1e-12


def test_a10_worker_invariance_and_schedule_replay(fx, std, tmp_path):
    """A10: the recorded parallel schedule replayed with worker_count 1, 2, 4,
    8 commits bitwise-identical images every epoch, equal to the reference's
    (oracle replay, hash-pinned) within 1e-10; the same schedule through
    dump_schedule / parse_schedule (sampling.py:185-225) replays bitwise."""
    f, H = fx
    dev, ora, y, xt = std
    sched = unflatten(f["a10_plans"])
    xs_o = []
    oracle_run_gcsgd(ora, y, 10, 2.0, alpha=0.5, group_size=100, mode="parallel", seed=3,
                     schedule=sched, callback=lambda e, s, r: xs_o.append(s.x.copy()))
    assert [sha(v) for v in xs_o] == H["a10_x"]
    states = {}
    for workers in (1, 2, 4, 8):
        snaps, rec = [], {}
        run_gcsgd(dev, y, params(10, 2.0, 100, 3, "parallel", 0.5, workers=workers),
                  schedule=sched, plan_record=rec,
                  callback=lambda e, s, r: snaps.append(s.x.copy()))
        states[workers] = snaps
        for ep, visits in sched.items():
            assert [(j, np.concatenate(g).tolist()) for j, g in rec[ep]] == \
                   [(j, ids.tolist()) for j, ids in visits]
    for w in (2, 4, 8):
        assert all(np.array_equal(states[1][e], states[w][e]) for e in range(10))
    assert max(rel(a, b) for a, b in zip(states[1], xs_o)) <= 1e-10
    path = tmp_path / "schedule.txt"
    dump_schedule({e: [(j, [ids]) for j, ids in v] for e, v in sched.items()}, str(path))
    parsed = parse_schedule(str(path), n_row_blocks=dev.n_row_blocks,
                            n_col_blocks=dev.n_col_blocks)
    snaps = []
    run_gcsgd(dev, y, params(10, 2.0, 100, 3, "parallel", 0.5), schedule=parsed,
              callback=lambda e, s, r: snaps.append(s.x.copy()))
    assert all(np.array_equal(a, b) for a, b in zip(snaps, states[1]))


def test_a11_3d_smoke_run(fx):
    """A11 on the device: 3D random-sphere scan (8 volume blocks, 360 row
    blocks) traced on the device bit for bit; the b ladder (40, 20, 10, 5, 2;
    10 epochs, s=16) picks the reference's b, and 50 epochs at that b raise
    the SNR monotonically with the reference's trace and image."""
    f, H = fx
    geo, part = a11_geometry()
    dev = DeviceBlockSystem.scan(geo, partition=part, dtype="f64")
    assert panels_match(lambda j: (lambda p: (p.data, p.cols, p.indptr, p.rbp, p.l2g))(
        dev.panel(j)), H["a11_panels"])
    xt = f["a11_x_true"]
    y = oracle_forward_project(geo, xt)
    assert sha(y) == H["a11_y"]
    best = None
    for b, snr_ref, flag in f["a11_ladder"]:
        try:
            _, tr = run_gcsgd(dev, y, params(10, float(b), 16, 0), x_true=xt)
        except DivergenceError as exc:
            assert np.isnan(snr_ref) and exc.last_good_epoch == int(flag)
            continue
        snr = np.array([r.snr_db for r in tr.rows])
        mono = bool((np.diff(snr) > 0.0).all())
        assert mono == bool(flag)
        assert abs(snr[-1] - snr_ref) <= 1e-9 * abs(snr_ref)
        if mono and (best is None or snr[-1] > best[1]):
            best = (float(b), float(snr[-1]))
    assert best[0] == float(f["a11_b"])
    x, tr = run_gcsgd(dev, y, params(50, best[0], 16, 0), x_true=xt)
    snr = np.array([r.snr_db for r in tr.rows])
    assert (np.diff(snr) > 0.0).all()
    np.testing.assert_allclose(snr, f["a11_snr"], rtol=1e-9)
    ora = oracle_from_device(dev)
    x_o, _ = oracle_run_gcsgd(ora, y, 50, best[0], group_size=16, seed=0, x_true=xt)
    assert sha(x_o) == H["a11_x"]
    print(f"A11: b={best[0]:g}, 50-epoch SNR {snr[-1]:.4f} dB, x vs reference {rel(x, x_o):.2e}")
    assert rel(x, x_o) <= 1e-10
    dev.close()
