"""Parity of the CUDA path against the reference's own outputs (golden
fixtures made by tests/golden/make_golden.py) and against the CPU oracle.

Tolerances: bit-exact for the traced matrix, the table, the selection plans
and the bitwise set-up kernels; FP64 epochs within 1e-10 relative free-running
(north_star) and 1e-12 teacher-forced; FP32 storage within
1e-4 relative on the residual curve (north_star).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, fixture_system_arrays, golden, unflatten_plans

pytestmark = pytest.mark.gpu

bct = pytest.importorskip("paper_1709_00953_b200")
from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, EpochExecutor,  # noqa: E402
                                   ExecutorError, SamplingConfig, SolverParams, SolverState,
                                   run_gcsgd)
from paper_1709_00953_b200.geometry import ParallelBeamSpec  # noqa: E402

VARIANTS = {
    "p1": dict(epochs=500, b=0.5, group_size=1, seed=1234, execution_mode="serial_faithful",
               sampling=SamplingConfig(alpha=0.25)),
    "ser_g2": dict(epochs=20, b=0.5, group_size=2, seed=11, execution_mode="serial_faithful",
                   sampling=SamplingConfig(alpha=1.0)),
    "par_full": dict(epochs=20, b=0.25, group_size=4, seed=12, execution_mode="parallel",
                     sampling=SamplingConfig(alpha=1.0)),
    "par_mixed": dict(epochs=20, b=0.3, group_size=1, seed=13, execution_mode="parallel",
                      sampling=SamplingConfig(strategy="mixed", alpha=0.5, gamma=0.5, theta0=0.2,
                                              theta_step=0.1)),
    "ser_random": dict(epochs=20, b=0.5, group_size=3, seed=14, execution_mode="serial_faithful",
                       sampling=SamplingConfig(strategy="random", alpha=0.75)),
}


def _hash(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def cfg1_system():
    return DeviceBlockSystem.parallel_beam(CONFIGS[1].spec, dtype="f64")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------------------
# the device-built operator is the reference's, bit for bit
# ---------------------------------------------------------------------------

def test_builder_small_matches_reference_panels():
    g = golden("pb_small.npz")
    spec = ParallelBeamSpec(16, 20, 24, 4, 4)
    sysm = DeviceBlockSystem.parallel_beam(spec, dtype="f64")
    for j in range(4):
        p = sysm.panel(j)
        np.testing.assert_array_equal(p.data, g[f"data{j}"])
        np.testing.assert_array_equal(p.cols, g[f"cols{j}"])
        np.testing.assert_array_equal(p.indptr, g[f"indptr{j}"])
        np.testing.assert_array_equal(p.rbp, g[f"rbp{j}"])
        np.testing.assert_array_equal(p.l2g, g[f"l2g{j}"])
    np.testing.assert_array_equal(sysm.table.values, g["table"])
    # bitwise forward projection (projector.py:692-702 order)
    np.testing.assert_array_equal(sysm.forward(g["x_true"]), g["y_clean"])


@pytest.mark.parametrize("key", [1, 2])
def test_builder_matches_reference_hashes(key):
    hashes = json.load(open(os.path.join(GOLDEN, "pb_hashes.json")))
    sysm = DeviceBlockSystem.parallel_beam(CONFIGS[key].spec, dtype="f64")
    for j, h in enumerate(hashes[f"cfg{key}"]):
        p = sysm.panel(j)
        assert p.data.size == h["nnz"] and p.l2g.size == h["rows"]
        assert _hash(p.data) == h["data"], f"panel {j} values"
        assert _hash(p.cols) == h["cols"], f"panel {j} cols"
        assert _hash(p.indptr) == h["indptr"]
        assert _hash(p.rbp) == h["rbp"]
        assert _hash(p.l2g) == h["l2g"]
    assert _hash(sysm.table.values) == hashes[f"cfg{key}_table_sha"]


# ---------------------------------------------------------------------------
# free-running runs against the reference (config 1)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", list(VARIANTS))
def test_free_running_matches_reference(cfg1_system, cfg1_runs, name):
    g = cfg1_runs
    np.testing.assert_array_equal(cfg1_system.forward(g["x_true"]), g["y_clean"])
    rec = {}
    x, tr = run_gcsgd(cfg1_system, g["y"], SolverParams(**VARIANTS[name]), x_true=g["x_true"],
                      plan_record=rec)
    # the selection stream is replayed exactly
    want = unflatten_plans(g[f"{name}_plans"])
    assert sorted(rec) == sorted(want)
    for ep, visits in want.items():
        got = [(j, np.concatenate(gr) if gr else np.empty(0, np.int64)) for j, gr in rec[ep]]
        assert [j for j, _ in got] == [j for j, _ in visits]
        for (_, a), (_, b) in zip(got, visits):
            np.testing.assert_array_equal(a, b)
    xr = g[f"{name}_x"]
    assert rel(x, xr) <= 1e-10
    A_res = np.linalg.norm(g["y"] - cfg1_system.forward(x))
    A_ref = np.linalg.norm(g["y"] - cfg1_system.forward(xr))
    assert abs(A_res - A_ref) / A_ref <= 1e-10
    gaps = np.array([r.obs_gap_db for r in tr.rows])
    np.testing.assert_allclose(gaps, g[f"{name}_gap"], rtol=1e-9)
    snrs = np.array([r.snr_db for r in tr.rows])
    np.testing.assert_allclose(snrs, g[f"{name}_snr"], rtol=1e-9)
    assert [r.n_tasks for r in tr.rows] == list(g[f"{name}_n_tasks"])
    assert [r.bytes_moved for r in tr.rows] == list(g[f"{name}_bytes_moved"])


@pytest.fixture(scope="module")
def cfg1_system_f32():
    return DeviceBlockSystem.parallel_beam(CONFIGS[1].spec, dtype="f32")


@pytest.mark.parametrize("name", list(VARIANTS))
def test_fp32_residual_curve_matches_reference(cfg1_system_f32, cfg1_runs, name):
    """FP32 value storage (FP32 streamed inner products over FP32-staged
    (g, x), FP64 reductions and state; csrc/epoch.cu header): the residual-versus-iteration
    curve of the reference (f64) run within 1e-4 relative (north_star), with
    the identical selection stream."""
    g = cfg1_runs
    rec = {}
    _, tr = run_gcsgd(cfg1_system_f32, g["y"], SolverParams(**VARIANTS[name]),
                      x_true=g["x_true"], plan_record=rec)
    ynorm = np.linalg.norm(g["y"])
    r_dev = ynorm / 10.0 ** (np.array([r.obs_gap_db for r in tr.rows]) / 20.0)
    r_ref = ynorm / 10.0 ** (g[f"{name}_gap"] / 20.0)
    assert np.max(np.abs(r_dev - r_ref) / r_ref) <= 1e-4
    want = unflatten_plans(g[f"{name}_plans"])
    for ep, visits in want.items():
        assert [j for j, _ in rec[ep]] == [j for j, _ in visits]


@pytest.mark.parametrize("name", ["ser_g2", "par_full", "par_mixed", "ser_random"])
def test_teacher_forced_epoch(cfg1_system, cfg1_runs, name):
    g = cfg1_runs
    p = SolverParams(**VARIANTS[name])
    plans = unflatten_plans(g[f"{name}_plans"])
    state = SolverState.initialize(cfg1_system, g["y"])
    z = g[f"{name}_snap10_z"]
    zs, off = [], 0
    for j in range(cfg1_system.n_col_blocks):
        n = cfg1_system.n_local_rows(j)
        zs.append(z[off:off + n])
        off += n
    state.load(g[f"{name}_snap10_x"], g[f"{name}_snap10_r"], zs)
    from paper_1709_00953_b200.sampling import group_beta
    loops = [(j, [(ids[a:a + p.group_size], group_beta(cfg1_system.table, p.b, j,
                                                         ids[a:a + p.group_size]))
                  for a in range(0, ids.size, p.group_size)]) for j, ids in plans[11]]
    EpochExecutor(p.execution_mode).run_epoch(11, loops, state, cfg1_system)
    cfg1_system.commit_epoch()
    assert rel(state.x, g[f"{name}_snap11_x"]) <= 1e-12
    assert rel(state.r, g[f"{name}_snap11_r"]) <= 1e-12
    assert rel(np.concatenate(state.z), g[f"{name}_snap11_z"]) <= 1e-12


# ---------------------------------------------------------------------------
# the reference tests' own systems (fan beam)
# ---------------------------------------------------------------------------

def test_known_answer_final_snr():
    """tests/test_solvers.py:196-202: final SNR 6.416697928678968 +- 1e-9."""
    f = golden("fan12.npz")
    panels, rows, vidx, table, nm, nv = fixture_system_arrays(f)
    sysm = DeviceBlockSystem.from_panels(panels, rows, vidx, table, nm, nv, dtype="f64")
    np.testing.assert_array_equal(sysm.forward(f["x_true"]), f["y"])
    x, tr = run_gcsgd(sysm, f["y"], SolverParams(epochs=30, b=6.0, seed=3), x_true=f["x_true"])
    assert tr.rows[-1].snr_db == pytest.approx(6.416697928678968, abs=1e-9)
    assert rel(x, f["final_x"]) <= 1e-12


@pytest.mark.parametrize("gs", [1, 3])
@pytest.mark.parametrize("mode", ["serial_faithful", "parallel"])
def test_literal_epochs(gs, mode):
    """tests/test_solvers.py:125-145 (LiteralSequential at 1e-12)."""
    f = golden("fan10.npz")
    panels, rows, vidx, table, nm, nv = fixture_system_arrays(f)
    sysm = DeviceBlockSystem.from_panels(panels, rows, vidx, table, nm, nv, dtype="f64")
    rec = {}
    x, _ = run_gcsgd(sysm, f["y"], SolverParams(epochs=4, b=6.0, group_size=gs, seed=17,
                                               execution_mode=mode,
                                               sampling=SamplingConfig(alpha=0.5)),
                     x_true=f["x_true"], plan_record=rec)
    want = f[f"x_{gs}_{mode}"]
    assert np.abs(x - want).max() <= 1e-12 * max(np.abs(want).max(), 1.0)


@pytest.fixture(scope="module")
def exec_system():
    f = golden("exec10.npz")
    panels, rows, vidx, table, nm, nv = fixture_system_arrays(f)
    return f, DeviceBlockSystem.from_panels(panels, rows, vidx, table, nm, nv, dtype="f64")


EXEC_PLANS = {
    "barrier": [(0, [(np.array([2, 3]), 0.7)]), (1, [(np.array([2, 3]), 0.7)])],
    "workers": [(0, [(np.array([0, 5]), 0.8), (np.array([2, 7]), 0.6)]),
                (1, [(np.array([1, 4, 6]), 0.5)]), (3, [(np.array([3]), 0.9)])],
    "mutate": [(0, [(np.array([0, 5]), 0.8)]), (2, [(np.array([3]), 0.5)])],
}


@pytest.mark.parametrize("name", list(EXEC_PLANS))
@pytest.mark.parametrize("mode", ["serial_faithful", "parallel"])
def test_executor_matches_reference(exec_system, name, mode):
    f, sysm = exec_system
    state = SolverState.initialize(sysm, f["y"], x0=f["x0"])
    stats = EpochExecutor(mode, 1).run_epoch(1, EXEC_PLANS[name], state, sysm)
    tol = 1e-12
    np.testing.assert_allclose(state.xhat, f[f"{name}_{mode}_xhat"], atol=tol, rtol=0)
    np.testing.assert_allclose(state.r, f[f"{name}_{mode}_r"], atol=tol, rtol=0)
    np.testing.assert_allclose(np.concatenate(state.z), f[f"{name}_{mode}_z"], atol=tol, rtol=0)
    np.testing.assert_array_equal(state.counts, f[f"{name}_{mode}_counts"])
    st = f[f"{name}_{mode}_stats"]
    assert (stats.n_tasks, stats.n_loops, stats.bytes_moved, stats.n_degenerate) == tuple(st)
    sysm.commit_epoch()
    np.testing.assert_allclose(state.x, f[f"{name}_{mode}_x"], atol=tol, rtol=0)


def test_degenerate_tasks_accumulate_unchanged_image(exec_system):
    """tests/test_executor.py:131-140."""
    f, sysm = exec_system
    state = SolverState.initialize(sysm, f["y"], x0=f["x0"])
    sysm.set_r(np.zeros(sysm.n_measurements))
    ex = EpochExecutor("serial_faithful", 1)
    stats = ex.run_epoch(1, [(0, [(np.array([0]), 0.8), (np.array([5]), 0.8)])], state, sysm)
    assert stats.n_degenerate == 2
    assert list(ex.last_statuses) == [1, 1]
    v = sysm.voxel_indices(0)
    np.testing.assert_array_equal(state.xhat[v], 2.0 * f["x0"][v])


def test_failed_batch_leaves_no_trace(exec_system):
    """tests/test_executor.py:143-153."""
    f, sysm = exec_system
    state = SolverState.initialize(sysm, f["y"])
    r0 = state.r.copy()
    with pytest.raises(ExecutorError) as info:
        EpochExecutor("serial_faithful", 1).run_epoch(1, [(0, [(np.array([999]), 0.8)])],
                                                      state, sysm)
    assert info.value.task is not None
    assert not np.any(state.xhat) and not np.any(state.counts)
    np.testing.assert_array_equal(state.r, r0)
    assert not np.any(sysm.projection_sum())


def test_warm_start_and_audit(exec_system):
    f, sysm = exec_system
    state = SolverState.initialize(sysm, f["y"], x0=f["x0"])
    assert sysm.audit_drift() == 0.0
    r = state.r
    r[3] += 1e-3
    sysm.set_r(r)
    assert abs(sysm.audit_drift() - 1e-3 / np.abs(f["y"]).max()) < 1e-15


# ---------------------------------------------------------------------------
# device sampler (bct_sample_epoch) == host BlockScheduler, bit for bit
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", list(VARIANTS))
def test_device_sampler_replays_host_plans(cfg1_system, name):
    """Same variates -> same plans, betas and trajectory (x bitwise)."""
    kw = dict(VARIANTS[name])
    kw["epochs"] = min(kw["epochs"], 12)
    p = SolverParams(**kw)
    f = golden("pb_cfg1_runs.npz")
    y, xt = f["y"], f["x_true"]
    rec_h, rec_d = {}, {}
    x_h, tr_h = run_gcsgd(cfg1_system, y, p, x_true=xt, plan_record=rec_h)
    x_d, tr_d = run_gcsgd(cfg1_system, y, p, x_true=xt, plan_record=rec_d, device_sampling=True)
    for e in rec_h:
        assert [(j, [g.tolist() for g in gs]) for j, gs in rec_h[e]] == \
               [(j, [g.tolist() for g in gs]) for j, gs in rec_d[e]]
    assert np.array_equal(x_h, x_d)
    assert [r.bytes_moved for r in tr_h.rows] == [r.bytes_moved for r in tr_d.rows]
    assert [r.snr_db for r in tr_h.rows] == [r.snr_db for r in tr_d.rows]


@pytest.mark.parametrize("gs,alpha,strategy", [(150, 1.0, "importance"), (20, 0.5, "importance"),
                                                (9, 0.3, "mixed"), (150, 1.0, "random")])
def test_device_sampler_many_row_blocks(gs, alpha, strategy):
    """m = 150 row blocks: numpy's pairwise sum in all three regimes
    (<8, 8-accumulator, halved) for the betas, stable ties in the race."""
    spec = ParallelBeamSpec(32, 180, 46, 150, 2)
    sysm = DeviceBlockSystem.parallel_beam(spec, dtype="f64")
    from paper_1709_00953_b200.geometry import add_noise, random_ellipses
    xt = random_ellipses(32, 5, 3)
    y, _ = add_noise(sysm.forward(xt), 0.01, 4)
    p = SolverParams(epochs=4, b=0.2, group_size=gs, seed=21, execution_mode="parallel",
                     sampling=SamplingConfig(strategy=strategy, alpha=alpha, theta0=0.25,
                                             theta_step=0.25))
    rec_h, rec_d = {}, {}
    x_h, _ = run_gcsgd(sysm, y, p, x_true=xt, plan_record=rec_h)
    x_d, _ = run_gcsgd(sysm, y, p, x_true=xt, plan_record=rec_d, device_sampling=True)
    for e in rec_h:
        assert [(j, [g.tolist() for g in gs_]) for j, gs_ in rec_h[e]] == \
               [(j, [g.tolist() for g in gs_]) for j, gs_ in rec_d[e]]
    assert np.array_equal(x_h, x_d)


# ---------------------------------------------------------------------------
# sharded parallel mode on the device (NCCL, world size 1: the pool has one
# GPU; the 2-rank protocol is covered on CPU by tests/test_sharded_gloo.py)
# ---------------------------------------------------------------------------

def test_sharded_device_path_single_rank(cfg1_system):
    import socket

    import torch
    import torch.distributed as dist

    from paper_1709_00953_b200.distributed import run_gcsgd_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1)
    try:
        f = golden("pb_cfg1_runs.npz")
        p = SolverParams(epochs=8, b=0.25, group_size=2, seed=19, execution_mode="parallel",
                         sampling=SamplingConfig(alpha=0.75))
        x_ref, tr_ref = run_gcsgd(cfg1_system, f["y"], p, x_true=f["x_true"])
        x_sh, tr_sh = run_gcsgd_sharded(cfg1_system, f["y"], p, x_true=f["x_true"])
    finally:
        dist.destroy_process_group()
    assert np.array_equal(x_sh, x_ref)
    assert [r.snr_db for r in tr_sh.rows] == [r.snr_db for r in tr_ref.rows]
    assert [r.obs_gap_db for r in tr_sh.rows] == pytest.approx(
        [r.obs_gap_db for r in tr_ref.rows], rel=1e-12)


# ---------------------------------------------------------------------------
# full BASELINE sizes: size-independent properties (the oracle is too slow at
# 512^2 / 1024^2 within a test, so these check invariants instead)
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def cfg3_system():
    return DeviceBlockSystem.parallel_beam(CONFIGS[3].spec, dtype="f32")


def _cfg_params(cfg, epochs, seed=1234):
    return SolverParams(epochs=epochs, b=cfg.b, group_size=cfg.group_size,
                        execution_mode=cfg.mode, seed=seed,
                        sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))


def test_full_size_audit_and_determinism(cfg3_system):
    """512^2 (config 3, batched path): residual bookkeeping audit <= 1e-8
    (tests/test_acceptance.py:146-160) and bitwise run-to-run determinism."""
    from paper_1709_00953_b200.geometry import add_noise, random_ellipses
    cfg = CONFIGS[3]
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, cfg.phantom_seed)
    y, _ = add_noise(cfg3_system.forward(xt), cfg.noise_frac, cfg.noise_seed)
    p = _cfg_params(cfg, 6)
    x1, tr1 = run_gcsgd(cfg3_system, y, p, x_true=xt)
    assert cfg3_system.audit_drift() <= 1e-8
    x2, tr2 = run_gcsgd(cfg3_system, y, p, x_true=xt)
    assert np.array_equal(x1, x2)
    assert [r.obs_gap_db for r in tr1.rows] == [r.obs_gap_db for r in tr2.rows]
    snr = [r.snr_db for r in tr1.rows]
    assert all(b > a for a, b in zip(snr, snr[1:]))   # b = 1/16 converges monotonically


def test_full_size_fixed_point(cfg3_system):
    """x0 = x_true and y = A x_true: every task sees r = 0 exactly (zero
    gradient, status 1) and the image is unchanged bit for bit
    (tests/test_solvers.py:162-168 holds this at 1e-13)."""
    from paper_1709_00953_b200.geometry import random_ellipses
    cfg = CONFIGS[3]
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, cfg.phantom_seed)
    y = cfg3_system.forward(xt)
    x, tr = run_gcsgd(cfg3_system, y, _cfg_params(cfg, 1), x0=xt)
    assert np.array_equal(x, xt)


# ---------------------------------------------------------------------------
# edge cases: empty / excluded column blocks, the largest mask (256 row
# blocks), zero epochs
# ---------------------------------------------------------------------------

def _device_from_oracle(ora, dtype="f64"):
    from paper_1709_00953_b200.system import PanelArrays
    panels = [PanelArrays(ora.data[j], ora.cols[j], ora.indptr[j], ora.rbp[j], ora.l2g[j])
              for j in range(ora.n_col_blocks)]
    return DeviceBlockSystem.from_panels(panels, ora.row_meas, ora.vidx, ora.table.values,
                                         ora.n_measurements, ora.n_voxels, dtype=dtype)


@pytest.mark.parametrize("mode,gs,alpha", [("parallel", 2, 1.0), ("serial_faithful", 1, 0.5)])
def test_empty_panel_is_excluded_and_untouched(mode, gs, alpha):
    """A column block with no entries has a zero table column: the scheduler
    never visits it (sampling.py active_cols), its voxels keep x0, and the rest
    matches the oracle (empty panels also exercise the zero-size layout)."""
    from oracle.oracle import OracleTable, oracle_run_gcsgd
    from paper_1709_00953_b200.geometry import add_noise, random_ellipses
    ora = __import__("oracle.oracle", fromlist=["OracleSystem"]).OracleSystem.parallel_beam(
        16, 20, 24, 4, 4)
    j0 = 2
    ora.data[j0] = np.empty(0)
    ora.cols[j0] = np.empty(0, np.int32)
    ora.indptr[j0] = np.zeros(1, np.int64)
    ora.rbp[j0] = np.zeros(5, np.int64)
    ora.l2g[j0] = np.empty(0, np.int64)
    vals = ora.table.values.copy()
    vals[:, j0] = 0.0
    ora.table = OracleTable(vals, vals.sum(axis=0))
    sysm = _device_from_oracle(ora)
    xt = random_ellipses(16, 3, 0)
    y, _ = add_noise(ora.forward(xt), 0.01, 1)
    rec = {}
    x, _ = run_gcsgd(sysm, y, SolverParams(epochs=6, b=0.4, group_size=gs, seed=9,
                                          execution_mode=mode,
                                          sampling=SamplingConfig(alpha=alpha)),
                     x_true=xt, plan_record=rec)
    assert all(j != j0 for plan in rec.values() for j, _ in plan)
    assert np.all(x[ora.vidx[j0]] == 0.0)
    x_ref, _ = oracle_run_gcsgd(ora, y, 6, 0.4, alpha=alpha, group_size=gs, mode=mode, seed=9)
    assert rel(x, x_ref) <= 1e-10
    assert sysm.audit_drift() <= 1e-12


@pytest.mark.parametrize("mode,gs,alpha", [("serial_faithful", 5, 0.1), ("parallel", 256, 1.0),
                                           ("parallel", 100, 0.7)])
def test_256_row_blocks(mode, gs, alpha):
    """m = BCT_MAX_M = 256 (every mask word in use): device vs oracle."""
    from oracle.oracle import OracleSystem, oracle_run_gcsgd
    from paper_1709_00953_b200.geometry import add_noise, random_ellipses
    spec = ParallelBeamSpec(24, 256, 34, 256, 3)
    ora = OracleSystem.parallel_beam(24, 256, 34, 256, 3)
    sysm = DeviceBlockSystem.parallel_beam(spec, dtype="f64")
    xt = random_ellipses(24, 4, 2)
    y, _ = add_noise(ora.forward(xt), 0.01, 3)
    x, _ = run_gcsgd(sysm, y, SolverParams(epochs=3, b=0.3, group_size=gs, seed=5,
                                          execution_mode=mode,
                                          sampling=SamplingConfig(alpha=alpha)), x_true=xt)
    x_ref, _ = oracle_run_gcsgd(ora, y, 3, 0.3, alpha=alpha, group_size=gs, mode=mode, seed=5)
    assert rel(x, x_ref) <= 1e-10


def test_zero_epochs_returns_start(cfg1_system, cfg1_runs):
    x, tr = run_gcsgd(cfg1_system, cfg1_runs["y"], SolverParams(epochs=0, b=0.5, seed=1))
    assert np.all(x == 0.0) and len(tr.rows) == 0


@pytest.mark.parametrize("i,j", [(0, 0), (2, 1), (3, 3)])
def test_basic_iteration_dense_single_step(cfg1_system, i, j):
    """tests/test_solvers.py:83-101 analogue: one step on block (i, j) against a
    dense numpy computation of g, mu, x_new and z_i at 1e-10."""
    from paper_1709_00953_b200 import basic_iteration
    rng = np.random.default_rng(40 + i + 10 * j)
    rows = cfg1_system.measurement_rows([i])
    vox = cfg1_system.voxel_indices(j)
    pan = cfg1_system.panel(j)
    # dense A_ij (rows of block i x columns of panel j)
    A = np.zeros((rows.size, vox.size))
    rpos = {int(g): q for q, g in enumerate(rows)}
    for lr in range(int(pan.rbp[i]), int(pan.rbp[i + 1])):
        for p_ in range(int(pan.indptr[lr]), int(pan.indptr[lr + 1])):
            A[rpos[int(pan.l2g[lr])], int(pan.cols[p_])] = pan.data[p_]
    r_i = rng.normal(size=rows.size)
    x_j = rng.normal(size=vox.size)
    x_new, z_i, mu = basic_iteration(cfg1_system, i, j, r_i, x_j, 0.7)
    g = A.T @ r_i
    t = A @ g
    mu_ref = 0.7 * (g @ g) / (t @ t)
    assert abs(mu - mu_ref) <= 1e-10 * mu_ref
    assert rel(x_new, x_j + mu_ref * g) <= 1e-10
    assert rel(z_i, A @ (x_j + mu_ref * g)) <= 1e-10
    # zero residual: zero gradient, unchanged image, z = A x_j
    x0, z0, mu0 = basic_iteration(cfg1_system, i, j, np.zeros(rows.size), x_j, 0.7)
    assert mu0 == 0.0 and np.array_equal(x0, x_j) and rel(z0, A @ x_j) <= 1e-12
