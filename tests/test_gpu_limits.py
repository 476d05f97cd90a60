"""Device limits and plan shapes the reference supports: many row blocks
(m > 256: the reference's own fan-beam assets use 360 and 720), panels with
many super tiles, and scripted plans that visit a column block twice in one
epoch.  Every case is checked against the CPU oracle (FP64 at 1e-10
free-running, 1e-12 for one epoch)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

bct = pytest.importorskip("paper_1709_00953_b200")
from oracle.oracle import (OracleState, OracleSystem, OracleTable,  # noqa: E402
                           oracle_commit_epoch, oracle_run_epoch, oracle_run_gcsgd)
from paper_1709_00953_b200 import (DeviceBlockSystem, EpochExecutor, PanelArrays,  # noqa: E402
                                   SamplingConfig, SolverParams, SolverState, add_noise,
                                   random_ellipses, run_gcsgd)
from paper_1709_00953_b200.geometry import ParallelBeamSpec  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def device_from_oracle(ora, dtype="f64"):
    panels = [PanelArrays(ora.data[j], ora.cols[j], ora.indptr[j], ora.rbp[j], ora.l2g[j])
              for j in range(ora.n_col_blocks)]
    return DeviceBlockSystem.from_panels(panels, ora.row_meas, ora.vidx, ora.table.values,
                                         ora.n_measurements, ora.n_voxels, dtype=dtype)


# ---------------------------------------------------------------------------
# m > 256 row blocks
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def many_blocks():
    n, views, bins, m, nc = 24, 720, 34, 720, 3
    ora = OracleSystem.parallel_beam(n, views, bins, m, nc)
    dev = DeviceBlockSystem.parallel_beam(ParallelBeamSpec(n, views, bins, m, nc), dtype="f64")
    xt = random_ellipses(n, 4, 2)
    y, _ = add_noise(ora.forward(xt), 0.01, 3)
    return ora, dev, xt, y


@pytest.mark.parametrize("mode,gs,alpha,strategy", [
    ("serial_faithful", 5, 0.02, "importance"),
    ("serial_faithful", 1, 0.005, "mixed"),
    ("parallel", 720, 1.0, "importance"),
    ("parallel", 100, 0.7, "importance"),
    ("parallel", 37, 0.4, "random"),
])
def test_720_row_blocks_match_oracle(many_blocks, mode, gs, alpha, strategy):
    """m = 720 (the reference's standard asset has 360 views x 2 detector
    blocks = 720): plans, x and the residual against the oracle, host and
    device sampling."""
    ora, dev, xt, y = many_blocks
    E = 3
    sc = SamplingConfig(strategy=strategy, alpha=alpha, theta0=0.25, theta_step=0.25)
    p = SolverParams(epochs=E, b=0.3, group_size=gs, seed=5, execution_mode=mode, sampling=sc)
    rec_o = {}
    x_ref, _ = oracle_run_gcsgd(ora, y, E, 0.3, alpha=alpha, group_size=gs, mode=mode, seed=5,
                                strategy=strategy, theta0=0.25, theta_step=0.25,
                                plan_record=rec_o)
    for device_sampling in (False, True):
        rec = {}
        x, _ = run_gcsgd(dev, y, p, x_true=xt, plan_record=rec, device_sampling=device_sampling)
        for e in rec_o:
            assert [(j, [g.tolist() for g in gs_]) for j, gs_ in rec[e]] == \
                   [(j, [g.tolist() for g in gs_]) for j, gs_ in rec_o[e]]
        assert rel(x, x_ref) <= 1e-10
        assert dev.audit_drift() <= 1e-12


# ---------------------------------------------------------------------------
# panels with many super tiles (a large generic column block)
# ---------------------------------------------------------------------------

def random_system(n_meas, n_vox, m, nc, per_row, seed):
    """Sparse random blocked system in the reference's cached layout: rows
    with ``per_row`` random columns of a contiguous voxel block each."""
    rng = np.random.default_rng(seed)
    redges = np.round(np.linspace(0, n_meas, m + 1)).astype(np.int64)
    row_meas = [np.arange(redges[i], redges[i + 1], dtype=np.int64) for i in range(m)]
    cedges = np.round(np.linspace(0, n_vox, nc + 1)).astype(np.int64)
    vidx = [np.arange(cedges[j], cedges[j + 1], dtype=np.int64) for j in range(nc)]
    data, cols, indptr, rbp, l2g = [], [], [], [], []
    for j in range(nc):
        w = vidx[j].size
        d_parts, c_parts, cnt, hit = [], [], [], []
        rb = np.zeros(m + 1, np.int64)
        for i in range(m):
            h = 0
            for g in row_meas[i]:
                if rng.uniform() < 0.15:
                    continue   # rows missing the block are not stored
                cc = np.sort(rng.choice(w, size=per_row, replace=False)).astype(np.int32)
                d_parts.append(rng.uniform(0.05, 1.5, size=per_row))
                c_parts.append(cc)
                cnt.append(per_row)
                hit.append(g)
                h += 1
            rb[i + 1] = rb[i] + h
        ip = np.zeros(len(cnt) + 1, np.int64)
        np.cumsum(cnt, out=ip[1:])
        data.append(np.concatenate(d_parts)); cols.append(np.concatenate(c_parts))
        indptr.append(ip); rbp.append(rb); l2g.append(np.array(hit, np.int64))
    vals = np.zeros((m, nc))
    for j in range(nc):
        vals[:, j] = np.diff(indptr[j][rbp[j]]) + 1.0
    return OracleSystem(data, cols, indptr, rbp, l2g, row_meas, vidx,
                        OracleTable(vals, vals.sum(axis=0)), n_meas, n_vox)


@pytest.mark.parametrize("mode,gs,alpha", [("serial_faithful", 1, 0.5), ("parallel", 2, 1.0),
                                           ("parallel", 3, 1.0)])
def test_many_super_tiles_match_oracle(mode, gs, alpha):
    """One 330,000-voxel column block: 81 FP64 super tiles (the per-task
    record sizes its slice prefix from the context)."""
    ora = random_system(1500, 330000, 3, 1, 40, 7)
    dev = device_from_oracle(ora)
    x_true = np.random.default_rng(3).uniform(0, 1, ora.n_voxels)
    y = ora.forward(x_true)
    p = SolverParams(epochs=3, b=0.5, group_size=gs, seed=4, execution_mode=mode,
                     sampling=SamplingConfig(alpha=alpha))
    x, _ = run_gcsgd(dev, y, p, x_true=x_true)
    x_ref, _ = oracle_run_gcsgd(ora, y, 3, 0.5, alpha=alpha, group_size=gs, mode=mode, seed=4)
    assert rel(x, x_ref) <= 1e-10
    dev.close()


# ---------------------------------------------------------------------------
# scripted plans that revisit a column block within an epoch
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def small():
    ora = OracleSystem.parallel_beam(16, 20, 24, 4, 4)
    dev = device_from_oracle(ora)
    xt = random_ellipses(16, 3, 0)
    y, _ = add_noise(ora.forward(xt), 0.01, 1)
    return ora, dev, xt, y


FULL = np.arange(4)
REVISIT_PLANS = {
    # two visits of block 1, each a full panel (batched-path shape)
    "two_visits": [(1, [(FULL, 0.3)]), (0, [(FULL, 0.25)]), (1, [(FULL[::-1], 0.2)])],
    # one visit with two full-panel groups
    "two_groups": [(2, [(FULL, 0.3), (np.array([3, 1, 0, 2]), 0.15)]), (3, [(FULL, 0.2)])],
    "mixed": [(0, [(np.array([1, 2]), 0.3)]), (0, [(FULL, 0.2)]), (2, [(FULL, 0.1)])],
}


@pytest.mark.parametrize("name", list(REVISIT_PLANS))
@pytest.mark.parametrize("mode", ["parallel", "serial_faithful"])
def test_revisited_blocks_match_oracle(small, name, mode):
    """executor.py:200-213, 247-248: z commits in plan order (the last task
    wins), x_hat sums every task, counts every task."""
    ora, dev, xt, y = small
    loops = REVISIT_PLANS[name]
    st_o = OracleState.initialize(ora, y, x0=xt * 0.5)
    oracle_run_epoch(ora, st_o, loops, mode)
    xhat_o = st_o.xhat.copy()
    counts_o = st_o.counts.copy()
    oracle_commit_epoch(st_o, ora)
    st = SolverState.initialize(dev, y, x0=xt * 0.5)
    EpochExecutor(mode).run_epoch(1, loops, st, dev)
    assert rel(st.xhat, xhat_o) <= 1e-12
    np.testing.assert_array_equal(st.counts, counts_o)
    dev.commit_epoch()
    assert rel(st.x, st_o.x) <= 1e-12
    assert rel(st.r, st_o.r) <= 1e-12
    assert rel(np.concatenate(st.z), np.concatenate(st_o.z)) <= 1e-12


# ---------------------------------------------------------------------------
# single-buffered phase-1 bands (a shape whose two FP64 bands exceed shared
# memory: FP32 contexts at config 5's 1440 views take 8x8 tiles this way)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("mode,gs", [("serial_faithful", 2), ("parallel", 3), ("parallel", 6)])
def test_single_buffered_bands_match_double_buffered(monkeypatch, dtype, mode, gs):
    """The same 8x8-tile layout with one band buffer (BCT_TILE_NBUF1) and with
    two gives bitwise the same run on the per-task and batched paths, and the
    FP64 run matches the oracle."""
    n, views, bins, m, nc = 32, 48, 46, 6, 4
    spec = ParallelBeamSpec(n, views, bins, m, nc)
    xt = random_ellipses(n, 4, 5)
    ora = OracleSystem.parallel_beam(n, views, bins, m, nc)
    y, _ = add_noise(ora.forward(xt), 0.01, 6)
    p = SolverParams(epochs=4, b=0.3, group_size=gs, seed=9, execution_mode=mode,
                     sampling=SamplingConfig(alpha=0.6))
    xs = []
    for nbuf1 in (False, True):
        monkeypatch.setenv("BCT_TILE", "8x8")
        if nbuf1:
            monkeypatch.setenv("BCT_TILE_NBUF1", "1")
        else:
            monkeypatch.delenv("BCT_TILE_NBUF1", raising=False)
        dev = DeviceBlockSystem.parallel_beam(spec, dtype=dtype)
        x, _ = run_gcsgd(dev, y, p, x_true=xt)
        xs.append(np.array(x))
        dev.close()
    assert np.array_equal(xs[0], xs[1])
    if dtype == "f64":
        x_ref, _ = oracle_run_gcsgd(ora, y, 4, 0.3, alpha=0.6, group_size=gs, mode=mode, seed=9)
        assert rel(xs[1], x_ref) <= 1e-10


# ---------------------------------------------------------------------------
# column blocks wider than 128 pixel columns (the device tracer's fill kernel
# orders a ray's entries from the walk's directions, without a per-column table)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,views,bins,m,nc", [(160, 24, 230, 3, 1), (300, 16, 430, 2, 2)])
def test_wide_strip_panels_match_oracle(n, views, bins, m, nc):
    ora = OracleSystem.parallel_beam(n, views, bins, m, nc)
    dev = DeviceBlockSystem.parallel_beam(ParallelBeamSpec(n, views, bins, m, nc), dtype="f64")
    for j in range(nc):
        p = dev.panel(j)
        np.testing.assert_array_equal(p.data, ora.data[j])
        np.testing.assert_array_equal(p.cols, ora.cols[j])
        np.testing.assert_array_equal(p.indptr, ora.indptr[j])
        np.testing.assert_array_equal(p.rbp, ora.rbp[j])
        np.testing.assert_array_equal(p.l2g, ora.l2g[j])
    xt = random_ellipses(n, 4, 7)
    y = ora.forward(xt)
    np.testing.assert_array_equal(dev.forward(xt), y)
    p = SolverParams(epochs=3, b=0.4, group_size=m, seed=2, execution_mode="parallel")
    x, _ = run_gcsgd(dev, y, p, x_true=xt)
    x_ref, _ = oracle_run_gcsgd(ora, y, 3, 0.4, group_size=m, mode="parallel", seed=2)
    assert rel(x, x_ref) <= 1e-10
    dev.close()
