"""General scan geometry (fan / cone beam): host partition + silhouette table
pinned bitwise to the reference's own fan-beam fixtures, the oracle's general
assembly pinned to the fixture panels, and (GPU) the device tracer
(bct_create_scan) equal to both, including the reference's known-answer SNR
(tests/test_solvers.py:196-202 of the reference)."""

import numpy as np
import pytest

from conftest import golden
from paper_1709_00953_b200.errors import ConfigurationError, GeometryError
from paper_1709_00953_b200.scan import (DetectorModel, ScanGeometry, ViewPose, VolumeGrid,
                                        circular_trajectory, make_partition, probability_table)

# make_golden.py: fan(n_views, det_px, dims, radius), splits (2, 2), det_splits 2
FANS = {"fan12": (10, 14, (12, 12), 20.0), "fan10": (8, 12, (10, 10), 18.0)}


def fan_geometry(name):
    nv, px, dims, radius = FANS[name]
    return ScanGeometry(VolumeGrid(dims, (1.0, 1.0)), DetectorModel(px, 1.5),
                        tuple(circular_trajectory(nv, radius)))


def cone_geometry():
    """Small 3D cone beam with anisotropic voxels, an off-centre origin, a
    2D detector and a tilted circular orbit -- no reference fixture exists,
    so the device is checked against the oracle (pinned on the fan cases)."""
    grid = VolumeGrid((9, 7, 6), (1.0, 1.25, 0.8), origin=(-4.3, -4.1, -2.2))
    det = DetectorModel((11, 7), (1.6, 1.3))
    poses = []
    for k, pose in enumerate(circular_trajectory(7, 22.0, angular_start=0.3)):
        lift = np.array([0.0, 0.0, 1.5 * np.sin(0.9 * k)])
        poses.append(ViewPose(pose.source + lift, pose.detector_center - lift, pose.det_u,
                              pose.det_v))
    return ScanGeometry(grid, det, tuple(poses))


@pytest.mark.parametrize("name", list(FANS))
def test_partition_and_table_bitwise(name):
    f = golden(f"{name}.npz")
    geo = fan_geometry(name)
    part = make_partition(geo, (2, 2), 2)
    assert part.n_row_blocks == int(f["m"]) and part.n_col_blocks == int(f["nc"])
    for i in range(part.n_row_blocks):
        np.testing.assert_array_equal(part.rows[i], f[f"rows{i}"])
    for j in range(part.n_col_blocks):
        np.testing.assert_array_equal(part.vidx[j], f[f"vidx{j}"])
    vals, totals = probability_table(geo, part)
    assert vals.tobytes() == np.asarray(f["table"], np.float64).tobytes()
    assert totals.tobytes() == f["table"].sum(axis=0).tobytes()


def _panels_equal(a, b, j):
    for k in ("data", "cols", "indptr", "rbp", "l2g"):
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.shape == y.shape, (j, k)
        if k == "data":
            assert x.tobytes() == np.asarray(y, np.float64).tobytes(), (j, k)
        else:
            np.testing.assert_array_equal(x.astype(np.int64), y.astype(np.int64), err_msg=f"{j} {k}")


@pytest.mark.parametrize("name", list(FANS))
def test_oracle_scan_assembly_pinned(name):
    from oracle.oracle import OracleSystem
    f = golden(f"{name}.npz")
    geo = fan_geometry(name)
    part = make_partition(geo, (2, 2), 2)
    vals, _ = probability_table(geo, part)
    o = OracleSystem.scan(geo, part, vals)
    for j in range(part.n_col_blocks):
        _panels_equal({"data": o.data[j], "cols": o.cols[j], "indptr": o.indptr[j],
                       "rbp": o.rbp[j], "l2g": o.l2g[j]},
                      {k: f[f"{k}{j}"] for k in ("data", "cols", "indptr", "rbp", "l2g")}, j)


def test_cone_table_and_partition_shapes():
    geo = cone_geometry()
    part = make_partition(geo, (2, 2, 2), (2, 2))
    assert part.n_col_blocks == 8 and part.n_row_blocks == 7 * 4
    assert sum(v.size for v in part.vidx) == geo.grid.n_voxels
    assert np.array_equal(np.sort(np.concatenate(part.rows)), np.arange(geo.n_measurements))
    vals, totals = probability_table(geo, part)
    assert (vals >= 0).all() and (totals > 0).all()


def test_partition_errors():
    geo = fan_geometry("fan10")
    with pytest.raises(ConfigurationError):
        make_partition(geo, (11, 2), 2)
    with pytest.raises(ConfigurationError):
        make_partition(geo, (2, 2), 13)
    inside = ScanGeometry(geo.grid, geo.detector,
                          (ViewPose(np.array([0.2, 0.1, 0.0]), np.array([-9.0, 0.0, 0.0]),
                                    np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0])),))
    with pytest.raises(GeometryError):
        probability_table(inside, make_partition(inside, (2, 2), 1))


# ---------------------------------------------------------------------------
# device tracer
# ---------------------------------------------------------------------------

def _device_panels(sysm, j):
    p = sysm.panel(j)
    return {"data": p.data, "cols": p.cols, "indptr": p.indptr, "rbp": p.rbp, "l2g": p.l2g}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(FANS))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_device_scan_panels_bitwise(name, dtype):
    from paper_1709_00953_b200.system import DeviceBlockSystem
    f = golden(f"{name}.npz")
    sysm = DeviceBlockSystem.scan(fan_geometry(name), volume_splits=(2, 2), detector_splits=2,
                                  dtype=dtype)
    assert sysm.table.values.tobytes() == np.asarray(f["table"], np.float64).tobytes()
    for j in range(int(f["nc"])):
        p = _device_panels(sysm, j)
        want = {k: f[f"{k}{j}"] for k in ("data", "cols", "indptr", "rbp", "l2g")}
        if dtype == "f32":
            # the store keeps FP32 values; structure is exact, values rounded once
            np.testing.assert_array_equal(np.asarray(p["data"]),
                                          want["data"].astype(np.float32).astype(np.float64))
            p = dict(p, data=want["data"])
        _panels_equal(p, want, j)
    sysm.close()


@pytest.mark.gpu
def test_device_scan_known_answer_snr():
    """The reference's known answer on the device-traced fan-beam system."""
    from paper_1709_00953_b200 import SolverParams, run_gcsgd
    from paper_1709_00953_b200.system import DeviceBlockSystem
    f = golden("fan12.npz")
    sysm = DeviceBlockSystem.scan(fan_geometry("fan12"), volume_splits=(2, 2), detector_splits=2)
    np.testing.assert_array_equal(sysm.forward(f["x_true"]), f["y"])
    x, tr = run_gcsgd(sysm, f["y"], SolverParams(epochs=30, b=6.0, seed=3), x_true=f["x_true"])
    assert tr.rows[-1].snr_db == pytest.approx(6.416697928678968, abs=1e-9)
    assert np.abs(x - f["final_x"]).max() <= 1e-12 * np.abs(f["final_x"]).max()
    sysm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("splits", [((2, 2, 2), (2, 2)), ((3, 1, 2), (1, 3)), ((1, 1, 1), 1)])
def test_device_cone_beam_vs_oracle(splits):
    from oracle.oracle import OracleSystem
    from paper_1709_00953_b200.system import DeviceBlockSystem
    geo = cone_geometry()
    part = make_partition(geo, *splits)
    vals, _ = probability_table(geo, part)
    o = OracleSystem.scan(geo, part, vals)
    sysm = DeviceBlockSystem.scan(geo, partition=part)
    for j in range(part.n_col_blocks):
        _panels_equal(_device_panels(sysm, j),
                      {"data": o.data[j], "cols": o.cols[j], "indptr": o.indptr[j],
                       "rbp": o.rbp[j], "l2g": o.l2g[j]}, j)
    x = np.random.default_rng(5).random(geo.grid.n_voxels)
    np.testing.assert_array_equal(sysm.forward(x), o.forward(x))
    sysm.close()


@pytest.mark.gpu
def test_device_scan_geometry_errors():
    """projector.py:278-284 / 591-592: a source inside a block or a degenerate
    ray raise GeometryError (the table is passed in, so the device checks)."""
    from paper_1709_00953_b200.sampling import ProbabilityTable
    from paper_1709_00953_b200.system import DeviceBlockSystem
    geo = fan_geometry("fan10")
    e = (np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0]))
    inside = ScanGeometry(geo.grid, geo.detector,
                          (ViewPose(np.array([0.2, 0.1, 0.0]), np.array([-9.0, 0.0, 0.0]), *e),))
    part = make_partition(inside, (2, 2), 1)
    tab = ProbabilityTable(np.ones((1, 4)), np.ones(4))
    with pytest.raises(GeometryError):
        DeviceBlockSystem.scan(inside, partition=part, table=tab)
    src = np.array([-20.0, 0.0, 0.0])
    degen = ScanGeometry(geo.grid, DetectorModel(1, 1.0), (ViewPose(src, src.copy(), *e),))
    part = make_partition(degen, (2, 2), 1)
    with pytest.raises(GeometryError):
        DeviceBlockSystem.scan(degen, partition=part, table=tab)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["serial_faithful", "parallel"])
def test_device_cone_beam_solver_vs_oracle(mode):
    """run_gcsgd on the device-traced cone-beam system == the oracle run."""
    from oracle.oracle import OracleSystem, oracle_run_gcsgd
    from paper_1709_00953_b200 import SamplingConfig, SolverParams, run_gcsgd
    from paper_1709_00953_b200.system import DeviceBlockSystem
    geo = cone_geometry()
    part = make_partition(geo, (2, 2, 2), (2, 2))
    vals, _ = probability_table(geo, part)
    o = OracleSystem.scan(geo, part, vals)
    xt = np.random.default_rng(2).random(geo.grid.n_voxels)
    y = o.forward(xt)
    want, rows = oracle_run_gcsgd(o, y, 5, 4.0, alpha=0.5, group_size=2, mode=mode, seed=11,
                                  x_true=xt)
    sysm = DeviceBlockSystem.scan(geo, partition=part)
    x, tr = run_gcsgd(sysm, y, SolverParams(epochs=5, b=4.0, group_size=2, seed=11,
                                            execution_mode=mode,
                                            sampling=SamplingConfig(alpha=0.5)), x_true=xt)
    assert np.abs(x - want).max() <= 1e-10 * max(np.abs(want).max(), 1.0)
    assert tr.rows[-1].snr_db == pytest.approx(rows[-1]["snr_db"], abs=1e-8)
    sysm.close()
