"""The reference's own acceptance setups on the host (no GPU): the scan
geometry, partition, silhouette table, projections and the CPU oracle's runs
are bit-identical to the reference's (fixtures from
tests/golden/make_golden_acceptance.py).  This pins the oracle the device
acceptance tests (test_acceptance_device.py) compare against."""

import os

import numpy as np
import pytest

from _acceptance import (a11_geometry, fixtures, panels_match, sha, standard_geometry,
                         unflatten)
from oracle.oracle import OracleSystem, oracle_forward_project, oracle_run_gcsgd
from paper_1709_00953_b200 import scan as S

WORKERS = max(1, min(8, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def fx():
    return fixtures()


@pytest.fixture(scope="module")
def std(fx):
    f, H = fx
    geo, part = standard_geometry()
    vals, _ = S.probability_table(geo, part)
    ora = OracleSystem.scan(geo, part, vals)
    y = oracle_forward_project(geo, f["std_x_true"])
    return geo, part, vals, ora, y


def test_standard_asset_geometry_table_projections(fx, std):
    f, H = fx
    geo, part, vals, ora, y = std
    assert part.n_row_blocks == 720 and part.n_col_blocks == 4
    assert [sha(np.asarray(r, np.int64)) for r in part.rows] == H["std_rows"]
    np.testing.assert_array_equal(vals, f["std_table"])
    assert sha(y) == H["std_y"]      # simulate_projections (phantoms.py:161-170)
    assert panels_match(lambda j: (ora.data[j], ora.cols[j], ora.indptr[j], ora.rbp[j],
                                   ora.l2g[j]), H["std_panels"])


@pytest.mark.parametrize("mode,tag", [("serial_faithful", "ser"), ("parallel", "par")])
def test_a02_oracle_replays_reference(fx, std, mode, tag):
    """A02's runs (200 epochs, b=2, s=100, alpha=0.5, seed 0): the oracle's
    images at epochs 100, 101, 200 and its whole trace equal the reference's."""
    f, H = fx
    geo, part, vals, ora, y = std
    snaps, rec = {}, {}

    def cb(epoch, state, row):
        if epoch in (100, 101):
            snaps[epoch] = state.x.copy()

    x, rows = oracle_run_gcsgd(ora, y, 200, 2.0, alpha=0.5, group_size=100, mode=mode, seed=0,
                               x_true=f["std_x_true"], callback=cb, plan_record=rec,
                               workers=WORKERS)
    assert sha(snaps[100]) == H[f"a02_{tag}_x100"]
    assert sha(snaps[101]) == H[f"a02_{tag}_x101"]
    assert sha(x) == H[f"a02_{tag}_x"]
    np.testing.assert_array_equal([r["snr_db"] for r in rows], f[f"a02_{tag}_snr"])
    np.testing.assert_array_equal([r["obs_gap_db"] for r in rows], f[f"a02_{tag}_gap"])
    want = unflatten(f[f"a02_{tag}_plans"])
    for ep, visits in want.items():
        got = [(j, np.concatenate(g)) for j, g in rec[ep]]
        assert [j for j, _ in got] == [j for j, _ in visits]
        for (_, a), (_, b) in zip(got, visits):
            np.testing.assert_array_equal(a, b)


def test_a10_oracle_replays_reference(fx, std):
    """A10's recorded schedule (parallel, 10 epochs): x after every epoch."""
    f, H = fx
    geo, part, vals, ora, y = std
    sched = unflatten(f["a10_plans"])
    xs = []
    oracle_run_gcsgd(ora, y, 10, 2.0, alpha=0.5, group_size=100, mode="parallel", seed=3,
                     schedule=sched, callback=lambda e, st, r: xs.append(st.x.copy()),
                     workers=WORKERS)
    assert [sha(v) for v in xs] == H["a10_x"]


def test_a11_geometry_and_oracle_run(fx):
    """A11 (3D smoke run): random-sphere poses, partition, table, panels and
    y bitwise; the oracle's b ladder picks the reference's b and its 50-epoch
    image equals the reference's."""
    f, H = fx
    geo, part = a11_geometry()
    P = np.array([np.concatenate([p.source, p.detector_center, p.det_u, p.det_v])
                  for p in geo.poses])
    np.testing.assert_array_equal(P, f["a11_poses"])
    assert part.n_row_blocks == 360 and part.n_col_blocks == 8
    vals, _ = S.probability_table(geo, part)
    np.testing.assert_array_equal(vals, f["a11_table"])
    y = oracle_forward_project(geo, f["a11_x_true"])
    assert sha(y) == H["a11_y"]
    ora = OracleSystem.scan(geo, part, vals)
    assert panels_match(lambda j: (ora.data[j], ora.cols[j], ora.indptr[j], ora.rbp[j],
                                   ora.l2g[j]), H["a11_panels"])
    b = float(f["a11_b"])
    x, rows = oracle_run_gcsgd(ora, y, 50, b, group_size=16, seed=0, x_true=f["a11_x_true"])
    assert sha(x) == H["a11_x"]
    np.testing.assert_array_equal([r["snr_db"] for r in rows], f["a11_snr"])
