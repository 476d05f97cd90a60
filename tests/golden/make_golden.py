"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package itself (``/root/reference/pkg/src/blockct``) in this container.

Run once (needs /root/reference, numba and a writable NUMBA_CACHE_DIR):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Nothing at test time reads /root/reference: the tests load these .npz/.json
files only.  What each fixture pins:

* pb_small.npz      -- parallel-beam strip panels traced by the reference's
                       ``projector._trace_ray_kernel`` (16^2, 20 views x 24 bins,
                       4x4 blocks), stored in full.
* pb_hashes.json    -- sha256 of every panel array for configs 1 and 2 traced
                       the same way (too large to store; the device builder and
                       the C oracle must reproduce them bit for bit).
* pb_cfg1_runs.npz  -- reference ``run_gcsgd`` on the config-1 system injected
                       into a cached ``BlockSystem``: the P1 run
                       (serial, s=1, alpha=0.25, b=0.5, 500 epochs) plus grouped
                       and parallel variants; final x, per-epoch trace, plans,
                       and a mid-run state snapshot for teacher forcing.
* fan12.npz / fan10.npz / exec10.npz -- the reference tests' own fan-beam
                       systems (test_solvers.py:19-28, test_executor.py:14-23)
                       exported as panels, with the reference's outputs,
                       including the known-answer final SNR 6.416697928678968
                       (test_solvers.py:196-202).
"""

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from blockct import (BlockSystem, DetectorModel, ProbabilityTable,  # noqa: E402
                     SamplingConfig, ScanGeometry, SolverParams, SolverState,
                     VolumeGrid, build_probability_table, head_phantom,
                     make_circular_trajectory, make_partition, run_gcsgd)
from blockct import executor as ref_executor  # noqa: E402
from blockct import projector as ref_projector  # noqa: E402
from blockct import solvers as ref_solvers  # noqa: E402

from paper_1709_00953_b200.geometry import (CONFIGS, ParallelBeamSpec,  # noqa: E402
                                            add_noise, random_ellipses)


# ---------------------------------------------------------------------------
# parallel-beam harness around the reference tracer
# ---------------------------------------------------------------------------

class _RB:
    def __init__(self, index, meas):
        self.index = index
        self.measurement_indices = meas
        self.size = int(meas.size)


class _VB:
    def __init__(self, index, vox):
        self.index = index
        self.voxel_indices = vox
        self.size = int(vox.size)


class _Part:
    def __init__(self, rbs, vbs):
        self.row_blocks = tuple(rbs)
        self.col_blocks = tuple(vbs)
        self.n_row_blocks = len(rbs)
        self.n_col_blocks = len(vbs)


class _Grid:
    def __init__(self, n_voxels):
        self.n_voxels = n_voxels


class _Geo:
    def __init__(self, n_meas, n_vox):
        self.n_measurements = n_meas
        self.grid = _Grid(n_vox)


def ref_parallel_beam_panels(spec: ParallelBeamSpec):
    """Trace every (ray, strip) pair with the reference's numba kernel."""
    n, views, bins = spec.n, spec.views, spec.bins
    grid = VolumeGrid((n, n), (1.0, 1.0))
    origin = np.asarray(grid.origin, dtype=np.float64)
    vsize = np.asarray(grid.voxel_size, dtype=np.float64)
    c, s = spec.trig()
    u = np.arange(bins) - (bins - 1) / 2
    L = 4.0 * n
    cx = u[None, :] * (-s)[:, None]
    cy = u[None, :] * c[:, None]
    lc = (L * c)[:, None]
    ls = (L * s)[:, None]
    src = np.stack([(cx - lc).ravel(), (cy - ls).ravel(), np.zeros(views * bins)], 1)
    dst = np.stack([(cx + lc).ravel(), (cy + ls).ravel(), np.zeros(views * bins)], 1)
    aedges = spec.angle_edges() * bins
    xe = spec.strip_edges()
    panels = []
    for j in range(spec.nc):
        lo = np.array([xe[j], 0, 0], dtype=np.int64)
        hi = np.array([xe[j + 1], n, 1], dtype=np.int64)
        cap = int((hi - lo).sum() + 3)
        idx = np.empty(cap, dtype=np.int64)
        lng = np.empty(cap, dtype=np.float64)
        d_parts, c_parts, counts, hits = [], [], [], []
        for r in range(views * bins):
            cnt = ref_projector._trace_ray_kernel(np.ascontiguousarray(src[r]),
                                                  np.ascontiguousarray(dst[r]),
                                                  origin, vsize, lo, hi, idx, lng)
            assert cnt >= 0
            if cnt > 0:
                d_parts.append(lng[:cnt].copy())
                c_parts.append(idx[:cnt].astype(np.int32))
                counts.append(cnt)
                hits.append(r)
        l2g = np.array(hits, dtype=np.int64)
        indptr = np.zeros(len(counts) + 1, dtype=np.int64)
        np.cumsum(counts, out=indptr[1:])
        rbp = np.searchsorted(l2g, aedges, side="left").astype(np.int64)
        panels.append(dict(data=np.concatenate(d_parts), cols=np.concatenate(c_parts),
                           indptr=indptr, rbp=rbp, l2g=l2g))
    return panels


def density_table(spec, panels):
    vals = np.zeros((spec.m, spec.nc))
    rsz = np.array([r.size for r in spec.row_meas()])
    vox = spec.voxel_indices()
    for j, p in enumerate(panels):
        vals[:, j] = np.diff(p["indptr"][p["rbp"]]) / (rsz * vox[j].size)
    return vals


def inject(spec, panels, values):
    part = _Part([_RB(i, r) for i, r in enumerate(spec.row_meas())],
                 [_VB(j, v) for j, v in enumerate(spec.voxel_indices())])
    table = ProbabilityTable(values, values.sum(axis=0))
    system = BlockSystem(_Geo(spec.n_measurements, spec.n_voxels), part, table, "cached")
    system._data = [p["data"] for p in panels]
    system._cols = [p["cols"] for p in panels]
    system._indptr = [p["indptr"] for p in panels]
    system._rbp = [p["rbp"] for p in panels]
    system._l2g = [p["l2g"] for p in panels]
    system.nnz = int(sum(p["data"].size for p in panels))
    return system


def panel_hash(p):
    h = {}
    for k in ("data", "cols", "indptr", "rbp", "l2g"):
        h[k] = hashlib.sha256(np.ascontiguousarray(p[k]).tobytes()).hexdigest()
    h["nnz"] = int(p["data"].size)
    h["rows"] = int(p["l2g"].size)
    return h


def export_system(system):
    """Flatten a reference cached BlockSystem into npz-able arrays."""
    out = {}
    nc = system.partition.n_col_blocks
    m = system.partition.n_row_blocks
    out["nc"] = np.int64(nc)
    out["m"] = np.int64(m)
    out["n_meas"] = np.int64(system.n_measurements)
    out["n_vox"] = np.int64(system.n_voxels)
    for j in range(nc):
        out[f"data{j}"] = system._data[j]
        out[f"cols{j}"] = system._cols[j]
        out[f"indptr{j}"] = system._indptr[j]
        out[f"rbp{j}"] = system._rbp[j]
        out[f"l2g{j}"] = system._l2g[j]
        out[f"vidx{j}"] = np.asarray(system.voxel_indices(j), dtype=np.int64)
    for i in range(m):
        out[f"rows{i}"] = np.asarray(system.partition.row_blocks[i].measurement_indices,
                                     dtype=np.int64)
    out["table"] = np.asarray(system.table.values, dtype=np.float64)
    return out


def flatten_plans(rec):
    """plan_record -> (P, 3+max_ids) int64 table: epoch, j, group_size..."""
    rows = []
    for ep in sorted(rec):
        for j, groups in rec[ep]:
            ids = np.concatenate(groups) if groups else np.empty(0, np.int64)
            rows.append([ep, j, len(ids)] + [int(i) for i in ids])
    width = max(len(r) for r in rows)
    arr = -np.ones((len(rows), width), dtype=np.int64)
    for k, r in enumerate(rows):
        arr[k, :len(r)] = r
    return arr


def run_and_record(system, y, params, x_true=None, x0=None, snap_epochs=()):
    rec = {}
    snaps = {}

    def cb(epoch, state, row):
        if epoch in snap_epochs:
            snaps[epoch] = (state.x.copy(), state.r.copy(),
                            np.concatenate(state.z).copy())
    x, tr = run_gcsgd(system, y, params, x_true=x_true, x0=x0, plan_record=rec, callback=cb)
    out = dict(x=x, snr=np.array([r.snr_db for r in tr.rows]),
               gap=np.array([r.obs_gap_db for r in tr.rows]),
               n_tasks=np.array([r.n_tasks for r in tr.rows]),
               bytes_moved=np.array([r.bytes_moved for r in tr.rows]),
               plans=flatten_plans(rec))
    for ep, (sx, sr, sz) in snaps.items():
        out[f"snap{ep}_x"] = sx
        out[f"snap{ep}_r"] = sr
        out[f"snap{ep}_z"] = sz
    return out


# ---------------------------------------------------------------------------

def main():
    hashes = {}

    # 1. small parallel-beam system, stored whole
    small = ParallelBeamSpec(16, 20, 24, 4, 4)
    sp = ref_parallel_beam_panels(small)
    svals = density_table(small, sp)
    out = {"table": svals}
    for j, p in enumerate(sp):
        for k, v in p.items():
            out[f"{k}{j}"] = v
    sysm = inject(small, sp, svals)
    xs = random_ellipses(16, 4, 0)
    out["x_true"] = xs
    out["y_clean"] = sysm.forward(xs)
    np.savez_compressed(os.path.join(HERE, "pb_small.npz"), **out)
    hashes["small"] = [panel_hash(p) for p in sp]
    print("pb_small nnz", sum(p["data"].size for p in sp))

    # 2. configs 1 and 2 traced by the reference: hashes only
    for key in (1, 2):
        cfg = CONFIGS[key]
        panels = ref_parallel_beam_panels(cfg.spec)
        hashes[f"cfg{key}"] = [panel_hash(p) for p in panels]
        vals = density_table(cfg.spec, panels)
        hashes[f"cfg{key}_table_sha"] = hashlib.sha256(vals.tobytes()).hexdigest()
        print(f"cfg{key} nnz", sum(p["data"].size for p in panels))
        if key == 1:
            cfg1_panels, cfg1_vals = panels, vals
    with open(os.path.join(HERE, "pb_hashes.json"), "w") as fh:
        json.dump(hashes, fh, indent=1)

    # 3. reference runs on the injected config-1 system
    cfg = CONFIGS[1]
    system = inject(cfg.spec, cfg1_panels, cfg1_vals)
    x_true = random_ellipses(64, cfg.n_ellipses, cfg.phantom_seed)
    y_clean = system.forward(x_true)
    y, sigma = add_noise(y_clean, cfg.noise_frac, cfg.noise_seed)
    runs = {"x_true": x_true, "y_clean": y_clean, "y": y, "table": cfg1_vals}
    variants = {
        "p1": dict(params=SolverParams(epochs=500, b=0.5, group_size=1, seed=1234,
                                       execution_mode="serial_faithful",
                                       sampling=SamplingConfig(alpha=0.25)),
                   snaps=(100, 101, 499)),
        "ser_g2": dict(params=SolverParams(epochs=20, b=0.5, group_size=2, seed=11,
                                           execution_mode="serial_faithful",
                                           sampling=SamplingConfig(alpha=1.0)),
                       snaps=(10, 11)),
        "par_full": dict(params=SolverParams(epochs=20, b=0.25, group_size=4, seed=12,
                                             execution_mode="parallel",
                                             sampling=SamplingConfig(alpha=1.0)),
                         snaps=(10, 11)),
        "par_mixed": dict(params=SolverParams(
            epochs=20, b=0.3, group_size=1, seed=13, execution_mode="parallel",
            sampling=SamplingConfig(strategy="mixed", alpha=0.5, gamma=0.5, theta0=0.2,
                                    theta_step=0.1)), snaps=(10, 11)),
        "ser_random": dict(params=SolverParams(
            epochs=20, b=0.5, group_size=3, seed=14, execution_mode="serial_faithful",
            sampling=SamplingConfig(strategy="random", alpha=0.75)), snaps=(10, 11)),
    }
    for name, v in variants.items():
        res = run_and_record(system, y, v["params"], x_true=x_true, snap_epochs=v["snaps"])
        for k, val in res.items():
            runs[f"{name}_{k}"] = val
        print(name, "final snr", res["snr"][-1], "gap", res["gap"][-1])
    np.savez_compressed(os.path.join(HERE, "pb_cfg1_runs.npz"), **runs)

    # 4. the reference tests' own fan-beam systems
    def fan(n_views, det_px, dims, radius, splits=(2, 2), det_splits=2):
        grid = VolumeGrid(dims, (1.0, 1.0))
        det = DetectorModel(det_px, 1.5)
        geo = ScanGeometry(grid, det, make_circular_trajectory(n_views, radius))
        part = make_partition(geo, splits, det_splits)
        table = build_probability_table(geo, part)
        return BlockSystem.build(geo, part, table=table, cache="always"), grid

    s12, g12 = fan(10, 14, (12, 12), 20.0)
    xt = head_phantom(g12)
    y12 = s12.forward(xt)
    x, tr = run_gcsgd(s12, y12, SolverParams(epochs=30, b=6.0, seed=3), x_true=xt)
    assert abs(tr.rows[-1].snr_db - 6.416697928678968) < 1e-9
    out = export_system(s12)
    out.update(x_true=xt, y=y12, final_x=x, snr=np.array([r.snr_db for r in tr.rows]))
    np.savez_compressed(os.path.join(HERE, "fan12.npz"), **out)

    s10, g10 = fan(8, 12, (10, 10), 18.0)
    xt = head_phantom(g10)
    y10 = s10.forward(xt)
    out = export_system(s10)
    out.update(x_true=xt, y=y10)
    for gs in (1, 3):
        for mode in ("serial_faithful", "parallel"):
            params = SolverParams(epochs=4, b=6.0, group_size=gs, seed=17, execution_mode=mode,
                                  sampling=SamplingConfig(alpha=0.5))
            rec = {}
            x, tr = run_gcsgd(s10, y10, params, x_true=xt, plan_record=rec)
            out[f"x_{gs}_{mode}"] = x
            out[f"plans_{gs}_{mode}"] = flatten_plans(rec)
    np.savez_compressed(os.path.join(HERE, "fan10.npz"), **out)

    # executor-level fixture (test_executor.py:14-23)
    grid = VolumeGrid((10, 10), (1.0, 1.0))
    det = DetectorModel(12, 1.5)
    geo = ScanGeometry(grid, det, make_circular_trajectory(8, 18.0))
    part = make_partition(geo, (2, 2), 2)
    table = build_probability_table(geo, part)
    se = BlockSystem.build(geo, part, table=table, cache="always")
    x0 = 0.3 + 0.1 * head_phantom(grid)
    ye = se.forward(head_phantom(grid) + 0.5)
    out = export_system(se)
    out.update(x0=x0, y=ye)
    plans = {
        "barrier": [(0, [(np.array([2, 3]), 0.7)]), (1, [(np.array([2, 3]), 0.7)])],
        "workers": [(0, [(np.array([0, 5]), 0.8), (np.array([2, 7]), 0.6)]),
                    (1, [(np.array([1, 4, 6]), 0.5)]), (3, [(np.array([3]), 0.9)])],
        "mutate": [(0, [(np.array([0, 5]), 0.8)]), (2, [(np.array([3]), 0.5)])],
    }
    for name, loops in plans.items():
        for mode in ("serial_faithful", "parallel"):
            st = SolverState.initialize(se, ye, x0=x0)
            stats = ref_executor.EpochExecutor(mode, 1).run_epoch(1, loops, st, se)
            out[f"{name}_{mode}_xhat"] = st.xhat.copy()
            out[f"{name}_{mode}_r"] = st.r.copy()
            out[f"{name}_{mode}_z"] = np.concatenate(st.z).copy()
            out[f"{name}_{mode}_counts"] = st.counts.copy()
            out[f"{name}_{mode}_stats"] = np.array([stats.n_tasks, stats.n_loops,
                                                    stats.bytes_moved, stats.n_degenerate])
            ref_solvers._commit_epoch(st, se)
            out[f"{name}_{mode}_x"] = st.x.copy()
    np.savez_compressed(os.path.join(HERE, "exec10.npz"), **out)
    print("done")


if __name__ == "__main__":
    main()
