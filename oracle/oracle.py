"""CPU ORACLE -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU baseline.  The product package never imports it.

A numpy restatement of the reference solver's host logic around the C
restatement of its numba kernels (blockct_oracle.c):

* ``OracleSystem``          <- projector.py:507-793 (cached BlockSystem layout:
                               per-panel CSR over hit rows, rbp, l2g)
* ``oracle_epoch_plan``     <- sampling.py:63-157 (BlockScheduler.epoch_plan,
                               select_column_blocks, select_row_blocks, mixed)
* ``oracle_run_epoch``      <- executor.py:128-253 (EpochExecutor.run_epoch)
* ``oracle_commit_epoch``   <- solvers.py:180-185
* ``oracle_run_gcsgd``      <- solvers.py:188-269
* ``oracle_row_action`` / ``oracle_column_action`` <- solvers.py:303-379 (the
                               whole-system baselines, on ``OracleSystem.to_scipy``
                               <- projector.py:779-793)
* ``pb_trig`` / ``OracleSystem.parallel_beam`` <- the parallel-beam harness of
                               SURVEY §8c (reference tracer on strip panels).

Pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py) in tests/test_oracle_pins.py.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64


def lib():
    """Load (building if needed) the oracle C library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(_HERE, "libblockct_oracle.so")
    src = os.path.join(_HERE, "blockct_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", _HERE])
    L = ctypes.CDLL(path)
    L.oracle_trace_ray.restype = _i64
    L.oracle_trace_ray.argtypes = [_dp, _dp, _dp, _dp, _i64p, _i64p, _i64p, _dp]
    L.oracle_forward_rays.restype = _i64
    L.oracle_forward_rays.argtypes = [_i64, _dp, _dp, _dp, _dp, _i64p, _dp, _dp]
    L.oracle_trace_rays.restype = _i64
    L.oracle_trace_rays.argtypes = [_i64, _dp, _dp, _dp, _dp, _i64p, _i64p, _i64, _i64p, _dp,
                                    _i64p]
    L.oracle_pb_panel_counts.restype = None
    L.oracle_pb_panel_counts.argtypes = [_i64, _i64, _i64, _dp, _dp, _i64, _i64, _i64p]
    L.oracle_pb_panel_fill.restype = None
    L.oracle_pb_panel_fill.argtypes = [_i64, _i64, _i64, _dp, _dp, _i64, _i64, _i64p,
                                       _i64p, _i64, _dp, _i32p]
    L.oracle_run_tasks.restype = None
    L.oracle_run_tasks.argtypes = [_dp, _i32p, _i64p, _i64p, _i64p, _i64p, _i64p, _dp,
                                   _dp, _dp, _i64, _dp, _dp, _i64p, _dp, _i64p, _i64, _i64]
    L.oracle_run_tasks_threaded.restype = None
    L.oracle_run_tasks_threaded.argtypes = [_dp, _i32p, _i64p, _i64p, _i64p, _i64p, _i64p,
                                            _dp, _dp, _dp, _i64, _dp, _dp, _i64p, _dp,
                                            _i64p, _i64p, _i64]
    L.oracle_commit.restype = None
    L.oracle_commit.argtypes = [_dp, _i64p, _i64p, _i64, _dp]
    L.oracle_zsum.restype = None
    L.oracle_zsum.argtypes = [_dp, _i64p, _i64p, _i64p, _i64, _dp]
    L.oracle_csr_matvec.restype = None
    L.oracle_csr_matvec.argtypes = [_dp, _i32p, _i64p, _i64, _dp, _dp]
    L.oracle_csr_matvec_scatter.restype = None
    L.oracle_csr_matvec_scatter.argtypes = [_dp, _i32p, _i64p, _i64p, _i64, _dp, _dp]
    _LIB = L
    return L


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------------------
# parallel-beam geometry
# ---------------------------------------------------------------------------

def pb_trig(views):
    """Per-view (cos, sin) of theta_a = pi*a/views, computed with numpy."""
    theta = np.pi * np.arange(views) / views
    return np.cos(theta), np.sin(theta)


def pb_ray_endpoints(n, views, bins):
    """(src, dst) arrays of shape (views*bins, 3), the exact formula the C
    oracle (pb_ray) and the product's device tracer use."""
    c, s = pb_trig(views)
    u = np.arange(bins) - (bins - 1) / 2
    L = 4.0 * n
    cx = u[None, :] * (-s)[:, None]
    cy = u[None, :] * c[:, None]
    lc = (L * c)[:, None]
    ls = (L * s)[:, None]
    src = np.stack([(cx - lc).ravel(), (cy - ls).ravel(), np.zeros(views * bins)], 1)
    dst = np.stack([(cx + lc).ravel(), (cy + ls).ravel(), np.zeros(views * bins)], 1)
    return src, dst


def angle_block_edges(views, m):
    return np.round(np.linspace(0, views, m + 1)).astype(np.int64)


def strip_edges(n, nc):
    """Ceil-sized strips with the remainder in the last (geometry.py:356-378)."""
    base = -(-n // nc)
    return np.array([min(i * base, n) for i in range(nc)] + [n], dtype=np.int64)


# ---------------------------------------------------------------------------
# the cached blocked store (projector.py:507-793)
# ---------------------------------------------------------------------------

@dataclass
class OracleTable:
    values: np.ndarray
    totals: np.ndarray

    @property
    def active_cols(self):
        return np.flatnonzero(self.totals > 0.0)


@dataclass
class OracleSystem:
    data: list
    cols: list
    indptr: list
    rbp: list
    l2g: list
    row_meas: list          # per row block: global measurement ids
    vidx: list              # per column block: global voxel ids
    table: OracleTable
    n_measurements: int
    n_voxels: int

    @property
    def n_row_blocks(self):
        return len(self.row_meas)

    @property
    def n_col_blocks(self):
        return len(self.vidx)

    @property
    def row_sizes(self):
        return np.array([r.size for r in self.row_meas], dtype=np.int64)

    @property
    def col_sizes(self):
        return np.array([v.size for v in self.vidx], dtype=np.int64)

    @property
    def nnz(self):
        return int(sum(d.size for d in self.data))

    @classmethod
    def parallel_beam(cls, n, views, bins, m, nc, table="density", panels=None):
        """Trace the strip panels with the C restatement of the reference tracer.

        ``panels`` restricts tracing to a subset of column blocks (the others
        are left empty); used by the bounded CPU baseline sample.
        """
        L = lib()
        cosv, sinv = pb_trig(views)
        cosv, sinv = _c(cosv, np.float64), _c(sinv, np.float64)
        n_meas = views * bins
        aedges = angle_block_edges(views, m)
        row_meas = [np.arange(aedges[i] * bins, aedges[i + 1] * bins, dtype=np.int64)
                    for i in range(m)]
        xe = strip_edges(n, nc)
        vidx = [np.arange(xe[j] * n, xe[j + 1] * n, dtype=np.int64) for j in range(nc)]
        data, cols, indptr, rbp, l2g = [], [], [], [], []
        for j in range(nc):
            if panels is not None and j not in panels:
                data.append(np.empty(0)); cols.append(np.empty(0, np.int32))
                indptr.append(np.zeros(1, np.int64)); rbp.append(np.zeros(m + 1, np.int64))
                l2g.append(np.empty(0, np.int64))
                continue
            counts = np.empty(n_meas, dtype=np.int64)
            L.oracle_pb_panel_counts(n, views, bins, cosv, sinv, int(xe[j]), int(xe[j + 1]),
                                     counts)
            hit = np.flatnonzero(counts > 0).astype(np.int64)
            ip = np.zeros(hit.size + 1, dtype=np.int64)
            np.cumsum(counts[hit], out=ip[1:])
            d = np.empty(int(ip[-1]))
            cl = np.empty(int(ip[-1]), dtype=np.int32)
            L.oracle_pb_panel_fill(n, views, bins, cosv, sinv, int(xe[j]), int(xe[j + 1]),
                                   hit, ip, hit.size, d, cl)
            rb = np.searchsorted(hit, aedges * bins, side="left").astype(np.int64)
            data.append(d); cols.append(cl); indptr.append(ip); rbp.append(rb); l2g.append(hit)
        if table == "density":
            vals = np.zeros((m, nc))
            for j in range(nc):
                nnz_ij = np.diff(indptr[j][rbp[j]])
                vals[:, j] = nnz_ij / (np.array([r.size for r in row_meas]) * vidx[j].size)
        else:
            vals = np.asarray(table, dtype=np.float64)
        tab = OracleTable(vals, vals.sum(axis=0))
        return cls(data, cols, indptr, rbp, l2g, row_meas, vidx, tab, n_meas, n * n)

    @classmethod
    def scan(cls, geometry, partition, values):
        """_assemble (projector.py:563-626) for a general scan: every column
        block's rays traced per row block in order with the C restatement of
        _trace_ray_kernel (hit rows only, entries in the tracer's sorted
        order); pixel centres as geometry.py:227-240."""
        L = lib()
        g = geometry.grid
        origin = _c(g.origin, np.float64)
        vsize = _c(g.voxel_size, np.float64)
        per = geometry.detector.pixels_per_view
        centers = [oracle_pixel_centers(geometry, v) for v in range(geometry.n_views)]
        sources = np.array([p.source for p in geometry.poses], dtype=np.float64)
        m, nc = partition.n_row_blocks, partition.n_col_blocks
        ray_src, ray_dst = [], []
        for meas in partition.rows:
            meas = np.asarray(meas, dtype=np.int64)
            ray_src.append(_c(sources[meas // per], np.float64))
            ray_dst.append(_c(np.array([centers[int(v)][int(q)] for v, q in
                                        zip(meas // per, meas % per)]).reshape(-1, 3),
                              np.float64))
        data, cols, indptr, rbp, l2g = [], [], [], [], []
        for j in range(nc):
            lo = _c(partition.vol_lo[j], np.int64)
            hi = _c(partition.vol_hi[j], np.int64)
            cap = int((hi - lo).sum() + 3)
            d_parts, c_parts, counts_all, rows = [], [], [], []
            rb = np.zeros(m + 1, np.int64)
            for i, meas in enumerate(partition.rows):
                n = len(meas)
                idx = np.empty(n * cap, np.int64)
                lng = np.empty(n * cap)
                cnt = np.empty(n, np.int64)
                bad = L.oracle_trace_rays(n, ray_src[i], ray_dst[i], origin, vsize, lo, hi, cap,
                                          idx, lng, cnt)
                if bad >= 0:
                    raise ValueError("degenerate ray")
                hit = np.flatnonzero(cnt > 0)
                for q in hit:
                    k = int(cnt[q])
                    d_parts.append(lng[q * cap:q * cap + k])
                    c_parts.append(idx[q * cap:q * cap + k].astype(np.int32))
                    counts_all.append(k)
                rows.extend(int(v) for v in np.asarray(meas, np.int64)[hit])
                rb[i + 1] = rb[i] + hit.size
            ip = np.zeros(len(counts_all) + 1, np.int64)
            np.cumsum(counts_all, out=ip[1:])
            data.append(np.concatenate(d_parts) if d_parts else np.empty(0))
            cols.append(np.concatenate(c_parts) if c_parts else np.empty(0, np.int32))
            indptr.append(ip)
            rbp.append(rb)
            l2g.append(np.array(rows, np.int64))
        vals = np.asarray(values, dtype=np.float64)
        tab = OracleTable(vals, vals.sum(axis=0))
        return cls(data, cols, indptr, rbp, l2g, list(partition.rows), list(partition.vidx),
                   tab, geometry.n_measurements, g.n_voxels)

    def voxel_indices(self, j):
        return self.vidx[j]

    def measurement_rows(self, ids):
        if len(ids) == 0:
            return np.empty(0, dtype=np.int64)
        return np.concatenate([self.row_meas[i] for i in ids])

    def new_z_store(self):
        return [np.zeros(l.size) for l in self.l2g]

    def forward(self, x):
        x = _c(x, np.float64)
        out = np.zeros(self.n_measurements)
        for j in range(self.n_col_blocks):
            lib().oracle_csr_matvec_scatter(self.data[j], self.cols[j], self.indptr[j],
                                            self.l2g[j], self.l2g[j].size,
                                            _c(x[self.vidx[j]], np.float64), out)
        return out

    def fill_z_from_image(self, z, x):
        for j in range(self.n_col_blocks):
            out = np.empty(self.l2g[j].size)
            lib().oracle_csr_matvec(self.data[j], self.cols[j], self.indptr[j],
                                    self.l2g[j].size, _c(x[self.vidx[j]], np.float64), out)
            z[j][:] = out

    def projection_sum(self, z):
        out = np.zeros(self.n_measurements)
        for j in range(self.n_col_blocks):
            np.add.at(out, self.l2g[j], z[j])
        return out

    def accumulate_z_rows(self, z, ids, out):
        ids = _c(ids, np.int64)
        for j in range(self.n_col_blocks):
            lib().oracle_zsum(z[j], self.l2g[j], self.rbp[j], ids, ids.size, out)

    def to_scipy(self):
        """projector.py:779-793: COO of every panel -> CSR."""
        import scipy.sparse as sp
        rows, cols, vals = [], [], []
        for j in range(self.n_col_blocks):
            rows.append(np.repeat(self.l2g[j], np.diff(self.indptr[j])))
            cols.append(self.vidx[j][self.cols[j]])
            vals.append(self.data[j])
        mat = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                            shape=(self.n_measurements, self.n_voxels))
        return mat.tocsr()

    def dense(self):
        A = np.zeros((self.n_measurements, self.n_voxels))
        for j in range(self.n_col_blocks):
            rows = np.repeat(self.l2g[j], np.diff(self.indptr[j]))
            A[rows, self.vidx[j][self.cols[j]]] = self.data[j]
        return A


def oracle_pixel_centers(geometry, view):
    """ScanGeometry.pixel_centers (geometry.py:227-240): detector centre +
    u offset * det_u + v offset * det_v, the reference's numpy expression."""
    det = geometry.detector
    nu, nv = det.pixel_counts
    du, dv = det.pixel_spacing
    u = (np.arange(nu) - (nu - 1) / 2.0) * du
    v = (np.arange(nv) - (nv - 1) / 2.0) * dv
    uu, vv = np.meshgrid(u, v)
    off = np.column_stack([uu.ravel(), vv.ravel()])
    pose = geometry.poses[view]
    return (pose.detector_center[None, :] + off[:, 0:1] * pose.det_u[None, :]
            + off[:, 1:] * pose.det_v[None, :])


def oracle_forward_project(geometry, x):
    """forward_project (projector.py:348-371): y = A x with every ray traced
    through the whole grid (simulate_projections with noise 'none',
    phantoms.py:161-170)."""
    g = geometry.grid
    per = geometry.detector.pixels_per_view
    nv = geometry.n_views
    src = np.repeat(np.array([p.source for p in geometry.poses], dtype=np.float64), per, axis=0)
    dst = np.concatenate([oracle_pixel_centers(geometry, v) for v in range(nv)])
    out = np.empty(nv * per)
    bad = lib().oracle_forward_rays(nv * per, _c(src, np.float64), _c(dst, np.float64),
                                    _c(g.origin, np.float64), _c(g.voxel_size, np.float64),
                                    _c(g.dims, np.int64), _c(x, np.float64), out)
    if bad >= 0:
        raise ValueError(f"degenerate ray {bad}")
    return out


# ---------------------------------------------------------------------------
# sampler (sampling.py:63-157)
# ---------------------------------------------------------------------------

def oracle_mixed_weights(raw, theta):
    raw = np.asarray(raw, dtype=np.float64)
    out = np.zeros_like(raw)
    sc = raw > 0.0
    if not np.any(sc):
        return out
    top = raw[sc].max()
    out[sc] = raw[sc] + theta * (top - raw[sc])
    return out


def oracle_select_row_blocks(w, k, rng):
    w = np.asarray(w, dtype=np.float64)
    scope = np.flatnonzero(w > 0.0)
    keys = rng.exponential(size=scope.size)
    if k > scope.size:
        raise RuntimeError("cannot draw")
    if k == 0:
        return np.empty(0, dtype=np.int64)
    keys = keys / w[scope]
    return scope[np.argsort(keys, kind="stable")[:k]]


def oracle_epoch_plan(table, rng, alpha=1.0, gamma=1.0, group_size=1, strategy="importance",
                      theta=0.0):
    m = table.values.shape[0]
    active = table.active_cols
    k = math.ceil(gamma * active.size)
    target = math.ceil(alpha * m)
    plan = []
    for j in active[rng.choice(active.size, size=k, replace=False)]:
        raw = table.values[:, j]
        w = raw if strategy == "importance" else oracle_mixed_weights(raw, theta)
        scope_n = int(np.count_nonzero(w > 0.0))
        draws = min(group_size * math.ceil(target / group_size), scope_n)
        ids = oracle_select_row_blocks(w, draws, rng)
        plan.append((int(j), [ids[p:p + group_size] for p in range(0, ids.size, group_size)]))
    return plan


def oracle_group_beta(table, b, j, ids):
    return b * float(table.values[ids, j].sum()) / float(table.totals[j])


# ---------------------------------------------------------------------------
# executor and driver (executor.py:128-253, solvers.py:50-269)
# ---------------------------------------------------------------------------

@dataclass
class OracleState:
    x: np.ndarray
    y: np.ndarray
    r: np.ndarray
    z: list
    xhat: np.ndarray
    counts: np.ndarray
    epoch: int = 0

    @classmethod
    def initialize(cls, system, y, x0=None):
        y = _c(y, np.float64).copy()
        z = system.new_z_store()
        if x0 is None:
            x = np.zeros(system.n_voxels)
            r = y.copy()
        else:
            x = _c(x0, np.float64).copy()
            if np.any(x != 0.0):
                system.fill_z_from_image(z, x)
            r = y - system.projection_sum(z)
        return cls(x, y, r, z, np.zeros(system.n_voxels),
                   np.zeros(system.n_col_blocks, dtype=np.int64))

    def copy(self):
        return OracleState(self.x.copy(), self.y.copy(), self.r.copy(),
                           [z.copy() for z in self.z], self.xhat.copy(),
                           self.counts.copy(), self.epoch)


@dataclass
class OracleStats:
    n_tasks: int = 0
    n_loops: int = 0
    bytes_moved: int = 0
    n_degenerate: int = 0
    mus: list = field(default_factory=list)
    statuses: list = field(default_factory=list)


def _run_visit(system, j, groups, r, x_j, workers=1):
    ids = [_c(g, np.int64) for g, _ in groups]
    sel = np.concatenate(ids) if ids else np.empty(0, np.int64)
    sizes = np.array([g.size for g in ids], dtype=np.int64)
    gptr = np.zeros(sizes.size + 1, dtype=np.int64)
    np.cumsum(sizes, out=gptr[1:])
    betas = np.array([b for _, b in groups], dtype=np.float64)
    T = sizes.size
    rbp = system.rbp[j]
    row_counts = (rbp[1:] - rbp[:-1])[sel]
    task_rows = np.add.reduceat(row_counts, gptr[:-1]) if row_counts.size else np.zeros(T, np.int64)
    z_off = np.zeros(T + 1, dtype=np.int64)
    np.cumsum(task_rows, out=z_off[1:])
    x_news = np.empty((T, x_j.size))
    z_all = np.empty(int(z_off[-1]))
    mus = np.empty(T)
    st = np.zeros(T, dtype=np.int64)
    args = (system.data[j], system.cols[j], system.indptr[j], rbp, system.l2g[j], sel, gptr,
            betas, r, x_j, x_j.size, x_news, z_all, z_off, mus, st)
    if workers > 1 and T > 1:
        bounds = np.linspace(0, T, workers + 1).astype(np.int64)
        lib().oracle_run_tasks_threaded(*args, bounds, workers)
    else:
        lib().oracle_run_tasks(*args, 0, T)
    return dict(j=j, ids=ids, sel=sel, gptr=gptr, z_all=z_all, z_off=z_off,
                x_news=x_news, mus=mus, st=st, T=T)


def _commit_visit(system, state, run, stats):
    j = run["j"]
    for k in range(run["T"]):
        s = run["sel"][run["gptr"][k]:run["gptr"][k + 1]]
        lib().oracle_commit(state.z[j], system.rbp[j], _c(s, np.int64), s.size,
                            _c(run["z_all"][run["z_off"][k]:run["z_off"][k + 1]], np.float64))
    state.xhat[system.vidx[j]] += run["x_news"].sum(axis=0)
    state.counts[j] += run["T"]
    stats.n_tasks += run["T"]
    stats.n_degenerate += int(np.count_nonzero(run["st"]))
    stats.mus.extend(run["mus"].tolist())
    stats.statuses.extend(run["st"].tolist())
    pix = int(system.row_sizes[np.concatenate(run["ids"])].sum()) if run["ids"] else 0
    stats.bytes_moved += 16 * (pix + run["T"] * int(system.col_sizes[j]))


def _refresh(system, state, drawn):
    ids = np.unique(_c(drawn, np.int64))
    rows = system.measurement_rows(ids)
    if rows.size == 0:
        return
    acc = np.zeros(state.y.size)
    system.accumulate_z_rows(state.z, ids, acc)
    state.r[rows] = state.y[rows] - acc[rows]


def oracle_run_epoch(system, state, loops, mode="serial_faithful", workers=1):
    """EpochExecutor.run_epoch restated; loops = [(j, [(ids, beta), ...]), ...]."""
    stats = OracleStats(n_loops=len(loops))
    snaps = {}
    for j, _ in loops:
        if j not in snaps:
            snaps[j] = np.ascontiguousarray(state.x[system.vidx[j]])
    if mode == "serial_faithful":
        for j, groups in loops:
            run = _run_visit(system, j, groups, state.r, snaps[j], workers)
            _commit_visit(system, state, run, stats)
            _refresh(system, state, run["sel"])
    else:
        # parallel mode: every visit reads the epoch-start r and its own x_J
        # snapshot, so the visits fan out over threads (executor.py:194-198
        # fans the runs over worker_count threads the same way; the C kernel
        # runs without the GIL).  Commits stay in plan order below.
        if workers > 1 and len(loops) > 1:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(workers) as pool:
                runs = list(pool.map(lambda jg: _run_visit(system, jg[0], jg[1], state.r,
                                                           snaps[jg[0]], 1), loops))
        else:
            runs = [_run_visit(system, j, groups, state.r, snaps[j], workers)
                    for j, groups in loops]
        for run in runs:
            _commit_visit(system, state, run, stats)
        if runs:
            _refresh(system, state, np.concatenate([run["sel"] for run in runs]))
    return stats


def oracle_commit_epoch(state, system):
    for j in np.flatnonzero(state.counts):
        v = system.vidx[j]
        state.x[v] = state.xhat[v] / state.counts[j]
        state.xhat[v] = 0.0
    state.counts[:] = 0


def _snr(ref, est):
    ref_n = np.linalg.norm(ref)
    err = np.linalg.norm(ref - est)
    return math.inf if err == 0.0 else 20.0 * math.log10(ref_n / err)


def oracle_run_gcsgd(system, y, epochs, b, alpha=1.0, gamma=1.0, group_size=1,
                     mode="serial_faithful", seed=None, x_true=None, x0=None,
                     strategy="importance", theta0=0.0, theta_step=0.0, schedule=None,
                     plan_record=None, callback=None, workers=1, divergence_factor=1e6):
    """run_gcsgd restated (solvers.py:188-269).  Returns (x, rows) where each
    row is a dict(epoch, snr_db, obs_gap_db, n_tasks, bytes_moved, n_degenerate).
    Raises RuntimeError('diverged', last_good_epoch) on divergence."""
    state = OracleState.initialize(system, y, x0=x0)
    rng = np.random.default_rng(seed)
    theta = {"importance": 0.0, "random": 1.0}.get(strategy, theta0)
    rows = []
    y_scale = float(np.linalg.norm(state.y))
    ref_norm = None
    for epoch in range(1, epochs + 1):
        if schedule is not None:
            plan = [(j, [np.asarray(ids, np.int64)[p:p + group_size]
                         for p in range(0, len(ids), group_size)])
                    for j, ids in schedule[epoch]]
        else:
            plan = oracle_epoch_plan(system.table, rng, alpha, gamma, group_size, strategy,
                                     theta)
        if plan_record is not None:
            plan_record[epoch] = plan
        loops = [(j, [(ids, oracle_group_beta(system.table, b, j, ids)) for ids in groups])
                 for j, groups in plan]
        stats = oracle_run_epoch(system, state, loops, mode, workers)
        oracle_commit_epoch(state, system)
        if strategy == "mixed" and schedule is None:
            theta = min(1.0, theta + theta_step)
        state.epoch = epoch
        snr = _snr(x_true, state.x) if x_true is not None else math.nan
        gap = _snr(state.y, system.projection_sum(state.z)) if y_scale > 0 else math.nan
        row = dict(epoch=epoch, snr_db=snr, obs_gap_db=gap, n_tasks=stats.n_tasks,
                   bytes_moved=stats.bytes_moved, n_degenerate=stats.n_degenerate)
        rows.append(row)
        nx = float(np.linalg.norm(state.x))
        if ref_norm is None:
            ref_norm = max(nx, 1e-12)
        if not math.isfinite(nx) or nx > divergence_factor * ref_norm:
            raise RuntimeError("diverged", epoch - 1)
        if callback is not None:
            callback(epoch, state, row)
    return state.x.copy(), rows


# ---------------------------------------------------------------------------
# whole-system baselines (solvers.py:303-379)
# ---------------------------------------------------------------------------

def _safe_inverse(v):
    """solvers.py:303-308."""
    v = np.asarray(v, dtype=np.float64).ravel()
    out = np.zeros_like(v)
    nz = v > 0.0
    out[nz] = 1.0 / v[nz]
    return out


def _scaling(sub, rule, axis):
    if rule == "identity":
        return np.ones(sub.shape[1 - axis])
    if rule == "sum_inverse":
        return _safe_inverse(np.asarray(sub.sum(axis=axis)))
    return _safe_inverse(np.asarray(sub.multiply(sub).sum(axis=axis)))


def oracle_row_action(system, y, epochs, omega, m_rule="norm_inverse"):
    """solvers.py:317-346: per row block in partition order,
    x += omega * A_I^T (M (y_I - A_I x)).  Returns x and the per-epoch A x."""
    A = system.to_scipy()
    blocks = []
    for meas in system.row_meas:
        A_i = A[meas]
        blocks.append((A_i, meas, _scaling(A_i, m_rule, 1)))
    x = np.zeros(system.n_voxels)
    est = []
    for _ in range(epochs):
        for A_i, meas, m_diag in blocks:
            res = y[meas] - A_i @ x
            x += omega * (A_i.T @ (m_diag * res))
        est.append(A @ x)
    return x, est


def oracle_column_action(system, y, epochs, omega, m_rule="norm_inverse"):
    """solvers.py:349-379: per column block in partition order,
    dx = omega * (D (A_J^T r)); x_J += dx; r -= A_J dx.  Returns x and r."""
    A = system.to_scipy().tocsc()
    blocks = []
    for vox in system.vidx:
        A_j = A[:, vox]
        blocks.append((A_j, vox, _scaling(A_j, m_rule, 0)))
    x = np.zeros(system.n_voxels)
    r = np.asarray(y, dtype=np.float64).copy()
    for _ in range(epochs):
        for A_j, vox, d_diag in blocks:
            dx = omega * (d_diag * (A_j.T @ r))
            x[vox] += dx
            r -= A_j @ dx
    return x, r
