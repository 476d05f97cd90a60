"""Device-resident blocked operator: the B200 counterpart of the reference's
cached ``BlockSystem`` (projector.py:507-793).

A ``DeviceBlockSystem`` wraps one ``bct_ctx``: per-panel forward CSR and
panel CSC in HBM, the z store, x / xhat in panel-major order, y / r, and the
inverse row map used by the residual refresh.  It exposes the attributes the
reference solver and executor read (``table``, ``row_sizes``, ``col_sizes``,
``n_measurements``, ``n_voxels``, ``voxel_indices``, ``measurement_rows``,
``forward``, ``projection_sum``, ``nnz``, ``mode``) and owns exactly one live
solver state (``SolverState`` is a view of it).

Construction:
* ``from_panels`` -- the reference's panel arrays (data, cols, indptr, rbp, l2g)
  plus the partition and table, uploaded through ``bct_create``;
* ``from_reference`` -- the same, read off a reference ``BlockSystem`` object;
* ``parallel_beam`` -- traced on the device (``bct_create_parallel_beam``) for
  the BASELINE geometry;
* ``scan`` -- any fan / cone-beam ``ScanGeometry`` (scan.py), traced on the
  device (``bct_create_scan``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ConfigurationError, GeometryError
from .geometry import ParallelBeamSpec
from .sampling import ProbabilityTable


@dataclass(frozen=True)
class PanelArrays:
    data: np.ndarray
    cols: np.ndarray
    indptr: np.ndarray
    rbp: np.ndarray
    l2g: np.ndarray


def _dtype_code(dtype):
    if dtype in ("f64", "float64", np.float64):
        return N.BCT_F64
    if dtype in ("f32", "float32", np.float32):
        return N.BCT_F32
    raise ConfigurationError(f"dtype must be f64 or f32, got {dtype!r}")


class DeviceBlockSystem:
    mode = "cached"

    def __init__(self, ctx, row_meas, vidx, table, n_meas, n_vox, dtype, panel_range, device):
        self._ctx = ctypes.c_void_p(ctx)
        self._row_meas = [np.asarray(r, dtype=np.int64) for r in row_meas]
        self._vidx = [np.asarray(v, dtype=np.int64) for v in vidx]
        self.table = table
        self.n_measurements = int(n_meas)
        self.n_voxels = int(n_vox)
        self.dtype = dtype
        self.device = device
        self.panel_begin, self.panel_end = panel_range
        self.row_sizes = np.array([r.size for r in self._row_meas], dtype=np.int64)
        self.col_sizes = np.array([v.size for v in self._vidx], dtype=np.int64)
        info = np.zeros(8, dtype=np.int64)
        N.check(N.load().bct_info(self._ctx, N.ptr(info)), self._ctx, "bct_info")
        self.nnz = int(info[6])
        self.z_len = int(info[7])
        self._n_rows = {}
        self._nnz = {}
        for j in range(self.panel_begin, self.panel_end):
            nr = ctypes.c_int64()
            nz = ctypes.c_int64()
            N.check(N.load().bct_panel_info(self._ctx, j, ctypes.byref(nr), ctypes.byref(nz),
                                            None), self._ctx, "bct_panel_info")
            self._n_rows[j] = nr.value
            self._nnz[j] = nz.value

    # -- construction -------------------------------------------------------

    @classmethod
    def from_panels(cls, panels, row_meas, vidx, table_values, n_meas, n_vox, dtype="f64",
                    device=0, panel_range=None):
        L = N.load()
        m = len(row_meas)
        nc = len(vidx)
        pb, pe = panel_range if panel_range is not None else (0, nc)
        vals = N.f64(table_values)
        if vals.shape != (m, nc):
            raise ConfigurationError(f"table shape {vals.shape} != ({m}, {nc})")
        totals = N.f64(vals.sum(axis=0))
        rb_ptr = np.zeros(m + 1, dtype=np.int64)
        np.cumsum([len(r) for r in row_meas], out=rb_ptr[1:])
        rb_rows = N.i64(np.concatenate(row_meas) if m else np.empty(0))
        cb_ptr = np.zeros(nc + 1, dtype=np.int64)
        np.cumsum([len(v) for v in vidx], out=cb_ptr[1:])
        cb_vox = N.i64(np.concatenate(vidx))
        keep = []
        arr = (N.Panel * (pe - pb))()
        for lp, j in enumerate(range(pb, pe)):
            p = panels[j]
            d, c, ip, rb, lg = (N.f64(p.data), N.i32(p.cols), N.i64(p.indptr), N.i64(p.rbp),
                                N.i64(p.l2g))
            keep.append((d, c, ip, rb, lg))
            arr[lp] = N.Panel(lg.size, d.size, N.ptr(d), N.ptr(c), N.ptr(ip), N.ptr(rb),
                              N.ptr(lg))
        desc = N.SystemDesc(m, nc, int(n_meas), int(n_vox), N.ptr(rb_ptr), N.ptr(rb_rows),
                            N.ptr(cb_ptr), N.ptr(cb_vox), N.ptr(vals), N.ptr(totals), pb, pe,
                            _dtype_code(dtype), device)
        out = ctypes.c_void_p()
        N.check(L.bct_create(ctypes.byref(desc), arr, ctypes.byref(out)), None, "bct_create")
        return cls(out.value, row_meas, vidx, ProbabilityTable(vals, totals), n_meas, n_vox,
                   dtype, (pb, pe), device)

    @classmethod
    def from_reference(cls, ref_system, dtype="f64", device=0, panel_range=None):
        """Upload a reference cached BlockSystem (duck-typed)."""
        nc = ref_system.partition.n_col_blocks
        panels = [PanelArrays(ref_system._data[j], ref_system._cols[j], ref_system._indptr[j],
                              ref_system._rbp[j], ref_system._l2g[j]) for j in range(nc)]
        row_meas = [rb.measurement_indices for rb in ref_system.partition.row_blocks]
        vidx = [ref_system.voxel_indices(j) for j in range(nc)]
        return cls.from_panels(panels, row_meas, vidx, ref_system.table.values,
                               ref_system.n_measurements, ref_system.n_voxels, dtype, device,
                               panel_range)

    @classmethod
    def parallel_beam(cls, spec: ParallelBeamSpec, dtype="f64", device=0, panel_range=None):
        """Trace the strip panels of the BASELINE geometry on the device."""
        L = N.load()
        pb, pe = panel_range if panel_range is not None else (0, spec.nc)
        cosv, sinv = (N.f64(a) for a in spec.trig())
        desc = N.PBDesc(spec.n, spec.views, spec.bins, spec.m, spec.nc, N.ptr(cosv),
                        N.ptr(sinv), pb, pe, _dtype_code(dtype), device)
        out = ctypes.c_void_p()
        N.check(L.bct_create_parallel_beam(ctypes.byref(desc), ctypes.byref(out)), None,
                "bct_create_parallel_beam")
        vals = np.zeros((spec.m, spec.nc))
        totals = np.zeros(spec.nc)
        N.check(L.bct_get_table(ctypes.c_void_p(out.value), N.ptr(vals), N.ptr(totals)))
        return cls(out.value, spec.row_meas(), spec.voxel_indices(),
                   ProbabilityTable(vals, totals), spec.n_measurements, spec.n_voxels, dtype,
                   (pb, pe), device)

    @classmethod
    def scan(cls, geometry, partition=None, volume_splits=None, detector_splits=None,
             table=None, dtype="f64", device=0, panel_range=None):
        """BlockSystem.build(geometry, partition, table) for any ScanGeometry
        (scan.py): the partition and the silhouette table on the host, the
        blocked store traced on the device (bct_create_scan)."""
        from . import scan as S
        L = N.load()
        if partition is None:
            if volume_splits is None or detector_splits is None:
                raise ConfigurationError("need a partition or volume/detector splits")
            partition = S.make_partition(geometry, volume_splits, detector_splits)
        if table is None:
            vals, totals = S.probability_table(geometry, partition)
        else:
            vals = N.f64(table.values)
            totals = N.f64(table.totals)
        m, nc = partition.n_row_blocks, partition.n_col_blocks
        vals = N.f64(vals)
        totals = N.f64(totals)
        pb, pe = panel_range if panel_range is not None else (0, nc)
        g, det = geometry.grid, geometry.detector
        poses = N.f64(np.concatenate([np.concatenate([p.source, p.detector_center, p.det_u,
                                                      p.det_v]) for p in geometry.poses]))
        rb_ptr = np.zeros(m + 1, dtype=np.int64)
        np.cumsum([r.size for r in partition.rows], out=rb_ptr[1:])
        rb_rows = N.i64(np.concatenate(partition.rows))
        lo, hi = N.i64(partition.vol_lo), N.i64(partition.vol_hi)
        desc = N.ScanDesc((ctypes.c_int64 * 3)(*g.dims), (ctypes.c_double * 3)(*g.voxel_size),
                          (ctypes.c_double * 3)(*g.origin), det.pixel_counts[0],
                          det.pixel_counts[1], det.pixel_spacing[0], det.pixel_spacing[1],
                          geometry.n_views, N.ptr(poses), m, nc, N.ptr(rb_ptr), N.ptr(rb_rows),
                          N.ptr(lo), N.ptr(hi), N.ptr(vals), N.ptr(totals), pb, pe,
                          _dtype_code(dtype), device)
        out = ctypes.c_void_p()
        code = L.bct_create_scan(ctypes.byref(desc), ctypes.byref(out))
        if code == N.BCT_EINVAL:
            msg = L.bct_last_error(None).decode(errors="replace")
            if "inside" in msg or "degenerate" in msg:
                raise GeometryError(f"bct_create_scan: {msg}")
        N.check(code, None, "bct_create_scan")
        return cls(out.value, partition.rows, partition.vidx, ProbabilityTable(vals, totals),
                   geometry.n_measurements, g.n_voxels, dtype, (pb, pe), device)

    def close(self):
        if self._ctx is not None and self._ctx.value:
            N.load().bct_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- reference duck-type ---------------------------------------------------

    @property
    def ctx(self):
        return self._ctx

    @property
    def n_row_blocks(self):
        return len(self._row_meas)

    @property
    def n_col_blocks(self):
        return len(self._vidx)

    def voxel_indices(self, j):
        return self._vidx[j]

    def measurement_rows(self, i_ids):
        if len(i_ids) == 0:
            return np.empty(0, dtype=np.int64)
        return np.concatenate([self._row_meas[i] for i in i_ids])

    def n_local_rows(self, j):
        return self._n_rows[j]

    def _panel_nnz(self, j):
        return self._nnz[j]

    def x_len_owned(self):
        return int(sum(self.col_sizes[j] for j in range(self.panel_begin, self.panel_end)))

    def owns(self, j):
        return self.panel_begin <= j < self.panel_end

    def panel_l2g(self, j):
        """Global measurement id of each local row of panel j (no entry merge)."""
        L = N.load()
        lg = np.empty(self._n_rows[j], dtype=np.int64)
        N.check(L.bct_get_panel(self._ctx, j, None, None, None, None, N.ptr(lg)), self._ctx,
                "bct_get_panel")
        return lg

    def panel(self, j):
        """The panel's forward CSR as stored (f32 values are widened)."""
        nr = ctypes.c_int64()
        nz = ctypes.c_int64()
        L = N.load()
        N.check(L.bct_panel_info(self._ctx, j, ctypes.byref(nr), ctypes.byref(nz), None),
                self._ctx)
        d = np.empty(nz.value)
        c = np.empty(nz.value, dtype=np.int32)
        ip = np.empty(nr.value + 1, dtype=np.int64)
        rb = np.empty(self.n_row_blocks + 1, dtype=np.int64)
        lg = np.empty(nr.value, dtype=np.int64)
        N.check(L.bct_get_panel(self._ctx, j, N.ptr(d), N.ptr(c), N.ptr(ip), N.ptr(rb),
                                N.ptr(lg)), self._ctx, "bct_get_panel")
        return PanelArrays(d, c, ip, rb, lg)

    def forward(self, x):
        x = N.f64(x)
        if x.size != self.n_voxels:
            raise ConfigurationError(f"x has {x.size} entries, system has {self.n_voxels}")
        out = np.empty(self.n_measurements)
        N.check(N.load().bct_forward(self._ctx, N.ptr(x), N.ptr(out)), self._ctx, "forward")
        return out

    def projection_sum(self, z_store=None):
        """sum_j z^j from the device store (the argument is accepted for
        signature compatibility and must be None or this system's state)."""
        out = np.empty(self.n_measurements)
        N.check(N.load().bct_projection_sum(self._ctx, N.ptr(out)), self._ctx)
        return out

    def new_z_store(self):
        return [np.zeros(self._n_rows.get(j, 0)) for j in range(self.n_col_blocks)]

    # -- raw state access (used by SolverState) ---------------------------------

    def _get(self, fn, n):
        out = np.empty(n)
        N.check(fn(self._ctx, N.ptr(out)), self._ctx)
        return out

    def get_x(self):
        return self._get(N.load().bct_get_x, self.n_voxels)

    def get_xhat(self):
        return self._get(N.load().bct_get_xhat, self.n_voxels)

    def get_r(self):
        return self._get(N.load().bct_get_r, self.n_measurements)

    def get_z(self):
        out = []
        for j in range(self.n_col_blocks):
            if not self.owns(j):
                out.append(None)
                continue
            zj = np.empty(self._n_rows[j])
            N.check(N.load().bct_get_z(self._ctx, j, N.ptr(zj)), self._ctx)
            out.append(zj)
        return out

    def get_counts(self):
        out = np.zeros(self.n_col_blocks, dtype=np.int64)
        N.check(N.load().bct_get_counts(self._ctx, N.ptr(out)), self._ctx)
        return out

    def set_x(self, x):
        x = N.f64(x)
        N.check(N.load().bct_set_x(self._ctx, N.ptr(x)), self._ctx)

    def set_y(self, y):
        y = N.f64(y)
        N.check(N.load().bct_set_y(self._ctx, N.ptr(y)), self._ctx)

    def set_r(self, r):
        r = N.f64(r)
        N.check(N.load().bct_set_r(self._ctx, N.ptr(r)), self._ctx)

    def set_z(self, z):
        for j in range(self.n_col_blocks):
            if self.owns(j):
                zj = N.f64(z[j])
                if zj.size != self._n_rows[j]:
                    raise ConfigurationError(f"z[{j}] has {zj.size} rows, panel has "
                                             f"{self._n_rows[j]}")
                N.check(N.load().bct_set_z(self._ctx, j, N.ptr(zj)), self._ctx)

    def set_x_true(self, x_true):
        L = N.load()
        if x_true is None:
            N.check(L.bct_set_x_true(self._ctx, None), self._ctx)
        else:
            xt = N.f64(x_true)
            N.check(L.bct_set_x_true(self._ctx, N.ptr(xt)), self._ctx)

    def clear_state(self):
        """x = 0, z = 0, xhat = 0, counts = 0 on the device (no uploads)."""
        N.check(N.load().bct_clear_state(self._ctx), self._ctx)

    def reset_accumulators(self):
        N.check(N.load().bct_reset_accumulators(self._ctx), self._ctx)

    def fill_z_from_image(self, z_store=None, x=None):
        if x is not None:
            self.set_x(x)
        N.check(N.load().bct_fill_z_from_image(self._ctx), self._ctx)

    def reset_residual(self):
        N.check(N.load().bct_reset_residual(self._ctx), self._ctx)

    def commit_epoch(self):
        N.check(N.load().bct_commit_epoch(self._ctx), self._ctx)

    def audit_drift(self):
        d = ctypes.c_double()
        N.check(N.load().bct_audit(self._ctx, ctypes.byref(d)), self._ctx)
        return d.value

    def stream(self):
        s = ctypes.c_void_p()
        N.check(N.load().bct_get_stream(self._ctx, ctypes.byref(s)), self._ctx)
        return s.value
