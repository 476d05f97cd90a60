"""General scan geometry (fan / cone beam) for device-built systems.

Restates the reference's geometry model (geometry.py:42-312, 320-529,
586-672) on the host: the voxel grid, the flat detector, circular and
arbitrary view poses, the cuboid volume partition, the per-view detector
partition and the silhouette-area probability table.  The system matrix
itself is traced on the device (``DeviceBlockSystem.scan`` ->
``bct_create_scan``, builder.cu) with the reference tracer's arithmetic
(projector.py:51-198), so the panels equal the reference's bit for bit.

The probability table uses the same numpy expressions and float operation
order as the reference, so it is bit-identical too (selection and betas
depend on it).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, GeometryError
from .validation import check_count, check_positive

_AXIS_TOL = 1e-9


class VolumeGrid:
    """Voxel grid: dims (2 or 3 ints; 2D pads to a 1-voxel z slab of the x
    size), voxel sizes, low-corner origin (default: centred)."""

    def __init__(self, dims, voxel_size, origin=None):
        dims = tuple(int(d) for d in np.atleast_1d(dims))
        sizes = tuple(float(s) for s in np.atleast_1d(voxel_size))
        if len(dims) not in (2, 3) or len(sizes) != len(dims):
            raise ConfigurationError("grid dims / voxel_size must have 2 or 3 matching entries")
        if any(d < 1 for d in dims) or any(not (s > 0 and math.isfinite(s)) for s in sizes):
            raise ConfigurationError("grid dims and voxel sizes must be positive")
        self.input_ndim = len(dims)
        if len(dims) == 2:
            dims = dims + (1,)
            sizes = sizes + (sizes[0],)
            if origin is not None:
                origin = tuple(float(o) for o in np.atleast_1d(origin)) + (-0.5 * sizes[2],)
        if origin is None:
            origin = tuple(-0.5 * d * s for d, s in zip(dims, sizes))
        self.dims = dims
        self.voxel_size = sizes
        self.origin = tuple(float(o) for o in origin)

    @property
    def n_voxels(self):
        return self.dims[0] * self.dims[1] * self.dims[2]


class DetectorModel:
    """Flat detector; pixel (iu, iv) of a view has flat index iv*nu + iu."""

    def __init__(self, pixel_counts, pixel_spacing):
        counts = tuple(int(c) for c in np.atleast_1d(pixel_counts))
        spacing = tuple(float(s) for s in np.atleast_1d(pixel_spacing))
        if len(counts) not in (1, 2) or len(spacing) != len(counts):
            raise ConfigurationError("detector counts / spacing must have 1 or 2 matching entries")
        if len(counts) == 1:
            counts = counts + (1,)
            spacing = spacing + (spacing[0],)
        self.pixel_counts = counts
        self.pixel_spacing = spacing

    @property
    def pixels_per_view(self):
        return self.pixel_counts[0] * self.pixel_counts[1]

    def rect_bounds(self, u0, u1, v0, v1):
        nu, nv = self.pixel_counts
        du, dv = self.pixel_spacing
        return ((u0 - nu / 2.0) * du, (u1 - nu / 2.0) * du,
                (v0 - nv / 2.0) * dv, (v1 - nv / 2.0) * dv)


@dataclass(frozen=True)
class ViewPose:
    source: np.ndarray
    detector_center: np.ndarray
    det_u: np.ndarray
    det_v: np.ndarray

    @property
    def normal(self):
        axis = self.detector_center - self.source
        return axis / np.linalg.norm(axis)


def circular_trajectory(n_views, radius, rotation_center=(0.0, 0.0, 0.0), angular_start=0.0):
    """Equiangular circle in z = 0: source at angle start + 2 pi k / n, detector
    opposite, det_u the in-plane tangent, det_v = +z."""
    n_views = check_count("n_views", n_views)
    radius = check_positive("radius", radius)
    center = np.ascontiguousarray(rotation_center, dtype=np.float64)
    poses = []
    for k in range(n_views):
        th = angular_start + 2.0 * math.pi * k / n_views
        c, s = math.cos(th), math.sin(th)
        poses.append(ViewPose(center + radius * np.array([c, s, 0.0]),
                              center - radius * np.array([c, s, 0.0]),
                              np.array([-s, c, 0.0]), np.array([0.0, 0.0, 1.0])))
    return poses


def random_sphere_trajectory(n_views, radius, source_detector_distance, seed):
    """Random sphere scan about the origin (geometry.py:283-312): per view
    a ~ U[0, pi], b ~ U[0, 2 pi) from ``default_rng(seed)`` (all a's drawn
    first, then all b's); source at radius * (sin a cos b, sin a sin b, cos a),
    detector centre ``source_detector_distance`` along the inward axis w,
    det_u = normalised (h x w) with h = +z unless |w_z| >= 0.9 (then +x),
    det_v = w x det_u.  Same numpy/math operations, so the poses (and the
    traced panels) are bit-identical to the reference's."""
    n_views = check_count("n_views", n_views)
    radius = check_positive("radius", radius)
    dist = check_positive("source_detector_distance", source_detector_distance)
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, math.pi, size=n_views)
    b = rng.uniform(0.0, 2.0 * math.pi, size=n_views)
    poses = []
    for k in range(n_views):
        sa, ca = math.sin(a[k]), math.cos(a[k])
        sb, cb = math.sin(b[k]), math.cos(b[k])
        src = radius * np.array([sa * cb, sa * sb, ca])
        w = -src / radius
        det = src + dist * w
        h = np.array([0.0, 0.0, 1.0]) if abs(w[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
        u = np.cross(h, w)
        u /= np.linalg.norm(u)
        poses.append(ViewPose(src, det, u, np.cross(w, u)))
    return poses


@dataclass(frozen=True)
class ScanGeometry:
    grid: VolumeGrid
    detector: DetectorModel
    poses: tuple

    @property
    def n_views(self):
        return len(self.poses)

    @property
    def n_measurements(self):
        return self.n_views * self.detector.pixels_per_view


def _edges(size, splits, what):
    """ceil-sized blocks, remainder in the last; an empty block is an error."""
    if splits > size:
        raise ConfigurationError(f"{what} split count {splits} exceeds size {size}")
    base = -(-size // splits)
    e = [min(i * base, size) for i in range(splits)] + [size]
    if any(e[i] >= e[i + 1] for i in range(splits)):
        raise ConfigurationError(f"{what} splits {splits} leave an empty block (size {size})")
    return e


@dataclass(frozen=True)
class ScanPartition:
    vol_lo: np.ndarray      # [n, 3] voxel index bounds of each column block
    vol_hi: np.ndarray
    vidx: list              # per column block: flat voxel ids (C order in the box)
    det_blocks: list        # per row block: (view, u0, u1, v0, v1)
    rows: list              # per row block: global measurement ids
    vsplit: tuple
    dsplit: tuple

    @property
    def n_row_blocks(self):
        return len(self.rows)

    @property
    def n_col_blocks(self):
        return len(self.vidx)


def make_partition(geometry, volume_splits, detector_splits):
    """Cuboid volume blocks in C order of the split grid (x slowest) and, per
    view, detector sub-rectangles (v split slower than u): geometry.py:366-464."""
    g = geometry.grid
    vs = tuple(check_count("volume split", s) for s in np.atleast_1d(volume_splits))
    if len(vs) == 2 and g.input_ndim == 2:
        vs = vs + (1,)
    if len(vs) != 3:
        raise ConfigurationError("volume splits must match the grid dims")
    ds = tuple(check_count("detector split", s) for s in np.atleast_1d(detector_splits))
    if len(ds) == 1:
        ds = ds + (1,)
    ve = [_edges(g.dims[a], vs[a], "volume") for a in range(3)]
    nx, ny, nz = g.dims
    lo, hi, vidx = [], [], []
    for bx in range(vs[0]):
        for by in range(vs[1]):
            for bz in range(vs[2]):
                l = (ve[0][bx], ve[1][by], ve[2][bz])
                h = (ve[0][bx + 1], ve[1][by + 1], ve[2][bz + 1])
                ix, iy, iz = (np.arange(l[a], h[a]) for a in range(3))
                vidx.append(((ix[:, None, None] * ny + iy[None, :, None]) * nz
                             + iz[None, None, :]).ravel().astype(np.int64))
                lo.append(l)
                hi.append(h)
    nu, nv = geometry.detector.pixel_counts
    ue = _edges(nu, ds[0], "detector")
    vve = _edges(nv, ds[1], "detector")
    per = geometry.detector.pixels_per_view
    det_blocks, rows = [], []
    for view in range(geometry.n_views):
        for sv in range(ds[1]):
            for su in range(ds[0]):
                iv = np.arange(vve[sv], vve[sv + 1])
                iu = np.arange(ue[su], ue[su + 1])
                rows.append((view * per + (iv[:, None] * nu + iu[None, :]).ravel()).astype(np.int64))
                det_blocks.append((view, ue[su], ue[su + 1], vve[sv], vve[sv + 1]))
    return ScanPartition(np.array(lo, np.int64), np.array(hi, np.int64), vidx, det_blocks, rows,
                         vs, ds)


# -- silhouette areas (geometry.py:472-672) ----------------------------------

def _hull(points):
    """Convex hull, monotone chain, counter-clockwise from the lowest point."""
    pts = sorted(set(map(tuple, points)))
    if len(pts) < 3:
        return pts

    def turn(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])

    chains = []
    for seq in (pts, pts[::-1]):
        ch = []
        for p in seq:
            while len(ch) >= 2 and turn(ch[-2], ch[-1], p) <= 0:
                ch.pop()
            ch.append(p)
        chains.append(ch[:-1])
    return chains[0] + chains[1]


def _clip(poly, axis, bound, below):
    """Sutherland-Hodgman against one axis-aligned half plane."""
    out = []
    n = len(poly)
    for k in range(n):
        a, b = poly[k], poly[(k + 1) % n]
        ain = a[axis] <= bound if below else a[axis] >= bound
        bin_ = b[axis] <= bound if below else b[axis] >= bound
        if ain:
            out.append(a)
        if ain != bin_:
            t = (bound - a[axis]) / (b[axis] - a[axis])
            out.append((a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1])))
    return out


def _area(poly):
    if len(poly) < 3:
        return 0.0
    acc = 0.0
    for k in range(len(poly)):
        (u0, v0), (u1, v1) = poly[k], poly[(k + 1) % len(poly)]
        acc += u0 * v1 - u1 * v0
    return abs(acc) / 2.0


def _corners(grid, lo, hi):
    o = np.asarray(grid.origin)
    s = np.asarray(grid.voxel_size)
    plo = o + np.asarray(lo) * s
    phi = o + np.asarray(hi) * s
    c = np.array([(x, y, z) for x in (plo[0], phi[0]) for y in (plo[1], phi[1])
                  for z in (plo[2], phi[2])], dtype=np.float64)
    return c, plo, phi


def _project(pose, corners):
    src, n = pose.source, pose.normal
    dplane = float(np.dot(n, pose.detector_center - src))
    rel = corners - src[None, :]
    depth = rel @ n
    eps = _AXIS_TOL * dplane
    if np.all(depth <= eps):
        return None
    if np.any(depth <= eps):
        raise GeometryError("volume block straddles the source plane; projection undefined")
    t = dplane / depth
    pts = src[None, :] + rel * t[:, None] - pose.detector_center[None, :]
    return np.column_stack([pts @ pose.det_u, pts @ pose.det_v])


def probability_table(geometry, partition):
    """values[i, j] = area of column block j's silhouette clipped to row block
    i's detector rectangle; totals = column sums."""
    m, n = partition.n_row_blocks, partition.n_col_blocks
    values = np.zeros((m, n))
    by_view = {}
    for i, (view, u0, u1, v0, v1) in enumerate(partition.det_blocks):
        by_view.setdefault(view, []).append((i, u0, u1, v0, v1))
    for j in range(n):
        corners, plo, phi = _corners(geometry.grid, partition.vol_lo[j], partition.vol_hi[j])
        for view, blocks in by_view.items():
            pose = geometry.poses[view]
            if np.all(pose.source > plo) and np.all(pose.source < phi):
                raise GeometryError("source lies inside a volume block; projection undefined")
            uv = _project(pose, corners)
            if uv is None:
                continue
            hull = _hull(uv)
            if len(hull) < 3:
                continue
            for i, u0, u1, v0, v1 in blocks:
                ulo, uhi, vlo, vhi = geometry.detector.rect_bounds(u0, u1, v0, v1)
                poly = hull
                for axis, bound, below in ((0, ulo, False), (0, uhi, True), (1, vlo, False),
                                           (1, vhi, True)):
                    if not poly:
                        break
                    poly = _clip(poly, axis, bound, below)
                values[i, j] = _area(poly)
    return values, values.sum(axis=0)
