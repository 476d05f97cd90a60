"""Parallel-beam problem description: the BASELINE.json configurations.

The reference package has no parallel-beam geometry and no random-ellipse
phantom (SURVEY §0 finding 3).  Its ray/voxel weights come from the tracer at
``projector.py:51-198``, which this build runs on the device
(``csrc/builder.cu``) for the geometry restated here, following the harness in
SURVEY §8c:

* ``VolumeGrid((n, n), (1, 1))`` -- origin ``(-n/2, -n/2, -1/2)``, unit voxels,
  flat voxel id ``ix*n + iy`` (``geometry.py:42-94``).
* View ``a`` has ``theta_a = pi*a/views``; bin ``k`` sits at
  ``u_k = k - (bins-1)/2``; the ray runs from ``u*e_u - 4n*d`` to
  ``u*e_u + 4n*d`` with ``d = (cos, sin, 0)``, ``e_u = (-sin, cos, 0)``.
  Measurement id is ``a*bins + k``.
* Row blocks are contiguous angle groups with edges
  ``round(linspace(0, views, m+1))``; column blocks are horizontal strips of
  ``ceil(n/nc)`` image rows (``geometry.py:356-378``), so every x_J is a
  contiguous slice.
* The block-density table is ``nnz(A_ij) / (|I_i| |J_j|)``.

Per-view (cos, sin) are computed on the host with numpy so the device tracer
and the CPU oracle see bit-identical ray endpoints.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError
from .validation import check_count


@dataclass(frozen=True)
class ParallelBeamSpec:
    """Image side ``n``, ``views`` angles in [0, pi), ``bins`` detector bins,
    ``m`` row blocks (angle groups) by ``nc`` column blocks (strips)."""

    n: int
    views: int
    bins: int
    m: int
    nc: int

    def __post_init__(self):
        for name in ("n", "views", "bins", "m", "nc"):
            check_count(name, getattr(self, name))
        if self.m > self.views:
            raise ConfigurationError("more row blocks than views")
        if self.nc > self.n:
            raise ConfigurationError("more column blocks than image rows")

    @property
    def n_measurements(self):
        return self.views * self.bins

    @property
    def n_voxels(self):
        return self.n * self.n

    def trig(self):
        theta = np.pi * np.arange(self.views) / self.views
        return np.cos(theta), np.sin(theta)

    def angle_edges(self):
        return np.round(np.linspace(0, self.views, self.m + 1)).astype(np.int64)

    def strip_edges(self):
        base = -(-self.n // self.nc)
        edges = [min(i * base, self.n) for i in range(self.nc)] + [self.n]
        if any(edges[i] >= edges[i + 1] for i in range(self.nc)):
            raise ConfigurationError(f"{self.nc} strips leave an empty block for n={self.n}")
        return np.array(edges, dtype=np.int64)

    def row_meas(self):
        e = self.angle_edges() * self.bins
        return [np.arange(e[i], e[i + 1], dtype=np.int64) for i in range(self.m)]

    def voxel_indices(self):
        e = self.strip_edges() * self.n
        return [np.arange(e[j], e[j + 1], dtype=np.int64) for j in range(self.nc)]


@dataclass(frozen=True)
class ProblemConfig:
    """One BASELINE.json configuration: geometry, phantom, noise and run knobs."""

    name: str
    spec: ParallelBeamSpec
    n_ellipses: int
    noise_frac: float
    dtype: str              # value storage: "f64" or "f32"
    mode: str               # execution_mode
    group_size: int
    alpha: float
    gamma: float
    b: float
    epochs: int
    phantom_seed: int = 0
    noise_seed: int = 1
    solver_seed: int = 1234


# BASELINE.json configs[0..4]; b values from SURVEY §8(d) (BASELINE leaves b unset).
CONFIGS = {
    1: ProblemConfig("cfg1-64", ParallelBeamSpec(64, 90, 92, 4, 4), 10, 0.01, "f64",
                     "serial_faithful", 1, 0.25, 1.0, 0.5, 500),
    2: ProblemConfig("cfg2-256", ParallelBeamSpec(256, 180, 367, 8, 8), 15, 0.01, "f64",
                     "serial_faithful", 8, 1.0, 1.0, 0.5, 625),
    3: ProblemConfig("cfg3-512", ParallelBeamSpec(512, 360, 725, 16, 16), 20, 0.005, "f32",
                     "parallel", 16, 1.0, 1.0, 1.0 / 16, 50),
    4: ProblemConfig("cfg4-1024", ParallelBeamSpec(1024, 720, 1449, 32, 32), 30, 0.005, "f32",
                     "parallel", 64, 1.0, 1.0, 1.0 / 32, 20),
    5: ProblemConfig("cfg5-2048", ParallelBeamSpec(2048, 1440, 2897, 64, 64), 40, 0.005,
                     "f32", "parallel", 128, 1.0, 1.0, 1.0 / 64, 10),
}


def random_ellipses(n, k, seed):
    """Sum of ``k`` random ellipses on the n x n grid (flat id ix*n + iy).

    Draw order per ellipse from ``default_rng(seed)``: centre radius
    0.8*sqrt(U), centre angle U[0, 2pi), semi-axes U[0.05, 0.4] twice,
    rotation U[0, pi), intensity U[0.1, 1.0].  Voxel centres in the
    normalised [-1, 1] frame; intensities add where ellipses overlap.
    """
    rng = np.random.default_rng(seed)
    c = (np.arange(n) + 0.5) / n * 2.0 - 1.0
    px = c[:, None]
    py = c[None, :]
    vol = np.zeros((n, n))
    for _ in range(k):
        rad = 0.8 * math.sqrt(rng.uniform())
        ang = rng.uniform(0.0, 2.0 * math.pi)
        cx, cy = rad * math.cos(ang), rad * math.sin(ang)
        a = rng.uniform(0.05, 0.4)
        b = rng.uniform(0.05, 0.4)
        phi = rng.uniform(0.0, math.pi)
        inten = rng.uniform(0.1, 1.0)
        du, dv = px - cx, py - cy
        xr = math.cos(phi) * du + math.sin(phi) * dv
        yr = -math.sin(phi) * du + math.cos(phi) * dv
        vol[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += inten
    return vol.ravel()


def add_noise(y_clean, frac, seed):
    """y = y_clean + N(0, sigma) with sigma = frac * mean(y_clean), drawn as
    ``default_rng(seed).normal(0, sigma, size)`` (phantoms.py:169-170)."""
    sigma = frac * float(np.mean(y_clean))
    rng = np.random.default_rng(seed)
    return y_clean + rng.normal(0.0, sigma, size=y_clean.size), sigma
