"""The reference's acceptance setups (tests/test_acceptance.py:37-53, 444-483)
rebuilt with this package's scan geometry, plus the fixtures
tests/golden/make_golden_acceptance.py wrote by running the reference."""

import hashlib
import json
import os

import numpy as np

from conftest import GOLDEN
from paper_1709_00953_b200 import SamplingConfig, SolverParams
from paper_1709_00953_b200 import scan as S


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fixtures():
    return (np.load(os.path.join(GOLDEN, "acceptance.npz")),
            json.load(open(os.path.join(GOLDEN, "acceptance_hashes.json"))))


def standard_geometry():
    """64^2 grid, 360 views on a radius-115 circle, 187-pixel detector; 2x2
    volume blocks, 2 detector blocks per view (720 row blocks)."""
    grid = S.VolumeGrid((64, 64), (1.0, 1.0))
    geo = S.ScanGeometry(grid, S.DetectorModel(187, 1.0), tuple(S.circular_trajectory(360, 115.0)))
    return geo, S.make_partition(geo, (2, 2), 2)


def a11_geometry():
    """32^3 grid (0.25 voxels), 90 random-sphere views (radius 16.5, source-
    detector 33, seed 5), 52x52 detector (0.5); 2x2x2 volume blocks, 2x2
    detector blocks (360 row blocks)."""
    grid = S.VolumeGrid((32, 32, 32), (0.25, 0.25, 0.25))
    poses = S.random_sphere_trajectory(90, 16.5, 33.0, 5)
    geo = S.ScanGeometry(grid, S.DetectorModel((52, 52), (0.5, 0.5)), tuple(poses))
    return geo, S.make_partition(geo, (2, 2, 2), (2, 2))


def params(epochs, b, gs, seed, mode="serial_faithful", alpha=1.0, audit=0, workers=1):
    """tests/test_acceptance.py:56-66 (_snr_trace's SolverParams)."""
    return SolverParams(epochs=epochs, b=b, group_size=gs, execution_mode=mode,
                        audit_interval=audit, seed=seed, worker_count=workers,
                        sampling=SamplingConfig(strategy="importance", alpha=alpha))


def panels_match(get, hashes):
    """``get(j)`` -> (data, cols, indptr, rbp, l2g); all five sha256 equal."""
    for j, h in enumerate(hashes):
        d, c, ip, rb, lg = get(j)
        if (sha(d), sha(c), sha(ip), sha(rb), sha(lg)) != (h["data"], h["cols"], h["indptr"],
                                                           h["rbp"], h["l2g"]):
            return False
    return True


def unflatten(arr):
    out = {}
    for row in arr:
        ep, j, k = int(row[0]), int(row[1]), int(row[2])
        out.setdefault(ep, []).append((j, row[3:3 + k].astype(np.int64)))
    return out
