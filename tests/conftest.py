import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def cfg1_runs():
    return golden("pb_cfg1_runs.npz")


def unflatten_plans(arr):
    """Inverse of make_golden.flatten_plans -> {epoch: [(j, ids), ...]}."""
    out = {}
    for row in arr:
        ep, j, k = int(row[0]), int(row[1]), int(row[2])
        out.setdefault(ep, []).append((j, row[3:3 + k].astype(np.int64)))
    return out


def fixture_system_arrays(npz):
    """(panels, row_meas, vidx, table, n_meas, n_vox) of an exported reference system."""
    from paper_1709_00953_b200.system import PanelArrays
    nc, m = int(npz["nc"]), int(npz["m"])
    panels = [PanelArrays(npz[f"data{j}"], npz[f"cols{j}"], npz[f"indptr{j}"], npz[f"rbp{j}"],
                          npz[f"l2g{j}"]) for j in range(nc)]
    rows = [npz[f"rows{i}"] for i in range(m)]
    vidx = [npz[f"vidx{j}"] for j in range(nc)]
    return panels, rows, vidx, npz["table"], int(npz["n_meas"]), int(npz["n_vox"])
