"""Golden fixtures for the whole-system baselines, made by the
REFERENCE package itself in this container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_baselines.py

baselines.npz holds the reference's ``run_row_action`` (every m_rule) and
``run_column_action`` (every m_rule) outputs -- final x and the per-epoch SNR
and observation gap -- on the config-1 parallel-beam system (injected into a
cached BlockSystem exactly like make_golden.py) and on the reference tests'
12x12 fan-beam system (fan12.npz).  Nothing at test time reads
/root/reference.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (reference import + the config-1 harness)
from blockct import BaselineParams, run_column_action, run_row_action  # noqa: E402

from paper_1709_00953_b200.geometry import CONFIGS, add_noise, random_ellipses  # noqa: E402

RULES = ("identity", "sum_inverse", "norm_inverse")
# relaxation per (system, sweep, rule): stable choices (the reference tests'
# 0.9 on the fan-beam system; a 5-epoch scan elsewhere)
OMEGA = {"cfg1": {"row": {"identity": 1e-3, "sum_inverse": 0.03, "norm_inverse": 0.03},
                  "col": {"identity": 3e-4, "sum_inverse": 0.03, "norm_inverse": 0.03}},
         "fan12": {"row": {"identity": 0.05, "sum_inverse": 0.9, "norm_inverse": 0.9},
                   "col": {"identity": 0.02, "sum_inverse": 0.2, "norm_inverse": 0.2}}}


def runs(system, y, x_true, epochs, tag, out):
    for rule in RULES:
        for kind, fn in (("row", run_row_action), ("col", run_column_action)):
            p = BaselineParams(epochs=epochs, omega=OMEGA[tag][kind][rule], m_rule=rule)
            x, tr = fn(system, y, p, x_true=x_true)
            out[f"{tag}_{kind}_{rule}_x"] = x
            out[f"{tag}_{kind}_{rule}_snr"] = np.array([r.snr_db for r in tr.rows])
            out[f"{tag}_{kind}_{rule}_gap"] = np.array([r.obs_gap_db for r in tr.rows])
            print(tag, kind, rule, "snr", tr.rows[-1].snr_db)


def main():
    out = {f"{t}_omega_{k}": np.array([OMEGA[t][k][r] for r in RULES])
           for t in OMEGA for k in ("row", "col")}
    cfg = CONFIGS[1]
    panels = mg.ref_parallel_beam_panels(cfg.spec)
    vals = mg.density_table(cfg.spec, panels)
    system = mg.inject(cfg.spec, panels, vals)
    x_true = random_ellipses(64, cfg.n_ellipses, cfg.phantom_seed)
    y, _ = add_noise(system.forward(x_true), cfg.noise_frac, cfg.noise_seed)
    out["cfg1_y"] = y
    runs(system, y, x_true, 5, "cfg1", out)
    f12 = np.load(os.path.join(HERE, "fan12.npz"))
    s12, _ = mg_fan12()
    runs(s12, f12["y"], f12["x_true"], 5, "fan12", out)
    np.savez_compressed(os.path.join(HERE, "baselines.npz"), **out)
    print("done")


def mg_fan12():
    from blockct import (BlockSystem, DetectorModel, ScanGeometry, VolumeGrid,
                         build_probability_table, make_circular_trajectory, make_partition)
    grid = VolumeGrid((12, 12), (1.0, 1.0))
    det = DetectorModel(14, 1.5)
    geo = ScanGeometry(grid, det, make_circular_trajectory(10, 20.0))
    part = make_partition(geo, (2, 2), 2)
    table = build_probability_table(geo, part)
    return BlockSystem.build(geo, part, table=table, cache="always"), grid


if __name__ == "__main__":
    main()
