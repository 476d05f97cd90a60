"""Profiling helper: wall time of the whole-system baselines (row / column
action) per sweep on a BASELINE config.

    python tools/baseline_time.py [--config 3] [--epochs 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem  # noqa
from paper_1709_00953_b200.baselines import BaselineParams, run_column_action, run_row_action  # noqa
from paper_1709_00953_b200.geometry import add_noise, random_ellipses  # noqa


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--epochs", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype="f64")
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    for name, fn in (("row action", run_row_action), ("column action", run_column_action)):
        fn(s, y, BaselineParams(epochs=1, omega=1.0), x_true=xt)   # build + warm-up
        t0 = time.perf_counter()
        fn(s, y, BaselineParams(epochs=a.epochs, omega=1.0), x_true=xt)
        dt = (time.perf_counter() - t0) / a.epochs
        print(f"config {a.config} {name}: {1e3 * dt:.2f} ms per sweep (nnz {s.nnz:.3e})")


if __name__ == "__main__":
    main()
