"""Profiling helper: wall time of run_gcsgd (public API, host buffers) with
pageable vs pinned host inputs, against the device-only epoch time.

    python tools/e2e_probe.py --config 3 [--epochs 20] [--reps 5]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, SamplingConfig, SolverParams,
                                       add_noise, random_ellipses, run_gcsgd)
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    y_h = torch.empty(y.size, dtype=torch.float64).pin_memory().numpy()
    xt_h = torch.empty(xt.size, dtype=torch.float64).pin_memory().numpy()
    y_h[:] = y
    xt_h[:] = xt
    p = SolverParams(epochs=a.epochs, b=cfg.b, group_size=cfg.group_size, execution_mode=cfg.mode,
                     seed=5, sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
    for name, (yy, xx) in (("pageable", (y, xt)), ("pinned", (y_h, xt_h))):
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            _, tr = run_gcsgd(s, yy, p, x_true=xx)
            ts.append(time.perf_counter() - t0)
        km = np.mean([r.kernel_ms for r in tr.rows])
        print(f"config {a.config} {name}: run_gcsgd {a.epochs} epochs: "
              f"{' '.join('%.2f' % (1e3 * t) for t in ts)} ms; kernel {km:.3f} ms/epoch")


if __name__ == "__main__" and not os.environ.get("PARTS"):
    main()


def parts():
    """Host-side pieces of run_gcsgd's set-up with pinned inputs."""
    import torch

    from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, add_noise, random_ellipses
    from paper_1709_00953_b200.solvers import SolverState
    cfg = CONFIGS[int(os.environ.get("CFG", "4"))]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    y_h = torch.empty(y.size, dtype=torch.float64).pin_memory().numpy()
    xt_h = torch.empty(xt.size, dtype=torch.float64).pin_memory().numpy()
    y_h[:] = y
    xt_h[:] = xt
    for name, fn in (("set_y pageable", lambda: s.set_y(y)), ("set_y pinned", lambda: s.set_y(y_h)),
                     ("set_x_true pageable", lambda: s.set_x_true(xt)),
                     ("set_x_true pinned", lambda: s.set_x_true(xt_h)),
                     ("initialize pinned", lambda: SolverState.initialize(s, y_h)),
                     ("get_x", lambda: s.get_x()),
                     ("norm y", lambda: np.linalg.norm(y_h))):
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            fn()
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{name:22s} {min(ts):.3f} ms")


if __name__ == "__main__" and os.environ.get("PARTS"):
    parts()
