"""Profiling helper: where the end-to-end run_gcsgd time goes (host timers).

    python tools/e2e_profile.py [--config 4] [--epochs 10] [--device-sampling]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, SamplingConfig, SolverParams,  # noqa
                                   add_noise, random_ellipses, run_gcsgd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--device-sampling", action="store_true")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    p = SolverParams(epochs=a.epochs, b=cfg.b, group_size=cfg.group_size,
                     execution_mode=cfg.mode, seed=5,
                     sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
    run_gcsgd(s, y, p, x_true=xt, device_sampling=a.device_sampling)   # warm
    t = time.perf_counter()
    x, tr = run_gcsgd(s, y, p, x_true=xt, device_sampling=a.device_sampling)
    dt = time.perf_counter() - t
    k = sum(r.kernel_ms for r in tr.rows)
    print(f"config {a.config}: e2e {dt * 1e3:.1f} ms for {a.epochs} epochs, kernel sum {k:.1f} ms")
    pr = cProfile.Profile()
    pr.enable()
    run_gcsgd(s, y, p, x_true=xt, device_sampling=a.device_sampling)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
