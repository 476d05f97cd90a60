"""Profiling helper: host cost of submit/wait per epoch in the device loop.

    python tools/submit_profile.py [--config 3] [--epochs 30]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig  # noqa
from paper_1709_00953_b200 import _native as N  # noqa
from paper_1709_00953_b200.executor import pack_loops, submit, wait  # noqa
from paper_1709_00953_b200.geometry import add_noise, random_ellipses  # noqa
from paper_1709_00953_b200.sampling import BlockScheduler  # noqa
from paper_1709_00953_b200.solvers import SolverState, _loops  # noqa


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--epochs", type=int, default=30)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    SolverState.initialize(s, y)
    sch = BlockScheduler(s.table, SamplingConfig(alpha=cfg.alpha), cfg.group_size)
    rng = np.random.default_rng(5)
    plans = [pack_loops(_loops(sch.epoch_plan(e + 1, rng), s.table, cfg.b), s)
             for e in range(a.epochs)]
    flags = N.BCT_COMMIT | N.BCT_METRICS
    ts, tw, km = [], [], []
    t0 = time.perf_counter()
    submit(s, cfg.mode, plans[0], flags)
    for e in range(a.epochs):
        t = time.perf_counter()
        if e + 1 < a.epochs:
            submit(s, cfg.mode, plans[e + 1], flags)
        t1 = time.perf_counter()
        res = wait(s, plans[e].task_j.size)[0]
        t2 = time.perf_counter()
        ts.append(t1 - t)
        tw.append(t2 - t1)
        km.append(res.kernel_ms)
    tot = time.perf_counter() - t0
    print(f"config {a.config}: {tot / a.epochs * 1e3:.3f} ms/epoch wall, kernel {np.mean(km):.3f} ms, "
          f"submit {np.mean(ts) * 1e3:.3f} ms (max {np.max(ts) * 1e3:.3f}), "
          f"wait {np.mean(tw) * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
