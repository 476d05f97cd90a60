"""Profiling helper: is the batched epoch's per-CTA imbalance systematic?

    BCT_TIMELINE=1 python tools/balance_probe.py [--config 4] [--world 1] [--epochs 6]

Runs batched epochs, reads the timeline after each, and reports per CTA the
phase-A and phase-B durations, the SM it ran on, and how well a CTA's phase
time in one epoch predicts the next (correlation across epochs, by CTA and by
SM).  A systematic per-SM rate would make a measured-rate split pay."""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BCT_TIMELINE", "1")

from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig  # noqa
from paper_1709_00953_b200 import _native as N  # noqa
from paper_1709_00953_b200.executor import pack_loops, submit, wait  # noqa
from paper_1709_00953_b200.sampling import BlockScheduler  # noqa
from paper_1709_00953_b200.solvers import SolverState, _loops  # noqa
from paper_1709_00953_b200.geometry import random_ellipses, add_noise  # noqa


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=6)
    ap.add_argument("--world", type=int, default=1)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    pr = (0, cfg.spec.nc // a.world)
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype, panel_range=pr)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    SolverState.initialize(s, y)
    sch = BlockScheduler(s.table, SamplingConfig(alpha=cfg.alpha), cfg.group_size)
    rng = np.random.default_rng(5)
    A, B, C, SM, K = [], [], [], [], []
    for e in range(a.epochs):
        packed = pack_loops(_loops(sch.epoch_plan(e + 1, rng), s.table, cfg.b), s)
        submit(s, cfg.mode, packed,
               N.BCT_COMMIT | N.BCT_METRICS | (N.BCT_SHARDED if a.world > 1 else 0))
        res = wait(s, packed.task_j.size)[0]
        nt = packed.task_j.size
        grid = ctypes.c_int32()
        buf = np.zeros(8 * nt * 4096, dtype=np.int64)
        N.check(N.load().bct_debug_timeline(s.ctx, N.ptr(buf), nt, ctypes.byref(grid)), s.ctx)
        G = grid.value
        tl = buf[:nt * 8 * G].reshape(nt, 8, G)
        t = tl[0].astype(np.float64) / 1e3
        A.append(t[1] - t[0])
        B.append(t[3] - t[2])
        C.append(t[5] - t[4])
        SM.append(tl[3, 0].copy())
        K.append(res.kernel_ms)
    A, B, C, SM = map(np.array, (A, B, C, SM))
    print(f"config {a.config} world {a.world}: grid {G}, kernel ms per epoch "
          + " ".join(f"{k:.3f}" for k in K))
    same = all((SM[e] == SM[0]).all() for e in range(len(SM)))
    print("block -> SM mapping identical across epochs:", same)
    for name, D in (("A", A), ("B", B), ("C", C)):
        d = D[1:]   # skip the first epoch
        cors = [np.corrcoef(d[e], d[e + 1])[0, 1] for e in range(len(d) - 1)]
        # by SM: reorder each epoch's durations by SM id
        bysm = np.array([d[e][np.argsort(SM[e + 1])] for e in range(len(d))])
        cors_sm = [np.corrcoef(bysm[e], bysm[e + 1])[0, 1] for e in range(len(d) - 1)]
        mean = d.mean(axis=0)
        print(f"{name}: per-epoch max {d.max(axis=1).round(1)} mean {d.mean(axis=1).round(1)}; "
              f"epoch-to-epoch corr by CTA {np.round(cors, 2)} by SM {np.round(cors_sm, 2)}")
        print(f"   CTA-mean over epochs: min {mean.min():.1f} med {np.median(mean):.1f} "
              f"max {mean.max():.1f}; max/mean of the epoch mean {d.max(axis=1).mean() / d.mean():.3f}")
    print("SM ids (epoch 1):", " ".join(str(v) for v in SM[1][:40]), "...")
    bysm = B[1:][:, np.argsort(SM[1])].mean(axis=0)
    print("B by SM id (mean over epochs):", " ".join(f"{v:.0f}" for v in bysm))
    abysm = A[1:][:, np.argsort(SM[1])].mean(axis=0)
    print("A by SM id (mean over epochs):", " ".join(f"{v:.0f}" for v in abysm))


if __name__ == "__main__":
    main()
