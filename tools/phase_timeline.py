"""Profiling helper: per-phase timeline of the epoch kernel (BCT_TIMELINE=1).

    BCT_TIMELINE=1 python tools/phase_timeline.py [--config 4] [--epochs 3]

Prints, per task, the span of phase 1 (CSC SpMV^T), barrier 1, phase 2 (dual
SpMV), barrier 2 and phase 3, in microseconds, plus the spread of the blocks'
finish times (load imbalance)."""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BCT_TIMELINE", "1")

from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig, SolverParams  # noqa
from paper_1709_00953_b200 import _native as N  # noqa
from paper_1709_00953_b200.executor import pack_loops, submit, wait  # noqa
from paper_1709_00953_b200.sampling import BlockScheduler  # noqa
from paper_1709_00953_b200.solvers import SolverState, _loops  # noqa
from paper_1709_00953_b200.geometry import random_ellipses, add_noise  # noqa


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--batched", action="store_true")
    ap.add_argument("--world", type=int, default=1,
                    help="build rank 0's share of a W-way sharded system (BCT_SHARDED epochs)")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    pr = (0, cfg.spec.nc // a.world)
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype, panel_range=pr)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    SolverState.initialize(s, y)
    sch = BlockScheduler(s.table, SamplingConfig(alpha=cfg.alpha), cfg.group_size)
    rng = np.random.default_rng(5)
    for e in range(a.epochs):
        packed = pack_loops(_loops(sch.epoch_plan(e + 1, rng), s.table, cfg.b), s)
        submit(s, cfg.mode, packed,
               N.BCT_COMMIT | N.BCT_METRICS | (N.BCT_SHARDED if a.world > 1 else 0))
        res = wait(s, packed.task_j.size)[0]
    nt = packed.task_j.size
    grid = ctypes.c_int32()
    buf = np.zeros(16 * nt * 4096, dtype=np.int64)
    N.check(N.load().bct_debug_timeline(s.ctx, N.ptr(buf), nt, ctypes.byref(grid)), s.ctx)
    G = grid.value
    tl = buf[:nt * 8 * G].reshape(nt, 8, G).astype(np.float64) / 1e3  # us
    print(f"config {a.config}: kernel {res.kernel_ms:.3f} ms, {nt} tasks, grid {G}")
    if a.batched:
        t = tl[0]
        st = t[0].min()
        print("batched epoch (us): A(g) %.1f  barA %.1f  B(seg) %.1f  barB %.1f  C(rows) %.1f  D(step) %.1f"
              "  tail %.1f"
              % (t[1].max() - st, t[2].max() - t[1].max(), t[3].max() - t[2].min(),
                 t[4].max() - t[3].max(), t[5].max() - t[4].min(), t[6].max() - t[5].max(),
                 t[7].max() - t[6].max()))
        for name, d in (("A per block", t[1] - t[0]), ("B per block", t[3] - t[2]),
                        ("C per block", t[5] - t[4])):
            q = np.percentile(d, [0, 10, 50, 90, 100])
            print(f"{name:12s} min {q[0]:6.1f} p10 {q[1]:6.1f} med {q[2]:6.1f} p90 {q[3]:6.1f} max {q[4]:6.1f}")
        x2 = buf[nt * 8 * G:2 * nt * 8 * G].reshape(nt, 8, G).astype(np.float64) / 1e3
        if (x2[0, 0] > 0).all():
            print("tail: measurement pass per block med %.1f max %.1f us; voxel pass med %.1f max %.1f us"
                  % (np.median(x2[0, 0] - t[6]), (x2[0, 0] - t[6]).max(),
                     np.median(t[7] - x2[0, 0]), (t[7] - x2[0, 0]).max()))
        if tl.shape[0] > 1:
            t1 = tl[1]
            allB = t1[4] - t[2]
            fb = t1[5] - t[0]
            ft = t1[6] - t[0]
            for name, d in (("B all warps", allB), ("A first band", fb), ("A first tile", ft),
                            ("B fence", t1[7] - t1[4])):
                q = np.percentile(d, [0, 10, 50, 90, 100])
                print(f"{name:12s} min {q[0]:6.1f} p10 {q[1]:6.1f} med {q[2]:6.1f} p90 {q[3]:6.1f} "
                      f"max {q[4]:6.1f}")
            if tl.shape[0] > 2:
                ts = tl[2]
                dd = [np.median(ts[i + 1] - ts[i]) for i in range(7) if (ts[i + 1] > 0).all()]
                print("A tile durations (median over blocks, us):", " ".join(f"{v:.1f}" for v in dd))
            print("B: last warp done %.1f us after the first block started B; fenced %.1f; "
                  "barrier release %.1f" % (t1[4].max() - t[2].min(), t1[7].max() - t[2].min(),
                                            t[4].max() - t[2].min()))
        if os.environ.get("DUMP_BLOCKS") and tl.shape[0] > 1:
            ub, ue, nst, stg = (buf[(1 * 8 + q) * G:(1 * 8 + q + 1) * G] for q in range(4))
            print("B super-tile staging per block (us):",
                  " ".join(f"{v / 1e3:.0f}" for v in stg[:40]))
            dB = t[3] - t[2]
            order = np.argsort(dB)
            print("B slowest blocks (us, slices, super tiles):",
                  " ".join(f"{dB[i]:.0f}/{ue[i]-ub[i]}/{nst[i]}" for i in order[-12:]))
            print("B fastest blocks:", " ".join(f"{dB[i]:.0f}/{ue[i]-ub[i]}/{nst[i]}" for i in order[:12]))
        if os.environ.get("DUMP_BLOCKS"):
            for name, d in (("A", t[1] - t[0]), ("B", t[3] - t[2])):
                print(name, "by block:", " ".join(f"{v:.0f}" for v in d))
        return
    print("task     p1   bar1    p2a  bar2+p2b  bar3     p3   total   (us, to the last block)")
    tot = np.zeros(6)
    for k in range(nt):
        t = tl[k]
        start = t[0].min()
        row = np.array([t[1].max() - start, t[2].max() - t[1].max(), t[3].max() - t[2].min(),
                        t[4].max() - t[3].max(), t[5].max() - t[4].max(), t[6].max() - t[5].min()])
        tot += row
        if k < 3 or k == nt - 1:
            print(f"{k:4d} " + " ".join(f"{v:6.1f}" for v in row) + f" {t[6].max() - start:7.1f}")
    print("mean " + " ".join(f"{v / nt:6.1f}" for v in tot))
    d7 = (tl[:, 7, :] - tl[:, 0, :]).ravel()
    d7 = d7[(d7 > 0) & (d7 < 1e4)]
    if d7.size:
        q = np.percentile(d7, [0, 50, 100])
        print(f"p1 first band staged after (us): min {q[0]:.1f} med {q[1]:.1f} max {q[2]:.1f}")
    d1 = (tl[:, 1, :] - tl[:, 0, :]).ravel()
    d2 = (tl[:, 3, :] - tl[:, 2, :]).ravel()
    for name, d in (("p1 per block", d1), ("p2a per block", d2)):
        q = np.percentile(d, [0, 10, 50, 90, 100])
        print(f"{name:14s} min {q[0]:6.1f} p10 {q[1]:6.1f} med {q[2]:6.1f} p90 {q[3]:6.1f} max {q[4]:6.1f}")
    # sub-phases per block (second half of the buffer): median / max over blocks and tasks
    x = buf[nt * 8 * G:2 * nt * 8 * G].reshape(nt, 8, G).astype(np.float64) / 1e3
    parts = [("band staged", tl[:, 7] - tl[:, 0]), ("first item", x[:, 0] - tl[:, 7]),
             ("p1 rest+sum", tl[:, 1] - x[:, 0]), ("bar1 wait", tl[:, 2] - tl[:, 1]),
             ("2a stage", x[:, 1] - tl[:, 2]), ("2a units", tl[:, 3] - x[:, 1]),
             ("rows", tl[:, 4] - tl[:, 3]), ("bar2+sums", tl[:, 5] - tl[:, 4]),
             ("mu, xhat", x[:, 3] - tl[:, 5]), ("refresh", x[:, 4] - x[:, 3]),
             ("record", x[:, 5] - x[:, 4]), ("bar3 wait", tl[1:, 0] - x[:-1, 5])]
    print("sub-phase (us per block, tasks pooled)   p10    med    p90    max")
    for name, d in parts:
        d = d.ravel()
        d = d[(d > -1) & (d < 1e4)]
        if d.size:
            q = np.percentile(d, [10, 50, 90, 100])
            print(f"  {name:14s} " + " ".join(f"{v:6.2f}" for v in q))
    if os.environ.get("DUMP_BLOCKS"):
        # phase-2a units (super-tile staged -> units done) per block, by task
        u = (tl[:, 3] - x[:, 1])
        for k in range(min(nt, 4)):
            print(f"task {k} 2a units by block:", " ".join(f"{v:.1f}" for v in u[k]))
        if nt > 2:
            print("2a units: corr task0-task1 %.2f, task1-task2 %.2f" %
                  (np.corrcoef(u[0], u[1])[0, 1], np.corrcoef(u[1], u[2])[0, 1]))
            slow = np.argsort(u.mean(axis=0))[-8:]
            print("slowest blocks (mean over tasks):", slow, u.mean(axis=0)[slow].round(2))
    k = 0
    d2k = tl[k, 3, :] - tl[k, 2, :]
    print("task 0 p2a by block (every 8th):", " ".join(f"{v:.0f}" for v in d2k[::8]))


if __name__ == "__main__":
    main()
