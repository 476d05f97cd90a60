"""Profiling helper: bench.py's device loop followed by timed run_gcsgd calls
with wall-clock marks at every submit / wait (host-side gaps per epoch).

    python tools/e2e_trace.py --config 3
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1709_00953_b200.solvers as S
    from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, SamplingConfig, SolverParams,
                                       add_noise, random_ellipses, run_gcsgd)
    from paper_1709_00953_b200 import _native as N
    from paper_1709_00953_b200.executor import pack_loops, submit, wait
    from paper_1709_00953_b200.sampling import BlockScheduler
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--device-loop", type=int, default=1)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    p = SolverParams(epochs=20, b=cfg.b, group_size=cfg.group_size, execution_mode=cfg.mode,
                     seed=5, sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
    if a.device_loop:
        S.SolverState.initialize(s, y)
        sch = BlockScheduler(s.table, p.sampling, group_size=p.group_size)
        rng = np.random.default_rng(1)
        plans = [pack_loops(S._loops(sch.epoch_plan(e + 1, rng), s.table, p.b), s)
                 for e in range(23)]
        for pl in plans:
            submit(s, cfg.mode, pl, N.BCT_COMMIT | N.BCT_METRICS)
            wait(s, pl.task_j.size)
    y_h = torch.empty(y.size, dtype=torch.float64).pin_memory().numpy()
    xt_h = torch.empty(xt.size, dtype=torch.float64).pin_memory().numpy()
    y_h[:] = y
    xt_h[:] = xt
    marks = []
    ow, osub = S.wait, S.submit
    S.wait = lambda *x, **k: (lambda r: (marks.append(("wait", time.perf_counter())), r)[1])(ow(*x, **k))
    def sub(*x, **k):
        marks.append(("submit", time.perf_counter()))
        r = osub(*x, **k)
        marks.append(("submitted", time.perf_counter()))
        return r
    S.submit = sub
    import cProfile
    import pstats
    for rep in range(int(os.environ.get('REPS', '4'))):
        marks.clear()
        prof = cProfile.Profile() if rep == 0 and os.environ.get("PROFILE") else None
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        _, tr = run_gcsgd(s, y_h, p, x_true=xt_h)
        if prof:
            prof.disable()
            pstats.Stats(prof).sort_stats("cumulative").print_stats(18)
        t1 = time.perf_counter()
        gaps = [f"{marks[i + 1][0][:4]}+{1e3 * (marks[i + 1][1] - marks[i][1]):.2f}"
                for i in range(len(marks) - 1)]
        print(f"run {rep}: {1e3 * (t1 - t0):.2f} ms; first submit {1e3 * (marks[0][1] - t0):.2f} "
              f"ms; {' '.join(gaps[:10])} ...")
        waits = [m[1] for m in marks if m[0] == "wait"]
        iv = [1e3 * (b - a) for a, b in zip(waits, waits[1:])]
        kms = [r.kernel_ms for r in tr.rows]
        print(f"   kernel sum {sum(kms):.2f} ms (min {min(kms):.3f} max {max(kms):.3f}); "
              f"wait-to-wait max {max(iv):.2f} ms; last wait -> return {1e3 * (t1 - waits[-1]):.2f} ms")
        print("   wait-to-wait " + " ".join(f"{v:.2f}" for v in iv))
        print("   kernel_ms " + " ".join(f"{v:.3f}" for v in kms))


if __name__ == "__main__":
    main()
