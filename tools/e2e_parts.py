"""Profiling helper: host-side costs around the epochs of an end-to-end
run_gcsgd (state uploads, first plan, read-back), wall clock with syncs.

    python tools/e2e_parts.py [--config 4]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig  # noqa: E402
from paper_1709_00953_b200 import add_noise, random_ellipses  # noqa: E402
from paper_1709_00953_b200.executor import pack_loops  # noqa: E402
from paper_1709_00953_b200.sampling import BlockScheduler  # noqa: E402
from paper_1709_00953_b200.solvers import SolverState, _loops  # noqa: E402


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    print(f"config {a.config}: n_meas {y.size}, n_vox {xt.size}")
    print("set_y          %.2f ms" % t(lambda: s.set_y(y)))
    print("set_x_true     %.2f ms" % t(lambda: s.set_x_true(xt)))
    print("initialize     %.2f ms" % t(lambda: SolverState.initialize(s, y)))
    print("get_x          %.2f ms" % t(lambda: s.get_x()))
    sch = BlockScheduler(s.table, SamplingConfig(alpha=cfg.alpha), cfg.group_size)
    rng = np.random.default_rng(5)
    print("plan + pack    %.2f ms" % t(lambda: pack_loops(
        _loops(sch.epoch_plan(1, rng), s.table, cfg.b), s)))
    print("np.copy 8 MB   %.2f ms" % t(lambda: np.copy(y)))


if __name__ == "__main__":
    main()


def timeline(cfg_key=4, epochs=20):
    """Wall-clock marks inside one run_gcsgd (monkey-patched wait/submit)."""
    import paper_1709_00953_b200.solvers as S
    from paper_1709_00953_b200 import SolverParams, run_gcsgd
    cfg = CONFIGS[cfg_key]
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    marks = []
    ow, osub = S.wait, S.submit
    S.wait = lambda *a, **k: (lambda r: (marks.append(("wait", time.perf_counter())), r)[1])(ow(*a, **k))
    S.submit = lambda *a, **k: (marks.append(("submit", time.perf_counter())), osub(*a, **k))[1]
    p = SolverParams(epochs=epochs, b=cfg.b, group_size=cfg.group_size, execution_mode=cfg.mode,
                     seed=5, sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
    for rep in range(2):
        marks.clear()
        t0 = time.perf_counter()
        run_gcsgd(s, y, p, x_true=xt)
        t1 = time.perf_counter()
        print(f"run {rep}: total {1e3 * (t1 - t0):.2f} ms")
        for name, tm in marks[:4] + marks[-3:]:
            print(f"  {name:6s} {1e3 * (tm - t0):8.2f}")
    S.wait, S.submit = ow, osub


if __name__ == "__main__" and os.environ.get("E2E_TIMELINE"):
    timeline()
