"""Check: the one-thread-per-row bank permutation (layout.cu) equals the warp-
serial original bit for bit (same trajectory), and the build time of each.

    python tools/bankperm_check.py --config 3
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, SamplingConfig, SolverParams,
                                       add_noise, random_ellipses, run_gcsgd)
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    out = {}
    for name in ("old", "new"):
        if name == "old":
            os.environ["BCT_OLD_BANK_PERM"] = "1"
        else:
            os.environ.pop("BCT_OLD_BANK_PERM", None)
        t0 = time.perf_counter()
        s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
        tb = time.perf_counter() - t0
        y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
        p = SolverParams(epochs=3, b=cfg.b, group_size=cfg.group_size, execution_mode=cfg.mode,
                         seed=5, sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
        x, _ = run_gcsgd(s, y, p, x_true=xt)
        out[name] = x
        print(f"config {a.config} {name}: build {tb:.2f} s")
        s.close()
    print("bitwise equal:", np.array_equal(out["old"], out["new"]))


if __name__ == "__main__":
    main()
