"""Small batched + per-task epochs for compute-sanitizer runs (profiling aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, SamplingConfig,  # noqa: E402
                                   SolverParams, add_noise, random_ellipses, run_gcsgd)

key = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = CONFIGS[key]
s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
runs = (("parallel", cfg.spec.m, 1.0), ("serial_faithful", 1, 0.5))
if len(sys.argv) > 2:
    runs = [r for r in runs if r[0] == sys.argv[2]]
for mode, gs, alpha in runs:
    print("running", mode, flush=True)
    x, tr = run_gcsgd(s, y, SolverParams(epochs=2, b=0.1, group_size=gs, execution_mode=mode,
                                         seed=3, sampling=SamplingConfig(alpha=alpha)), x_true=xt)
    print(mode, tr.rows[-1].snr_db)
