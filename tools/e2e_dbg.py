import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig, SolverParams, add_noise, random_ellipses, run_gcsgd
cfg = CONFIGS[int(sys.argv[1])]
s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
y_h = torch.empty(y.size, dtype=torch.float64).pin_memory().numpy(); y_h[:] = y
xt_h = torch.empty(xt.size, dtype=torch.float64).pin_memory().numpy(); xt_h[:] = xt
stream = torch.cuda.ExternalStream(s.stream(), device=0)
for ep in (3, 3, 20, 20, 20, 20):
    p = SolverParams(epochs=ep, b=cfg.b, group_size=cfg.group_size, execution_mode=cfg.mode, seed=7, sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(stream)
    run_gcsgd(s, y_h, p, x_true=xt_h)
    e1.record(stream); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(ep, "wall %.2f ms, events %.2f ms" % (1e3*(t1-t0), e0.elapsed_time(e1)))
