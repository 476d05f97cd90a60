import os, sys, socket
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig
from paper_1709_00953_b200 import _native as N
from paper_1709_00953_b200.distributed import ShardedRunner, owned_range
from paper_1709_00953_b200.executor import pack_loops
from paper_1709_00953_b200.geometry import add_noise, random_ellipses
from paper_1709_00953_b200.sampling import BlockScheduler
from paper_1709_00953_b200.solvers import SolverState, _loops
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
cfg = CONFIGS[4]
sy = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype, panel_range=owned_range(cfg.spec.nc, 8, 0))
xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
y, _ = add_noise(sy.forward(xt), cfg.noise_frac, 1)
SolverState.initialize(sy, y)
sch = BlockScheduler(sy.table, SamplingConfig(alpha=cfg.alpha), cfg.group_size)
rng = np.random.default_rng(5)
runner = ShardedRunner(sy)
flags = N.BCT_COMMIT | N.BCT_METRICS
for e in range(3):
    runner.epoch(pack_loops(_loops(sch.epoch_plan(e + 1, rng), sy.table, cfg.b), sy), flags)
stream = torch.cuda.ExternalStream(sy.stream(), device=0)
be = runner.backend
torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
evs[0].record(stream)
for i in range(11):
    be.finish(0)
    evs[i + 1].record(stream)
torch.cuda.synchronize()
print("finish alone, back to back (us):", [round(1e3 * evs[i].elapsed_time(evs[i + 1]), 1) for i in range(11)])
# plain torch reference of the same traffic
n = sy.n_measurements
a = torch.randn(n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a); c = torch.empty_like(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): torch.sub(a, b, out=c)
e0.record(); 
for _ in range(10): torch.sub(a, b, out=c)
e1.record(); torch.cuda.synchronize()
print("torch sub (same n, f64) us:", round(1e3 * e0.elapsed_time(e1) / 10, 1))
dist.destroy_process_group()
