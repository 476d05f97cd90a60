"""Profiling helper: one rank's share of a W-way sharded epoch on one GPU.

Builds only the column blocks rank 0 of W would own, runs the sharded epoch
path (exchange buffer, NCCL all-reduce at world size 1, finish) and reports
device ms per epoch -- the per-rank cost the 8-GPU run will see, minus the
inter-GPU all-reduce time.

    python tools/shard_sim.py --config 4 --world 8 [--epochs 20]
"""
import argparse
import os
import socket
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem, SamplingConfig
    from paper_1709_00953_b200 import _native as N
    from paper_1709_00953_b200.distributed import ShardedRunner, owned_range
    from paper_1709_00953_b200.executor import pack_loops
    from paper_1709_00953_b200.geometry import add_noise, random_ellipses
    from paper_1709_00953_b200.sampling import BlockScheduler
    from paper_1709_00953_b200.solvers import SolverState, _loops

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--epochs", type=int, default=20)
    a = ap.parse_args()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    cfg = CONFIGS[a.config]
    pr = owned_range(cfg.spec.nc, a.world, 0)
    s = DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype, panel_range=pr)
    xt = random_ellipses(cfg.spec.n, cfg.n_ellipses, 0)
    y, _ = add_noise(s.forward(xt), cfg.noise_frac, 1)
    SolverState.initialize(s, y)
    sch = BlockScheduler(s.table, SamplingConfig(alpha=cfg.alpha), cfg.group_size)
    rng = np.random.default_rng(5)
    plans = [pack_loops(_loops(sch.epoch_plan(e + 1, rng), s.table, cfg.b), s)
             for e in range(a.epochs + 3)]
    runner = ShardedRunner(s)
    flags = N.BCT_COMMIT | N.BCT_METRICS
    stream = torch.cuda.ExternalStream(s.stream(), device=0)
    for e in range(3):
        runner.epoch(plans[e], flags)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    km = []
    t_sub = []
    t0 = time.perf_counter()
    runner.submit(plans[3], flags)
    for e in range(3, a.epochs + 3):
        if e + 1 < a.epochs + 3:
            ts = time.perf_counter()
            runner.submit(plans[e + 1], flags)
            t_sub.append(time.perf_counter() - ts)
        km.append(runner.collect().kernel_ms)
    ev1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.epochs
    ms = ev0.elapsed_time(ev1) / a.epochs
    print(f"config {a.config}, rank 0 of {a.world} (panels {pr}): {ms:.3f} ms/epoch, "
          f"epoch kernel {np.mean(km):.3f} ms; host submit {1e3 * np.mean(t_sub):.3f} ms/epoch, "
          f"wall {1e3 * wall:.3f} ms/epoch")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
