"""Profiling helper: where a sharded epoch's stream time goes outside the
epoch kernel (rank 0's share of a W-way run on one GPU, NCCL at world size 1).

Records CUDA events on the context stream around the three stream sections
of ShardedRunner.submit -- partial epoch (upload + cooperative launch),
all-reduce, finish (+ result copy) -- for back-to-back epochs, and prints the
median of each section next to the kernel's own event time.

    python tools/shard_parts.py --config 4 --world 8 [--epochs 20] [--noop-allreduce]
"""
import argparse
import os
import socket
import sys

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
    ap.add_argument("--noop-allreduce", action="store_true")
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
    n = a.epochs + 3
    plans = [pack_loops(_loops(sch.epoch_plan(e + 1, rng), s.table, cfg.b), s) for e in range(n)]
    ar = (lambda t: None) if a.noop_allreduce else None
    runner = ShardedRunner(s, allreduce=ar)
    be = runner.backend
    flags = N.BCT_COMMIT | N.BCT_METRICS
    stream = torch.cuda.ExternalStream(s.stream(), device=0)
    for e in range(3):
        runner.epoch(plans[e], flags)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.epochs)]
    km = []
    for i, e in enumerate(range(3, n)):
        ev = evs[i]
        ev[0].record(stream)
        tok = be.run_partial(plans[e], flags)
        ev[1].record(stream)
        with be.comm_stream():
            runner.allreduce(be.exchange())
        ev[2].record(stream)
        be.finish(flags)
        ev[3].record(stream)
        km.append(be.result(tok).kernel_ms)
    torch.cuda.synchronize()
    part = np.array([[ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                      ev[2].elapsed_time(ev[3]), ev[0].elapsed_time(ev[3])] for ev in evs]) * 1e3
    med = np.median(part, axis=0)
    kmed = 1e3 * np.median(km)
    print(f"config {a.config}, rank 0 of {a.world}{' (no-op all-reduce)' if ar else ''}: "
          f"partial {med[0]:.1f} us (kernel {kmed:.1f}, upload+launch {med[0] - kmed:.1f}), "
          f"all-reduce {med[1]:.1f} us, finish+copy {med[2]:.1f} us, epoch {med[3]:.1f} us "
          f"(unpipelined)")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
