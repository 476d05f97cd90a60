"""Multi-process (world size 2, gloo on CPU) test of the sharded epoch protocol.

The product's ShardedRunner (distributed.py) drives one sharded epoch as
partial epoch -> all-reduce of the exchange buffer -> finish.  On a GPU box the
backend is DeviceShard (the epoch kernel with BCT_SHARDED + NCCL); here each
rank runs the same runner over a test-side backend built from the CPU oracle
(owned column blocks only, epoch-start r), with torch.distributed over gloo as
the all-reduce.  The assembled image and the replicated residual must match a
single-process parallel run of the oracle (the per-j refresh fold
becomes a per-rank fold, so equality is to rounding, checked at 1e-12).
"""

import os
import socket
import sys
from types import SimpleNamespace

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

torch = pytest.importorskip("torch")

N, VIEWS, BINS, M, NC = 32, 30, 46, 4, 4
EPOCHS, B, GS, SEED = 4, 0.25, 2, 11


def _system():
    from oracle.oracle import OracleSystem
    return OracleSystem.parallel_beam(N, VIEWS, BINS, M, NC)


def _inputs(system):
    from paper_1709_00953_b200.geometry import add_noise, random_ellipses
    x_true = random_ellipses(N, 4, 0)
    y, _ = add_noise(system.forward(x_true), 0.01, 1)
    return x_true, y


def _plans(system):
    from oracle.oracle import oracle_epoch_plan, oracle_group_beta
    rng = np.random.default_rng(SEED)
    out = []
    for _ in range(EPOCHS):
        plan = oracle_epoch_plan(system.table, rng, 1.0, 1.0, GS)
        out.append([(j, [(ids, oracle_group_beta(system.table, B, j, ids)) for ids in groups])
                    for j, groups in plan])
    return out


class OracleShard:
    """ShardedRunner backend over the CPU oracle (test side only)."""

    def __init__(self, system, state, owned, x_true):
        self.sys, self.state, self.owned, self.x_true = system, state, owned, x_true
        self.n_meas = state.y.size
        self.buf = torch.zeros(self.n_meas + 2, dtype=torch.float64)
        self.drawn = None

    def run_partial(self, packed, flags):
        from oracle.oracle import OracleStats, _commit_visit, _run_visit, oracle_commit_epoch
        s, st = self.sys, self.state
        lo, hi = self.owned
        snaps = {j: np.ascontiguousarray(st.x[s.vidx[j]]) for j, _ in packed.loops}
        stats = OracleStats()
        runs = [_run_visit(s, j, groups, st.r, snaps[j]) for j, groups in packed.loops
                if lo <= j < hi]
        for run in runs:
            _commit_visit(s, st, run, stats)
        oracle_commit_epoch(st, s)
        part = np.zeros(self.n_meas)
        for j in range(lo, hi):                       # ascending j inside the rank
            np.add.at(part, s.l2g[j], st.z[j])
        vox = np.concatenate([s.vidx[j] for j in range(lo, hi)])
        self.buf[:self.n_meas] = torch.from_numpy(part)
        self.buf[self.n_meas] = float(np.sum(st.x[vox] ** 2))
        self.buf[self.n_meas + 1] = float(np.sum((self.x_true[vox] - st.x[vox]) ** 2))
        self.drawn = np.concatenate([np.concatenate([np.asarray(g) for g, _ in groups])
                                     for _, groups in packed.loops])
        return SimpleNamespace(kernel_ms=0.0, n_degenerate=stats.n_degenerate)

    def exchange(self):
        return self.buf

    def finish(self, flags):
        st = self.state
        S = self.buf[:self.n_meas].numpy()
        rows = self.sys.measurement_rows(np.unique(self.drawn))
        st.r[rows] = st.y[rows] - S[rows]
        resid_sq = float(np.sum((st.y - S) ** 2))
        return resid_sq, float(self.buf[self.n_meas]), float(self.buf[self.n_meas + 1])


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from oracle.oracle import OracleState
    from paper_1709_00953_b200.distributed import ShardedRunner, owned_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        system = _system()
        x_true, y = _inputs(system)
        state = OracleState.initialize(system, y)
        owned = owned_range(NC, world, rank)
        runner = ShardedRunner(system, backend=OracleShard(system, state, owned, x_true),
                               allreduce=dist.all_reduce)
        rows = []
        for loops in _plans(system):
            packed = SimpleNamespace(loops=loops,
                                     task_j=np.array([j for j, g in loops for _ in g]))
            res = runner.epoch(packed, 0)
            rows.append((res.resid_sq, res.x_sq, res.err_sq, res.n_tasks))
        mine = np.zeros(system.n_voxels)
        for j in range(*owned):
            mine[system.vidx[j]] = state.x[system.vidx[j]]
        t = torch.from_numpy(mine)
        dist.all_reduce(t)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=t.numpy(), r=state.r,
                 rows=np.array(rows))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_owned_range_partitions_every_block():
    from paper_1709_00953_b200.distributed import owned_range
    from paper_1709_00953_b200.errors import ConfigurationError
    for n in (4, 7, 32, 64):
        for world in (1, 2, 3, 4, 8):
            if world > n:
                with pytest.raises(ConfigurationError):
                    owned_range(n, world, 0)
                continue
            spans = [owned_range(n, world, p) for p in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1


def test_sharded_epochs_two_gloo_ranks_match_single_process(tmp_path):
    import torch.multiprocessing as mp
    from oracle.oracle import OracleState, oracle_commit_epoch, oracle_run_epoch
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    # replicated state agrees across ranks bit for bit
    assert np.array_equal(r0["x"], r1["x"])
    assert np.array_equal(r0["r"], r1["r"])
    assert np.array_equal(r0["rows"], r1["rows"])
    # single-process parallel oracle on the same plans
    system = _system()
    x_true, y = _inputs(system)
    st = OracleState.initialize(system, y)
    for loops in _plans(system):
        oracle_run_epoch(system, st, loops, mode="parallel")
        oracle_commit_epoch(st, system)
    rel_x = np.linalg.norm(r0["x"] - st.x) / np.linalg.norm(st.x)
    rel_r = np.linalg.norm(r0["r"] - st.r) / np.linalg.norm(st.r)
    assert rel_x <= 1e-12 and rel_r <= 1e-12, (rel_x, rel_r)
    # trace norms of the last epoch (sum over ranks of the owned partials)
    resid_sq, x_sq, err_sq, n_tasks = r0["rows"][-1]
    assert n_tasks == sum(len(g) for _, g in _plans(system)[-1])
    assert abs(x_sq - np.sum(st.x ** 2)) <= 1e-12 * np.sum(st.x ** 2)
    assert abs(err_sq - np.sum((x_true - st.x) ** 2)) <= 1e-12 * np.sum((x_true - st.x) ** 2)
    S = system.projection_sum(st.z)
    assert abs(resid_sq - np.sum((y - S) ** 2)) <= 1e-10 * np.sum((y - S) ** 2)
