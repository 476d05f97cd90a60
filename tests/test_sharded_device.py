"""The sharded device path with more than one shard, on one GPU:
two contexts own column blocks [0, 2) and [2, 4) of config 1 and run the
product's ``run_gcsgd_sharded`` / ``ShardedRunner`` / ``DeviceShard`` in two
threads.  The all-reduce is test-side: both exchange buffers summed in rank
order after a device synchronize (the contexts' kernels never wait on each
other, so both ranks' epochs are independent launches).  The result must match
the single-context run and the oracle at 1e-12: the sharded refresh folds
(z0 + z1) + (z2 + z3) where one context folds ((z0 + z1) + z2) + z3."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

bct = pytest.importorskip("paper_1709_00953_b200")
torch = pytest.importorskip("torch")
from conftest import golden  # noqa: E402
from oracle.oracle import OracleSystem, oracle_run_gcsgd  # noqa: E402
from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, DivergenceError,  # noqa: E402
                                   SamplingConfig, SolverParams, run_gcsgd)
from paper_1709_00953_b200.distributed import ShardedRunner, run_gcsgd_sharded  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


class ThreadAllReduce:
    """In-place sum of one device tensor per rank-thread, in rank order."""

    def __init__(self, n):
        self.n = n
        self.slots = [None] * n
        self.rank = {}
        self.barrier = threading.Barrier(n)

    def register(self, r):
        self.rank[threading.get_ident()] = r

    def __call__(self, t):
        r = self.rank[threading.get_ident()]
        self.slots[r] = t
        self.barrier.wait()
        if r == 0:
            torch.cuda.synchronize()
            acc = self.slots[0].clone()
            for q in range(1, self.n):
                acc += self.slots[q]
            for q in range(self.n):
                self.slots[q].copy_(acc)
            torch.cuda.synchronize()
        self.barrier.wait()


def run_shards(spec, y, p, xt, ranges, dtype="f64"):
    ar = ThreadAllReduce(len(ranges))
    systems = [DeviceBlockSystem.parallel_beam(spec, dtype=dtype, panel_range=pr)
               for pr in ranges]
    out = [None] * len(ranges)

    def worker(r):
        ar.register(r)
        torch.cuda.set_device(0)
        try:
            out[r] = run_gcsgd_sharded(systems[r], y, p, x_true=xt, allreduce=ar,
                                       runner=ShardedRunner(systems[r], allreduce=ar))
        except Exception as exc:  # re-raised by the caller
            out[r] = exc
            ar.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(len(ranges))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out, systems


@pytest.fixture(scope="module")
def cfg1():
    g = golden("pb_cfg1_runs.npz")
    spec = CONFIGS[1].spec
    return spec, g["y"], g["x_true"], DeviceBlockSystem.parallel_beam(spec, dtype="f64")


@pytest.mark.parametrize("ranges", [[(0, 2), (2, 4)], [(0, 1), (1, 3), (3, 4)]])
def test_sharded_contexts_match_single_context(cfg1, ranges):
    spec, y, xt, full = cfg1
    p = SolverParams(epochs=8, b=0.25, group_size=2, seed=19, execution_mode="parallel",
                     sampling=SamplingConfig(alpha=0.75))
    x_ref, tr_ref = run_gcsgd(full, y, p, x_true=xt)
    ora = OracleSystem.parallel_beam(spec.n, spec.views, spec.bins, spec.m, spec.nc)
    x_ora, rows = oracle_run_gcsgd(ora, y, 8, 0.25, alpha=0.75, group_size=2, mode="parallel",
                                   seed=19, x_true=xt)
    out, systems = run_shards(spec, y, p, xt, ranges)
    for r in out:
        assert not isinstance(r, Exception), r
    for x_sh, tr_sh in out:
        assert rel(x_sh, x_ref) <= 1e-12
        assert rel(x_sh, x_ora) <= 1e-12
        np.testing.assert_allclose([r.obs_gap_db for r in tr_sh.rows],
                                   [r["obs_gap_db"] for r in rows], rtol=1e-12)
        np.testing.assert_allclose([r.snr_db for r in tr_sh.rows],
                                   [r.snr_db for r in tr_ref.rows], rtol=1e-12)
    # every rank ends with the same replicated residual
    r0 = systems[0].get_r()
    for s in systems[1:]:
        assert np.array_equal(s.get_r(), r0)
    assert rel(r0, full.get_r()) <= 1e-12


def test_sharded_divergence_guard(cfg1):
    """Full-panel parallel epochs with b=4 diverge within a few epochs: the
    sharded run raises at the single-context run's epoch, and the guarded
    (already enqueued) next epoch leaves every shard at the diverged epoch's
    state."""
    spec, y, xt, full = cfg1
    p = SolverParams(epochs=50, b=4.0, group_size=4, seed=3, execution_mode="parallel",
                     sampling=SamplingConfig(alpha=1.0))
    with pytest.raises(DivergenceError) as exc:
        run_gcsgd(full, y, p, x_true=xt)
    last = exc.value.last_good_epoch
    x_full = full.get_x()
    out, systems = run_shards(spec, y, p, xt, [(0, 2), (2, 4)])
    for r in out:
        assert isinstance(r, DivergenceError) and r.last_good_epoch == last
    x = np.zeros_like(x_full)
    for s in systems:
        xl = s.get_x()
        for j in range(s.panel_begin, s.panel_end):
            v = s.voxel_indices(j)
            x[v] = xl[v]
    assert rel(x, x_full) <= 1e-9


@pytest.mark.parametrize("dtype,world,tol", [("f64", 2, 1e-12), ("f32", 2, 1e-6), ("f32", 4, 1e-6)])
def test_sharded_batched_epochs_at_config3(dtype, world, tol):
    """The path a multi-GPU bench run takes: config 3's parallel full-panel
    epochs (the batched epoch kernel with BCT_SHARDED, exchange, finish) over
    2 and 4 shards against the one-context run of the same dtype.  FP64 folds
    the shards' projection sums in a different order (1e-12); the FP32 store's
    (t, ax) pairs are FP32, so a different fold of S moves r at the 1e-7 level."""
    cfg = CONFIGS[3]
    spec = cfg.spec
    from paper_1709_00953_b200 import add_noise, random_ellipses
    full = DeviceBlockSystem.parallel_beam(spec, dtype=dtype)
    xt = random_ellipses(spec.n, cfg.n_ellipses, cfg.phantom_seed)
    y, _ = add_noise(full.forward(xt), cfg.noise_frac, cfg.noise_seed)
    p = SolverParams(epochs=6, b=cfg.b, group_size=cfg.group_size, seed=1234,
                     execution_mode=cfg.mode,
                     sampling=SamplingConfig(alpha=cfg.alpha, gamma=cfg.gamma))
    x_ref, tr_ref = run_gcsgd(full, y, p, x_true=xt)
    r_ref = full.get_r()
    full.close()
    nc = spec.nc
    ranges = [(q * nc // world, (q + 1) * nc // world) for q in range(world)]
    out, systems = run_shards(spec, y, p, xt, ranges, dtype=dtype)
    for r in out:
        assert not isinstance(r, Exception), r
    for x_sh, tr_sh in out:
        assert rel(x_sh, x_ref) <= tol
        np.testing.assert_allclose([r.obs_gap_db for r in tr_sh.rows],
                                   [r.obs_gap_db for r in tr_ref.rows], rtol=max(tol, 1e-11))
        np.testing.assert_allclose([r.snr_db for r in tr_sh.rows],
                                   [r.snr_db for r in tr_ref.rows], rtol=max(tol, 1e-11))
    r0 = systems[0].get_r()
    for s in systems[1:]:
        assert np.array_equal(s.get_r(), r0)
    assert rel(r0, r_ref) <= 10 * tol
    for s in systems:
        s.close()
