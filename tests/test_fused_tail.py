"""The fused batched tail (EpochHeader::fuse_tail): full-panel parallel epochs
keep z in (t, ax) form and form z = ax + mu t where the tail sums it, with no
phase D.  Every result must be bit for bit the one of the unfused path
(BCT_NO_FUSE_TAIL=1, phase D storing z): x after every epoch, r, and z once
it is read back (materialised), including when batched epochs alternate with
per-task epochs (partial groups) that read the stored z, and after a
teacher-forced load."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

bct = pytest.importorskip("paper_1709_00953_b200")
from conftest import golden  # noqa: E402
from paper_1709_00953_b200 import (CONFIGS, DeviceBlockSystem, EpochExecutor,  # noqa: E402
                                   SamplingConfig, SolverParams, SolverState, run_gcsgd)
from paper_1709_00953_b200.sampling import BlockScheduler  # noqa: E402
from paper_1709_00953_b200.solvers import _loops  # noqa: E402


@pytest.fixture(scope="module", params=["f64", "f32"])
def cfg1(request):
    g = golden("pb_cfg1_runs.npz")
    dev = DeviceBlockSystem.parallel_beam(CONFIGS[1].spec, dtype=request.param)
    return dev, g["y"], g["x_true"]


class fused:
    """Run the block with the fused tail on (default) or off."""

    def __init__(self, on):
        self.on = on

    def __enter__(self):
        if self.on:
            os.environ.pop("BCT_NO_FUSE_TAIL", None)
        else:
            os.environ["BCT_NO_FUSE_TAIL"] = "1"

    def __exit__(self, *exc):
        os.environ.pop("BCT_NO_FUSE_TAIL", None)


def run(dev, y, xt, fuse, p, schedule=None):
    xs = []
    with fused(fuse):
        x, tr = run_gcsgd(dev, y, p, x_true=xt, schedule=schedule,
                          callback=lambda e, s, r: xs.append(s.x.copy()))
        return xs, x, dev.get_r(), [z.copy() for z in dev.get_z()], [r.snr_db for r in tr.rows]


def same(a, b):
    xs_a, x_a, r_a, z_a, s_a = a
    xs_b, x_b, r_b, z_b, s_b = b
    assert len(xs_a) == len(xs_b)
    assert all(np.array_equal(p, q) for p, q in zip(xs_a, xs_b))
    assert np.array_equal(x_a, x_b)
    assert np.array_equal(r_a, r_b)
    assert all(np.array_equal(p, q) for p, q in zip(z_a, z_b))
    assert s_a == s_b


def test_fused_tail_bitwise_full_panel_epochs(cfg1):
    """Parallel epochs of full groups (the batched path) fused and unfused."""
    dev, y, xt = cfg1
    p = SolverParams(epochs=12, b=0.4, group_size=4, seed=7, execution_mode="parallel",
                     sampling=SamplingConfig(alpha=0.75))
    same(run(dev, y, xt, True, p), run(dev, y, xt, False, p))


def test_fused_tail_alternating_with_per_task_epochs(cfg1):
    """Scripted plan: odd epochs visit every column block with all 4 row
    blocks (batched, z left in (t, ax) form), even epochs draw two row blocks
    per visit (per-task path: z is written out first), the last epochs skip a
    column block so a panel stays in (t, ax) form over a batched epoch."""
    dev, y, xt = cfg1
    full = np.arange(4, dtype=np.int64)
    sched = {}
    for e in range(1, 11):
        if e >= 8:
            sched[e] = [(j, full) for j in (0, 2, 3)]
        elif e % 2:
            sched[e] = [(j, full) for j in range(4)]
        else:
            sched[e] = [(j, np.array([(j + e) % 4, (j + e + 1) % 4], dtype=np.int64))
                        for j in range(4)]
    p = SolverParams(epochs=10, b=0.3, group_size=4, seed=2, execution_mode="parallel")
    same(run(dev, y, xt, True, p, sched), run(dev, y, xt, False, p, sched))


def test_fused_tail_after_teacher_forced_load(cfg1):
    """Fused epochs, then a load of another state (set_z over a panel in
    (t, ax) form), then one batched epoch: equal to the unfused sequence."""
    dev, y, xt = cfg1
    rng = np.random.default_rng(3)
    xl = rng.standard_normal(dev.n_voxels) * 0.1
    zl = [rng.standard_normal(dev.n_local_rows(j)) for j in range(dev.n_col_blocks)]
    rl = rng.standard_normal(dev.n_measurements)
    sch = BlockScheduler(dev.table, SamplingConfig(alpha=1.0), group_size=4)
    plan = sch.epoch_plan(1, np.random.default_rng(0))
    loops = _loops(plan, dev.table, 0.3)
    outs = []
    for fuse in (True, False):
        with fused(fuse):
            st = SolverState.initialize(dev, y)
            for e in range(3):
                EpochExecutor("parallel").run_epoch(e + 1, loops, st, dev)
                dev.commit_epoch()
            st.load(xl, rl, zl)
            EpochExecutor("parallel").run_epoch(4, loops, st, dev)
            dev.commit_epoch()
            outs.append((st.x.copy(), st.r.copy(), [z.copy() for z in st.z]))
    (xa, ra, za), (xb, rb, zb) = outs
    assert np.array_equal(xa, xb) and np.array_equal(ra, rb)
    assert all(np.array_equal(p, q) for p, q in zip(za, zb))
