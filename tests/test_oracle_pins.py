"""Pin the CPU oracle to the reference before trusting it: every golden
vector here was produced by running the reference package itself
(tests/golden/make_golden.py).  Bit-exact throughout -- the oracle restates
the reference's strict-order, no-FMA numba kernels."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, unflatten_plans
from oracle.oracle import (OracleState, OracleSystem, OracleTable, oracle_commit_epoch,
                           oracle_run_epoch, oracle_run_gcsgd)

VARIANTS = {
    "p1": dict(epochs=500, b=0.5, group_size=1, seed=1234, mode="serial_faithful", alpha=0.25),
    "ser_g2": dict(epochs=20, b=0.5, group_size=2, seed=11, mode="serial_faithful"),
    "par_full": dict(epochs=20, b=0.25, group_size=4, seed=12, mode="parallel"),
    "par_mixed": dict(epochs=20, b=0.3, group_size=1, seed=13, mode="parallel",
                      strategy="mixed", alpha=0.5, gamma=0.5, theta0=0.2, theta_step=0.1),
    "ser_random": dict(epochs=20, b=0.5, group_size=3, seed=14, mode="serial_faithful",
                       strategy="random", alpha=0.75),
}


def _h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def cfg1():
    return OracleSystem.parallel_beam(64, 90, 92, 4, 4)


def fixture_oracle(npz):
    nc, m = int(npz["nc"]), int(npz["m"])
    vals = npz["table"]
    return OracleSystem([npz[f"data{j}"] for j in range(nc)], [npz[f"cols{j}"] for j in range(nc)],
                        [npz[f"indptr{j}"] for j in range(nc)], [npz[f"rbp{j}"] for j in range(nc)],
                        [npz[f"l2g{j}"] for j in range(nc)], [npz[f"rows{i}"] for i in range(m)],
                        [npz[f"vidx{j}"] for j in range(nc)],
                        OracleTable(vals, vals.sum(axis=0)), int(npz["n_meas"]),
                        int(npz["n_vox"]))


def test_tracer_reproduces_reference_small_system():
    g = golden("pb_small.npz")
    s = OracleSystem.parallel_beam(16, 20, 24, 4, 4)
    for j in range(4):
        for k, arr in (("data", s.data), ("cols", s.cols), ("indptr", s.indptr),
                       ("rbp", s.rbp), ("l2g", s.l2g)):
            np.testing.assert_array_equal(arr[j], g[f"{k}{j}"])
    np.testing.assert_array_equal(s.table.values, g["table"])
    np.testing.assert_array_equal(s.forward(g["x_true"]), g["y_clean"])


@pytest.mark.parametrize("key,shape", [(1, (64, 90, 92, 4, 4)), (2, (256, 180, 367, 8, 8))])
def test_tracer_reproduces_reference_hashes(key, shape):
    H = json.load(open(os.path.join(GOLDEN, "pb_hashes.json")))
    s = OracleSystem.parallel_beam(*shape)
    for j, h in enumerate(H[f"cfg{key}"]):
        assert s.data[j].size == h["nnz"]
        for k in ("data", "cols", "indptr", "rbp", "l2g"):
            assert _h(getattr(s, k)[j]) == h[k], (j, k)
    assert _h(s.table.values) == H[f"cfg{key}_table_sha"]


@pytest.mark.parametrize("name", list(VARIANTS))
def test_oracle_runs_bitwise_equal_reference(cfg1, cfg1_runs, name):
    g = cfg1_runs
    rec = {}
    x, rows = oracle_run_gcsgd(cfg1, g["y"], x_true=g["x_true"], plan_record=rec,
                               **VARIANTS[name])
    np.testing.assert_array_equal(x, g[f"{name}_x"])
    np.testing.assert_array_equal([r["obs_gap_db"] for r in rows], g[f"{name}_gap"])
    np.testing.assert_array_equal([r["snr_db"] for r in rows], g[f"{name}_snr"])
    want = unflatten_plans(g[f"{name}_plans"])
    for ep, visits in want.items():
        got = [(j, np.concatenate(gr)) for j, gr in rec[ep]]
        assert [j for j, _ in got] == [j for j, _ in visits]
        for (_, a), (_, b) in zip(got, visits):
            np.testing.assert_array_equal(a, b)


def test_oracle_known_answer_snr():
    """The reference's own golden: tests/test_solvers.py:196-202."""
    f = golden("fan12.npz")
    s = fixture_oracle(f)
    np.testing.assert_array_equal(s.forward(f["x_true"]), f["y"])
    x, rows = oracle_run_gcsgd(s, f["y"], 30, 6.0, seed=3, x_true=f["x_true"])
    assert rows[-1]["snr_db"] == pytest.approx(6.416697928678968, abs=1e-9)
    np.testing.assert_array_equal(x, f["final_x"])


@pytest.mark.parametrize("gs", [1, 3])
@pytest.mark.parametrize("mode", ["serial_faithful", "parallel"])
def test_oracle_literal_epochs(gs, mode):
    f = golden("fan10.npz")
    s = fixture_oracle(f)
    x, _ = oracle_run_gcsgd(s, f["y"], 4, 6.0, alpha=0.5, group_size=gs, mode=mode, seed=17,
                            x_true=f["x_true"])
    np.testing.assert_array_equal(x, f[f"x_{gs}_{mode}"])


EXEC_PLANS = {
    "barrier": [(0, [(np.array([2, 3]), 0.7)]), (1, [(np.array([2, 3]), 0.7)])],
    "workers": [(0, [(np.array([0, 5]), 0.8), (np.array([2, 7]), 0.6)]),
                (1, [(np.array([1, 4, 6]), 0.5)]), (3, [(np.array([3]), 0.9)])],
    "mutate": [(0, [(np.array([0, 5]), 0.8)]), (2, [(np.array([3]), 0.5)])],
}


@pytest.mark.parametrize("name", list(EXEC_PLANS))
@pytest.mark.parametrize("mode", ["serial_faithful", "parallel"])
@pytest.mark.parametrize("workers", [1, 4])
def test_oracle_executor_bitwise(name, mode, workers):
    f = golden("exec10.npz")
    s = fixture_oracle(f)
    st = OracleState.initialize(s, f["y"], x0=f["x0"])
    stats = oracle_run_epoch(s, st, EXEC_PLANS[name], mode, workers=workers)
    np.testing.assert_array_equal(st.xhat, f[f"{name}_{mode}_xhat"])
    np.testing.assert_array_equal(st.r, f[f"{name}_{mode}_r"])
    np.testing.assert_array_equal(np.concatenate(st.z), f[f"{name}_{mode}_z"])
    np.testing.assert_array_equal(st.counts, f[f"{name}_{mode}_counts"])
    assert (stats.n_tasks, stats.n_loops, stats.bytes_moved, stats.n_degenerate) == \
        tuple(f[f"{name}_{mode}_stats"])
    oracle_commit_epoch(st, s)
    np.testing.assert_array_equal(st.x, f[f"{name}_{mode}_x"])


def test_oracle_teacher_forced_snapshots(cfg1, cfg1_runs):
    """Epoch 11 of each grouped reference run from its epoch-10 snapshot."""
    g = cfg1_runs
    from oracle.oracle import oracle_group_beta
    for name in ("ser_g2", "par_full", "par_mixed", "ser_random"):
        v = VARIANTS[name]
        st = OracleState.initialize(cfg1, g["y"])
        st.x[:] = g[f"{name}_snap10_x"]
        st.r[:] = g[f"{name}_snap10_r"]
        z = g[f"{name}_snap10_z"]
        off = 0
        for j in range(4):
            n = st.z[j].size
            st.z[j][:] = z[off:off + n]
            off += n
        gs = v["group_size"]
        plan = unflatten_plans(g[f"{name}_plans"])[11]
        loops = [(j, [(ids[a:a + gs], oracle_group_beta(cfg1.table, v["b"], j, ids[a:a + gs]))
                      for a in range(0, ids.size, gs)]) for j, ids in plan]
        oracle_run_epoch(cfg1, st, loops, v["mode"])
        oracle_commit_epoch(st, cfg1)
        np.testing.assert_array_equal(st.x, g[f"{name}_snap11_x"])
        np.testing.assert_array_equal(st.r, g[f"{name}_snap11_r"])
        np.testing.assert_array_equal(np.concatenate(st.z), g[f"{name}_snap11_z"])
