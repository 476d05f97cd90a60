"""Host-side logic of the drop-in (no GPU): selection stream, schedules,
parameter validation, plan packing, geometry/partition, metrics, and the
C-ABI library surface (loads and exports every declared symbol)."""

import math
import os
import re

import numpy as np
import pytest

from conftest import REPO, golden, unflatten_plans
from paper_1709_00953_b200 import (CONFIGS, BlockScheduler, ConfigurationError, ConvergenceTrace,
                                   ProbabilityTable, SamplingConfig, ScheduleError,
                                   ScriptedScheduler, SolverParams, TraceRow, dump_schedule,
                                   mixed_weights, parse_schedule, random_ellipses,
                                   select_column_blocks, select_row_blocks, snr_db)
from paper_1709_00953_b200 import _native as N
from paper_1709_00953_b200.geometry import ParallelBeamSpec
from paper_1709_00953_b200.sampling import group_beta


def _table(seed=0, m=10, n=3):
    v = np.random.default_rng(seed).uniform(0.1, 2.0, size=(m, n))
    return ProbabilityTable(v, v.sum(axis=0))


# ---------------------------------------------------------------------------
# selection (sampling.py), with the reference tests' golden values
# ---------------------------------------------------------------------------

def test_first_draw_counts_golden():
    """tests/test_sampling.py:84-93 -- pins the exponential stream."""
    w = np.array([0.5, 0.25, 0.125, 0.125])
    rng = np.random.default_rng(12)
    counts = np.zeros(4, dtype=np.int64)
    for _ in range(4000):
        counts[select_row_blocks(w, 1, rng)[0]] += 1
    np.testing.assert_array_equal(counts, [2002, 992, 513, 493])


def test_select_row_blocks_k_independent_and_scale_free():
    w = np.array([0.7, 1.4, 0.2, 2.0, 1.1])
    r1, r2 = np.random.default_rng(21), np.random.default_rng(21)
    one = select_row_blocks(w, 1, r1)
    all5 = select_row_blocks(w, 5, r2)
    assert one[0] == all5[0]
    assert r1.random() == r2.random()
    a = select_row_blocks(w, 4, np.random.default_rng(5))
    np.testing.assert_array_equal(a, select_row_blocks(w * 7.3, 4, np.random.default_rng(5)))
    w0 = np.array([1.0, 0.0, 2.0, 3.0, 0.5])
    ids = select_row_blocks(w0, 4, np.random.default_rng(11))
    assert 1 not in ids and np.unique(ids).size == 4
    with pytest.raises(ScheduleError):
        select_row_blocks(w0, 5, np.random.default_rng(0))
    assert select_row_blocks(w0, 0, np.random.default_rng(0)).size == 0


def test_mixed_weights_and_column_draws():
    raw = np.array([4.0, 1.0, 0.0, 2.0])
    np.testing.assert_array_equal(mixed_weights(raw, 0.0), raw)
    np.testing.assert_array_equal(mixed_weights(raw, 1.0), [4.0, 4.0, 0.0, 4.0])
    np.testing.assert_allclose(mixed_weights(raw, 0.5), [4.0, 2.5, 0.0, 3.0])
    np.testing.assert_array_equal(mixed_weights(np.zeros(3), 0.5), np.zeros(3))
    el = np.array([0, 2, 3, 5, 6])
    np.testing.assert_array_equal(np.sort(select_column_blocks(el, 1.0,
                                                               np.random.default_rng(3))), el)
    assert select_column_blocks(el, 0.5, np.random.default_rng(4)).size == 3
    with pytest.raises(ScheduleError):
        select_column_blocks(np.empty(0, np.int64), 1.0, np.random.default_rng(0))


@pytest.mark.parametrize("strategy,theta0,step", [("importance", 0, 0), ("random", 0, 0),
                                                  ("mixed", 0.3, 0.25)])
@pytest.mark.parametrize("alpha,gamma,gs", [(1.0, 1.0, 1), (0.5, 0.67, 3), (0.25, 1.0, 64)])
def test_variate_bundle_replays_plan(strategy, theta0, step, alpha, gamma, gs):
    """The device sampler's input (one choice + one bulk exponential call per
    epoch), raced for all visits at once (epoch_plan), reproduces the
    reference's visit-by-visit draws (epoch_plan_per_visit) exactly, epoch
    after epoch."""
    tab = _table(seed=2, m=12, n=5)
    cfg = SamplingConfig(strategy=strategy, alpha=alpha, gamma=gamma, theta0=theta0,
                         theta_step=step)
    a, b = BlockScheduler(tab, cfg, gs), BlockScheduler(tab, cfg, gs)
    ra, rb = np.random.default_rng(9), np.random.default_rng(9)
    for ep in range(1, 6):
        pa = a.epoch_plan_per_visit(ep, ra)
        v = b.epoch_variates(ep, rb)
        pb = b.plan_from_variates(v)
        assert [j for j, _ in pa] == [j for j, _ in pb]
        for (_, ga), (_, gb) in zip(pa, pb):
            assert len(ga) == len(gb)
            for x, y in zip(ga, gb):
                np.testing.assert_array_equal(x, y)
        a.advance_epoch()
        b.advance_epoch()
    assert ra.random() == rb.random()


def test_scheduler_plans_match_reference_records(cfg1_runs):
    """The product scheduler reproduces the reference's recorded plans."""
    g = cfg1_runs
    tab = ProbabilityTable(g["table"], g["table"].sum(axis=0))
    for name, cfg, gs, seed in (
            ("p1", SamplingConfig(alpha=0.25), 1, 1234),
            ("par_mixed", SamplingConfig(strategy="mixed", alpha=0.5, gamma=0.5, theta0=0.2,
                                         theta_step=0.1), 1, 13),
            ("ser_random", SamplingConfig(strategy="random", alpha=0.75), 3, 14)):
        want = unflatten_plans(g[f"{name}_plans"])
        sch = BlockScheduler(tab, cfg, gs)
        rng = np.random.default_rng(seed)
        for ep in sorted(want):
            plan = sch.epoch_plan(ep, rng)
            sch.advance_epoch()
            assert [j for j, _ in plan] == [j for j, _ in want[ep]]
            for (_, gr), (_, ids) in zip(plan, want[ep]):
                np.testing.assert_array_equal(np.concatenate(gr), ids)


def test_schedule_dump_parse_roundtrip(tmp_path):
    plans = {1: [(0, [np.array([3, 1]), np.array([2])]), (2, [np.array([0])])],
             2: [(1, [np.array([1, 2, 3])])]}
    path = tmp_path / "s.txt"
    dump_schedule(plans, path)
    entries = parse_schedule(path, n_row_blocks=4, n_col_blocks=3)
    assert [j for j, _ in entries[1]] == [0, 2]
    np.testing.assert_array_equal(entries[1][0][1], [3, 1, 2])
    sch = ScriptedScheduler(entries, group_size=2)
    got = sch.epoch_plan(2, None)
    np.testing.assert_array_equal(got[0][1][0], [1, 2])
    np.testing.assert_array_equal(got[0][1][1], [3])
    with pytest.raises(ScheduleError):
        sch.epoch_plan(9, None)
    for bad in ("1 0 1 1\n", "1 0 7\n", "1 5 1\n", "1 -1 0\n", "1 0\n", "x 0 1\n"):
        (tmp_path / "b.txt").write_text(bad)
        with pytest.raises(ScheduleError):
            parse_schedule(tmp_path / "b.txt", n_row_blocks=4, n_col_blocks=3)


def test_group_beta_uses_numpy_sum():
    tab = _table(seed=4, m=40, n=2)
    ids = np.array([5, 3, 9, 1, 0, 33, 2, 7, 8, 10, 11])
    assert group_beta(tab, 0.7, 1, ids) == 0.7 * float(tab.values[ids, 1].sum()) / \
        float(tab.totals[1])
    bad = ProbabilityTable(np.zeros((3, 2)), np.zeros(2))
    with pytest.raises(ScheduleError):
        group_beta(bad, 1.0, 0, np.array([0]))


# ---------------------------------------------------------------------------
# parameters, partitions, metrics
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kw", [dict(epochs=-1), dict(epochs=1, b=0.0),
                                dict(epochs=1, group_size=0),
                                dict(epochs=1, execution_mode="threaded"),
                                dict(epochs=1, worker_count=0), dict(epochs=1, audit_interval=-1),
                                dict(epochs=1, divergence_factor=0.0)])
def test_solver_params_validation(kw):
    with pytest.raises(ConfigurationError):
        SolverParams(**kw)


@pytest.mark.parametrize("kw", [dict(strategy="stratified"), dict(alpha=0.0), dict(alpha=1.5),
                                dict(gamma=-0.5), dict(theta0=1.2), dict(theta_step=-0.1)])
def test_sampling_config_validation(kw):
    with pytest.raises(ConfigurationError):
        SamplingConfig(**kw)


def test_partitions_match_oracle_layout():
    from oracle.oracle import angle_block_edges, strip_edges
    for key, cfg in CONFIGS.items():
        s = cfg.spec
        np.testing.assert_array_equal(s.angle_edges(), angle_block_edges(s.views, s.m))
        np.testing.assert_array_equal(s.strip_edges(), strip_edges(s.n, s.nc))
        rows = s.row_meas()
        assert rows[0][0] == 0 and rows[-1][-1] == s.n_measurements - 1
        assert sum(r.size for r in rows) == s.n_measurements
        assert sum(v.size for v in s.voxel_indices()) == s.n_voxels
    with pytest.raises(ConfigurationError):
        ParallelBeamSpec(4, 3, 5, 4, 2)


def test_random_ellipses_deterministic():
    a = random_ellipses(32, 5, 0)
    np.testing.assert_array_equal(a, random_ellipses(32, 5, 0))
    assert a.shape == (1024,) and a.min() >= 0 and a.max() > 0
    assert not np.array_equal(a, random_ellipses(32, 5, 1))


def test_trace_csv_roundtrip(tmp_path):
    tr = ConvergenceTrace()
    for e in range(1, 4):
        tr.append(TraceRow(e, 0.5 * e, 1.0 + e, 2.0 * e, 0.1 * e, "parallel", 0.0))
    tr.to_csv(tmp_path / "t.csv")
    back = ConvergenceTrace.from_csv(tmp_path / "t.csv")
    assert [r.snr_db for r in back.rows] == [2.0, 3.0, 4.0]
    assert back.snr_at_effective(1.25) == pytest.approx(3.5)
    assert snr_db([1.0, 0.0], [1.0, 0.0]) == math.inf
    with pytest.raises(ConfigurationError):
        snr_db([0.0], [1.0])


# ---------------------------------------------------------------------------
# C ABI surface (loads without a GPU; no compute calls here)
# ---------------------------------------------------------------------------

def test_library_exports_every_declared_symbol():
    header = open(os.path.join(REPO, "include", "blockct.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char \*)\s*(bct_\w+)\(", header, re.M))
    assert len(declared) >= 30
    L = N.load()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(N.EXPORTED)
    assert L.bct_version() == 2


def test_oracle_is_not_imported_by_the_product():
    pkg = os.path.join(REPO, "paper_1709_00953_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h")):
                text = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f
                assert "libblockct_oracle" not in text, f


def _np_pairwise(a):
    """Restatement of numpy's pairwise_sum (loops_utils.h.src), the order the
    device sampler (csrc/sampler.cu np_pairwise) uses for the betas."""
    n = len(a)
    if n < 8:
        res = 0.0
        for v in a:
            res = res + v
        return res
    if n <= 128:
        r = list(a[:8])
        i = 8
        while i < n - (n % 8):
            for k in range(8):
                r[k] = r[k] + a[i + k]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _np_pairwise(a[:n2]) + _np_pairwise(a[n2:])


def test_numpy_sum_is_the_pairwise_order_of_the_device_sampler():
    rng = np.random.default_rng(0)
    for n in list(range(1, 140)) + [200, 255, 256]:
        for _ in range(5):
            a = rng.random(n) * 10.0 ** rng.integers(-6, 6, n)
            assert _np_pairwise(a) == float(np.sum(a))


def test_vectorised_plan_matches_per_visit_draws_on_random_tables():
    """epoch_plan (one variate stream, a stable sort by (visit, E/w)) equals
    the per-visit loop on random tables with empty columns, zero blocks and
    tied weights, for every strategy and group size; the RNG ends in the same
    state."""
    rs = np.random.default_rng(0)
    checked = 0
    for trial in range(120):
        m, n = int(rs.integers(1, 60)), int(rs.integers(1, 30))
        vals = rs.random((m, n)) * (rs.random((m, n)) > rs.random() * 0.6)
        if rs.random() < 0.3:
            vals[:, rs.integers(0, n)] = 0.0
        vals[rs.random((m, n)) < 0.05] = 0.5
        tab = ProbabilityTable(vals, vals.sum(0))
        if tab.active_cols.size == 0:
            continue
        strategy = ["importance", "random", "mixed"][trial % 3]
        cfg = SamplingConfig(alpha=float(rs.choice([0.1, 0.25, 0.5, 1.0])),
                             gamma=float(rs.choice([0.5, 1.0])), strategy=strategy,
                             theta0=0.2, theta_step=0.3)
        gs = int(rs.integers(1, 9))
        a, b = BlockScheduler(tab, cfg, gs), BlockScheduler(tab, cfg, gs)
        ra, rb = np.random.default_rng(trial), np.random.default_rng(trial)
        for ep in range(1, 5):
            pa, pb = a.epoch_plan(ep, ra), b.epoch_plan_per_visit(ep, rb)
            assert [j for j, _ in pa] == [j for j, _ in pb]
            for (_, ga), (_, gb) in zip(pa, pb):
                assert len(ga) == len(gb)
                for x, y in zip(ga, gb):
                    np.testing.assert_array_equal(x, y)
            a.advance_epoch()
            b.advance_epoch()
        assert ra.random() == rb.random()
        checked += 1
    assert checked > 100
