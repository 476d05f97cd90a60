"""Whole-system baselines (solvers.py:283-379).

CPU: the oracle restatement (oracle/oracle.py oracle_row_action /
oracle_column_action) is pinned bitwise against the reference's own outputs
(tests/golden/baselines.npz, made by make_golden_baselines.py), and
BaselineParams validates like the reference (test_solvers.py:244-251).
GPU: the device sweeps (csrc/baseline.cu through bct_baseline_*) against the
same fixtures -- bitwise in FP64 -- on the config-1 parallel-beam system and
the reference tests' 12x12 fan-beam system."""

import numpy as np
import pytest
from conftest import fixture_system_arrays, golden
from test_oracle_pins import fixture_oracle

from oracle.oracle import OracleSystem, oracle_column_action, oracle_row_action
from paper_1709_00953_b200 import (CONFIGS, BaselineParams, ConfigurationError,
                                   DeviceBlockSystem, run_column_action, run_row_action)

RULES = ("identity", "sum_inverse", "norm_inverse")


def _omega(f, tag, kind, rule):
    return float(f[f"{tag}_omega_{kind}"][RULES.index(rule)])


def test_baseline_params_validation():
    with pytest.raises(ConfigurationError):
        BaselineParams(epochs=-1)
    with pytest.raises(ConfigurationError):
        BaselineParams(epochs=1, omega=0.0)
    with pytest.raises(ConfigurationError):
        BaselineParams(epochs=1, m_rule="jacobi")
    assert BaselineParams(epochs=0).m_rule == "norm_inverse"


@pytest.fixture(scope="module")
def cfg1_oracle():
    s = CONFIGS[1].spec
    return OracleSystem.parallel_beam(s.n, s.views, s.bins, s.m, s.nc)


@pytest.mark.parametrize("rule", RULES)
def test_oracle_row_action_pinned(cfg1_oracle, rule):
    f = golden("baselines.npz")
    x, _ = oracle_row_action(cfg1_oracle, f["cfg1_y"], 5, _omega(f, "cfg1", "row", rule), rule)
    np.testing.assert_array_equal(x, f[f"cfg1_row_{rule}_x"])
    fan = golden("fan12.npz")
    x, _ = oracle_row_action(fixture_oracle(fan), fan["y"], 5,
                             _omega(f, "fan12", "row", rule), rule)
    np.testing.assert_array_equal(x, f[f"fan12_row_{rule}_x"])


@pytest.mark.parametrize("rule", RULES)
def test_oracle_column_action_pinned(cfg1_oracle, rule):
    f = golden("baselines.npz")
    x, r = oracle_column_action(cfg1_oracle, f["cfg1_y"], 5, _omega(f, "cfg1", "col", rule),
                                rule)
    np.testing.assert_array_equal(x, f[f"cfg1_col_{rule}_x"])
    # the maintained residual matches a fresh evaluation (test_solvers.py:299)
    np.testing.assert_allclose(f["cfg1_y"] - cfg1_oracle.to_scipy() @ x, r, atol=1e-8)
    fan = golden("fan12.npz")
    x, _ = oracle_column_action(fixture_oracle(fan), fan["y"], 5,
                                _omega(f, "fan12", "col", rule), rule)
    np.testing.assert_array_equal(x, f[f"fan12_col_{rule}_x"])


# ---------------------------------------------------------------------------
# device
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def dev_cfg1():
    return DeviceBlockSystem.parallel_beam(CONFIGS[1].spec, dtype="f64")


@pytest.fixture(scope="module")
def dev_fan12():
    fan = golden("fan12.npz")
    panels, rows, vidx, table, nm, nv = fixture_system_arrays(fan)
    return DeviceBlockSystem.from_panels(panels, rows, vidx, table, nm, nv, dtype="f64")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["row", "col"])
@pytest.mark.parametrize("rule", RULES)
def test_device_baselines_match_reference(dev_cfg1, dev_fan12, kind, rule):
    f = golden("baselines.npz")
    fan = golden("fan12.npz")
    run = run_row_action if kind == "row" else run_column_action
    for tag, sysm, y, xt in (("cfg1", dev_cfg1, f["cfg1_y"], None),
                             ("fan12", dev_fan12, fan["y"], fan["x_true"])):
        p = BaselineParams(epochs=5, omega=_omega(f, tag, kind, rule), m_rule=rule)
        x, tr = run(sysm, y, p, x_true=xt)
        np.testing.assert_array_equal(x, f[f"{tag}_{kind}_{rule}_x"])
        assert len(tr) == 5
        assert tr.rows[-1].mode == ("row_action" if kind == "row" else "column_action")
        assert tr.rows[-1].effective_epoch == 5.0
        np.testing.assert_allclose([r.obs_gap_db for r in tr.rows], f[f"{tag}_{kind}_{rule}_gap"],
                                   rtol=1e-9)
        if xt is not None:
            np.testing.assert_allclose([r.snr_db for r in tr.rows],
                                       f[f"{tag}_{kind}_{rule}_snr"], rtol=1e-9)


@pytest.mark.gpu
def test_device_baseline_zero_epochs_and_rerun(dev_fan12):
    """epochs=0 returns x = 0 and an empty trace; a second run restarts from 0."""
    fan = golden("fan12.npz")
    x, tr = run_row_action(dev_fan12, fan["y"], BaselineParams(epochs=0))
    assert len(tr) == 0 and not np.any(x)
    p = BaselineParams(epochs=2, omega=0.5, m_rule="sum_inverse")
    x1, _ = run_column_action(dev_fan12, fan["y"], p)
    x2, _ = run_column_action(dev_fan12, fan["y"], p)
    np.testing.assert_array_equal(x1, x2)
