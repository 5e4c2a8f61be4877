"""Per-line parity of the FAST tridiagonal solvers on the worst-conditioned lines.

tests/golden/lines.npz (tests/golden/make_line_golden.py) holds lines assembled
by the reference's assemble_line_r/v/y (discretization.cpp:194-300) and their
solutions by the reference's thomas_solve_inplace (solver.cpp:22-57): config 4's
least diagonally dominant lines (y-line ratio (|l|+|u|)/|d| up to 3.94), the
super2 fold's lag branch (solver.cpp:36-39), and config 3's 512-row r-lines and
256-row y-lines (32- and 16-segment reduced systems). The device solves them
with the same device functions the march uses: "fast" = pass A's partition
solver (seg_solve + lane-scan reduced system), "fast_twisted" = pass B's twisted
segment solve; "strict" = the reference's sequential Thomas.
Bar: per line max|x - x_ref| <= TOL * max|x_ref| — the partition method only
reorders the elimination (the north star's allowed difference).
"""
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GROUPS = ["c4r", "c4v", "c4y", "lag", "c3r", "c3y"]
TOL = {"strict": 1e-15, "fast": 1e-13, "fast_twisted": 1e-13}


def load():
    return dict(np.load(os.path.join(HERE, "lines.npz")))


def line_err(x, ref):
    return np.max(np.abs(x - ref), axis=1) / np.max(np.abs(ref), axis=1)


@pytest.mark.parametrize("group", GROUPS)
def test_restatement_matches_reference_lines(oracle, group):
    """The C restatement's Thomas (the oracle) reproduces the golden lines bit for bit."""
    d = load()
    x, code, _ = oracle.thomas(d[f"{group}_lower"], d[f"{group}_diag"], d[f"{group}_upper"],
                               d[f"{group}_s2"], d[f"{group}_rhs"])
    assert code == 0
    assert np.array_equal(x, d[f"{group}_x"])


def test_golden_lines_are_hard():
    d = load()
    assert d["c4y_ratio"].max() > 3.0          # not diagonally dominant
    assert d["c4r_ratio"].max() > 0.99
    assert d["lag_upper"][0, 1] == 0.0 and d["lag_s2"][0] != 0.0
    assert d["c3r_x"].shape[1] == 512 and d["c3y_x"].shape[1] == 256


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["strict", "fast", "fast_twisted"])
@pytest.mark.parametrize("group", GROUPS)
def test_device_lines(gpu, group, mode):
    import paper_1108_1688_b200 as hj
    d = load()
    x = hj.thomas_batch(d[f"{group}_lower"], d[f"{group}_diag"], d[f"{group}_upper"], d[f"{group}_s2"],
                        d[f"{group}_rhs"], mode=mode)
    err = line_err(x, d[f"{group}_x"])
    print(f"{group} {mode}: worst line rel err {err.max():.2e}")
    assert err.max() <= TOL[mode], f"{group} {mode}: {err.max():.3e}"
