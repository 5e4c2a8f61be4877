"""The oracle restatement pinned against the compiled reference's golden vectors.

tests/golden/*.npz were produced by tests/golden/make_golden.py from oracle/_ref
(the unmodified reference sources). The restatement must reproduce them bit
for bit; inputs are regenerated from the seeded generator and fingerprinted.
"""
import json
import os

import numpy as np
import pytest

from paper_1108_1688_b200 import workloads as W
from paper_1108_1688_b200.problem import AxisSpec, mix_seed

from golden.make_golden import CASES, PREFIX, fingerprint, sinh_caplet  # noqa: F401

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(HERE, "meta.json")))

FAST_CASES = ["config0_reduced", "config2_reduced", "config4_batch", "sinh_caplet"]


def load(name):
    return np.load(os.path.join(HERE, f"{name}.npz"))


@pytest.mark.parametrize("name", FAST_CASES + ["config0_full"])
def test_restatement_matches_reference_golden(oracle, name):
    probs = CASES[name]()
    assert [fingerprint(p) for p in probs] == META[name]["fingerprints"], "generator drifted"
    gold = load(name)
    for q, p in enumerate(probs):
        g, rep, code, msg = oracle.run(p)
        assert code == 0, msg
        assert np.array_equal(g, gold["grids"][q]), f"{name}[{q}] grid differs"
        assert oracle.spot_price(p, g) == gold["prices"][q]
        assert rep["last_max_delta"] == gold["max_delta"][q]


def test_config1_prefix_checksum(oracle):
    p = CASES["config1_prefix2"]()[0]
    assert fingerprint(p) == META["config1_prefix2"]["fingerprints"][0]
    g, _, code, _ = oracle.run(p, steps=2)
    gold = load("config1_prefix2")
    assert np.array_equal(np.array([g.sum(), (g * g).sum(), g.min(), g.max()]), gold["checksum"])
    assert np.array_equal(g[::17, ::13, ::11], gold["sample"])


def test_stage_goldens(oracle):
    gold = load("stages")
    p = W.make_problem(2, 2, nr=24, nv=12, ny=16, steps=10)
    assert fingerprint(p) == META["stages"]["fingerprints"][0]
    u = gold["u"]
    assert np.array_equal(oracle.apply_operator(p, p.maturity, u), gold["apply_T"])
    assert np.array_equal(oracle.apply_operator(p, 0.5 * p.maturity, u), gold["apply_mid"])
    dt = p.maturity / 10
    step, md, code, _ = oracle.douglas_step(p, u, p.maturity, dt)
    assert code == 0 and np.array_equal(step, gold["step"]) and md == gold["step_max_delta"][0]
    for axis, (a, b) in enumerate([(3, 5), (4, 7), (5, 6)]):
        lo, di, up, s2 = oracle.assemble_line(p, axis, a, b, 0.5 * p.maturity, 0.5 * dt)
        assert np.array_equal(np.stack([lo, di, up]), gold[f"line{axis}"])
        assert s2 == gold[f"line{axis}_s2"][0]
    x, code, _ = oracle.thomas(gold["th_lower"], gold["th_diag"], gold["th_upper"], gold["th_s2"],
                               gold["th_rhs"])
    assert code == 0 and np.array_equal(x, gold["th_x"])


def test_error_goldens(oracle):
    e = META["errors"]
    pd = W.make_problem(0, 0)
    pd.v = AxisSpec.uniform(0.0, 30.0, 32)
    assert fingerprint(pd) == e["divergence"]["fingerprint"]
    _, rep, code, msg = oracle.run(pd, raise_on_error=False)
    assert (code, msg, rep["failed_step"]) == (e["divergence"]["code"], e["divergence"]["message"],
                                               e["divergence"]["failed_step"])
    pt = W.make_problem(3, 0, nr=4, nv=3, ny=3, steps=2000)
    pt.time_levels = 0
    _, _, code, msg = oracle.run(pt, raise_on_error=False)
    assert (code, msg) == (e["time_bug"]["code"], e["time_bug"]["message"])


def test_known_answers():
    k = META["known"]
    # SPEC.md:52 g_factor(20, 0.001) = 19.801327 (+-1e-6); SPEC.md:59 1.04^-10 = 0.6755642
    assert abs(k["g_factor_20_0.001"] - 19.801327) < 1e-6
    assert abs(k["zcb_flat104_T10"] - 0.6755642) < 1e-7
    assert [mix_seed(0x11081688, s) for s in range(8)] == k["mix_seed"]
