"""Monte Carlo validator (montecarlo.cpp:38-160): the device
path simulation vs the reference's own Monte Carlo. The generators differ
(counter-based Philox on the device, the reference's mt19937_64 stream per
8192-path batch), so parity is statistical: means agree within 4 combined
standard errors, and the ZCB estimate brackets the input discount p(0,T)."""
import math

import numpy as np
import pytest

import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import workloads as W


def test_reference_mc_zcb_brackets_discount(reference):
    p = W.make_problem(0, 2, nr=8, nv=4, ny=4, steps=4)
    p.maturity = 2.0
    mean, se, n = reference.mc_price(p, n_paths=20000, steps_per_year=24)
    disc = reference.curve_eval(p, 0, np.array([p.maturity]))[0]
    assert n == 20000 and se > 0
    assert abs(mean - disc) <= 4 * se + 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("cfg_id,idx", [(0, 1), (2, 3), (4, 7)])
def test_device_mc_matches_reference_mc(gpu, reference, cfg_id, idx):
    p = W.make_problem(cfg_id, idx, nr=8, nv=4, ny=4, steps=4)
    m_d, se_d, n_d = hj.mc_price(p, n_paths=100000, steps_per_year=48)
    m_r, se_r, n_r = reference.mc_price(p, n_paths=100000, steps_per_year=48)
    assert n_d == n_r == 100000
    tol = 4 * math.sqrt(se_d ** 2 + se_r ** 2)
    assert abs(m_d - m_r) <= tol, f"{m_d} vs {m_r} (tol {tol:.2e})"
    assert abs(se_d - se_r) <= 0.1 * se_r  # same variance of the estimator


@pytest.mark.gpu
def test_device_mc_deterministic_and_zcb_discount(gpu, reference):
    p = W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=4)
    a = hj.mc_price(p, n_paths=300000, steps_per_year=96)
    b = hj.mc_price(p, n_paths=300000, steps_per_year=96)
    assert a == b
    disc = reference.curve_eval(p, 0, np.array([p.maturity]))[0]
    assert abs(a[0] - disc) <= 4 * a[1] + 1e-4


@pytest.mark.gpu
def test_device_mc_model_functions(gpu, reference):
    """run_path evaluates lambda(t), gamma(t), eps(t) at every step's start
    (montecarlo.cpp:54-58); the device reads them from the per-step table."""
    # the reference calls the (Python) model functions once per path and step:
    # a bounded sample keeps that to a few million callbacks
    p = W.with_model_functions(W.make_problem(0, 3, nr=8, nv=4, ny=4, steps=4), amp=0.5)
    m_d, se_d, _ = hj.mc_price(p, n_paths=20000, steps_per_year=24)
    m_r, se_r, _ = reference.mc_price(p, n_paths=20000, steps_per_year=24)
    tol = 4 * math.sqrt(se_d ** 2 + se_r ** 2)
    assert abs(m_d - m_r) <= tol, f"{m_d} vs {m_r} (tol {tol:.2e})"
