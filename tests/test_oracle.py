"""Oracle checks on CPU: the restatement vs the live compiled reference (when
oracle/_ref exists) and the SPEC.md known-answer properties of the path."""
import numpy as np
import pytest

from paper_1108_1688_b200 import workloads as W
from paper_1108_1688_b200.problem import AxisSpec, ProblemSpec


@pytest.mark.parametrize("cfg,idx,kw", [
    (0, 5, dict(nr=20, nv=10, ny=12, steps=25)),
    (2, 7, dict(nr=20, nv=10, ny=12, steps=25)),
    (4, 9, dict(nr=20, nv=10, ny=12, steps=25)),
    (3, 0, dict(nr=20, nv=10, ny=12, steps=25)),
])
def test_restatement_bitexact_vs_reference(oracle, reference, cfg, idx, kw):
    p = W.make_problem(cfg, idx, **kw)
    g0, r0, c0, m0 = oracle.run(p)
    g1, r1, c1, m1 = reference.run(p)
    assert np.array_equal(g0, g1)
    assert r0["last_max_delta"] == r1["last_max_delta"]
    assert oracle.spot_price(p, g0) == reference.spot_price(p, g1)


def test_reference_time_levels_bitexact(oracle, reference):
    p = W.make_problem(2, 4, nr=16, nv=8, ny=8, steps=40)
    p.time_levels = 0  # run()'s repeated subtraction
    assert np.array_equal(oracle.run(p)[0], reference.run(p)[0])
    p.n_steps = 0      # run()'s own lround(steps_per_year * T) step count, via hjmsv::run itself
    assert np.array_equal(oracle.run(p)[0], reference.run(p)[0])


def test_first_and_second_order_boundaries(oracle, reference):
    from paper_1108_1688_b200.problem import SolverConfig
    p = W.make_problem(4, 3, nr=16, nv=8, ny=10, steps=20)
    for yo in (1, 2):
        for ro in (1, 2):
            cfg = SolverConfig(y_boundary_order=yo, r_boundary_order=ro, theta_cn=0.6, smoothing=yo == 2)
            assert np.array_equal(oracle.run(p, cfg)[0], reference.run(p, cfg)[0])


def test_host_helpers_bitexact(oracle, reference):
    assert all(np.array_equal(a, b) for a, b in zip(oracle.sinh_axis(3.0, 0.05, 0, 250, 50),
                                                    reference.sinh_axis(3.0, 0.05, 0, 250, 50)))
    p = W.make_problem(2, 0)
    t = np.linspace(-0.0, 35.0, 301)
    for what in (0, 1, 2):
        assert np.array_equal(oracle.curve_eval(p, what, t), reference.curve_eval(p, what, t))


def test_thomas_known_answers(oracle):
    """identity line; (-1,2,-1) round trip 1e-12; random dd vs dense < 1e-11."""
    n = 50
    rhs = np.arange(1.0, n + 1)[None, :]
    x, code, _ = oracle.thomas(np.zeros((1, n)), np.ones((1, n)), np.zeros((1, n)), np.zeros(1), rhs)
    assert code == 0 and np.array_equal(x, rhs)
    lo, di, up = -np.ones((1, n)), 2 * np.ones((1, n)), -np.ones((1, n))
    lo[0, 0] = up[0, -1] = 0
    xt = np.sin(np.arange(n))[None, :]
    A = np.diag(di[0]) + np.diag(lo[0, 1:], -1) + np.diag(up[0, :-1], 1)
    x, code, _ = oracle.thomas(lo, di, up, np.zeros(1), (A @ xt[0])[None, :])
    assert np.max(np.abs(x - xt)) < 1e-12
    rng = np.random.default_rng(1)
    lo, up = rng.uniform(-1, 1, (1, n)), rng.uniform(-1, 1, (1, n))
    di = 2.5 + rng.uniform(0, 1, (1, n))
    lo[0, 0] = up[0, -1] = 0
    b = rng.standard_normal(n)
    A = np.diag(di[0]) + np.diag(lo[0, 1:], -1) + np.diag(up[0, :-1], 1)
    x, code, _ = oracle.thomas(lo, di, up, np.zeros(1), b[None, :])
    assert np.max(np.abs(x[0] - np.linalg.solve(A, b))) < 1e-11


def test_thomas_super2_fold_matches_dense(oracle):
    """The (0,2) entry folded against row 1 (solver.cpp:28-40) solves the full system."""
    rng = np.random.default_rng(2)
    n = 12
    lo, up = rng.uniform(-1, 1, (1, n)), rng.uniform(-1, 1, (1, n))
    di = 3 + rng.uniform(0, 1, (1, n))
    lo[0, 0] = up[0, -1] = 0
    s2 = 0.4
    A = np.diag(di[0]) + np.diag(lo[0, 1:], -1) + np.diag(up[0, :-1], 1)
    A[0, 2] = s2
    b = rng.standard_normal(n)
    x, code, _ = oracle.thomas(lo, di, up, np.array([s2]), b[None, :])
    assert np.max(np.abs(x[0] - np.linalg.solve(A, b))) < 1e-12


def test_zcb_flat_curve_acceptance(oracle):
    """flat 4% ZCB, T=20, 100x40 (r x y), 12 steps/yr: |err| < 1e-5."""
    import math
    spot = math.log(1.04)
    from paper_1108_1688_b200 import _abi as A
    rax = AxisSpec.sinh(spot / 0.01, 0.05, 0.0, 25.0, 100)    # MeshSpec::zcb_default (instruments.cpp:24-35)
    yax = AxisSpec.sinh(0.0, 0.5, 0.0, 250.0, 40)
    p = ProblemSpec(r=rax, v=AxisSpec.singleton(0.0), y=yax, kappa=0.001, lam=0.15, gamma=0.9, eps=1.5,
                    theta=0.25, rho=-0.75, maturity=20.0, flat_base=1.04, n_steps=0,
                    time_levels=A.TIME_REFERENCE)
    g, rep, code, msg = oracle.run(p)
    assert code == 0, msg
    price = oracle.interpolate(p, g, spot / 0.01, 0.0, 0.0)
    assert rep["n_steps"] == 240
    assert abs(price - 1.04 ** -20) < 1e-5


def test_divergence_reported_with_step(oracle):
    p = W.make_problem(0, 0, nr=24, nv=24, ny=8, steps=200)
    p.v = AxisSpec.uniform(0.0, 30.0, 24)
    _, rep, code, msg = oracle.run(p, raise_on_error=False)
    if code:
        assert code in (3, 4) and msg.startswith(f"step {rep['failed_step']}/200: ")


def test_greeks_restatement_bitexact_vs_reference(oracle, reference):
    """extract_greeks (instruments.cpp:90-132) + finish()'s rho /= r0 on a solved
    sinh-mesh caplet level: restatement == reference, bit for bit."""
    p = W.make_problem(2, 2, nr=18, nv=9, ny=11, steps=15)
    p.r = AxisSpec.sinh(p.strike / p.r0, 0.05, 0.0, 250.0, 18)
    p.v = AxisSpec.sinh(0.5, 0.5, 0.0, 30.0, 9)
    g, _, _, _ = reference.run(p)
    for scale in (True, False):
        r0_, v0_ = oracle.greeks(p, g, scale)
        r1_, v1_ = reference.greeks(p, g, scale)
        assert np.array_equal(r0_, r1_) and np.array_equal(v0_, v1_)


@pytest.mark.parametrize("cfg,idx", [(0, 2), (2, 5), (4, 1)])
def test_model_functions_bitexact_vs_reference(oracle, reference, cfg, idx):
    """Time-dependent lambda(t), gamma(t), eps(t) (model.hpp:22-24): the
    restatement evaluates them at every step's half level exactly as
    HjmCoefficientField::prepare does (discretization.cpp:40-54)."""
    p = W.with_model_functions(W.make_problem(cfg, idx, nr=20, nv=10, ny=12, steps=25))
    g0, r0, c0, _ = oracle.run(p)
    g1, r1, c1, _ = reference.run(p)
    assert c0 == c1 == 0
    assert np.array_equal(g0, g1)
    assert r0["last_max_delta"] == r1["last_max_delta"]
    # and the model functions matter
    q = W.make_problem(cfg, idx, nr=20, nv=10, ny=12, steps=25)
    assert not np.array_equal(g0, oracle.run(q)[0])


def test_constant_model_functions_equal_constants(oracle, reference):
    """Functions that return the constants give the constant model bit for bit."""
    p = W.make_problem(2, 3, nr=16, nv=8, ny=10, steps=20)
    g_const = oracle.run(p)[0]
    lam, gam, eps = p.lam, p.gamma, p.eps
    p.lambda_fn, p.gamma_fn, p.eps_fn = (lambda t: lam), (lambda t: gam), (lambda t: eps)
    assert np.array_equal(oracle.run(p)[0], g_const)
    assert np.array_equal(reference.run(p)[0], g_const)


def test_model_function_validation(oracle, reference):
    """ModelParams::validate checks gamma_fn(0) in (0,1] (model.cpp:36-37)."""
    p = W.make_problem(0, 0, nr=12, nv=6, ny=6, steps=4)
    p.gamma_fn = lambda t: 1.5 if t == 0.0 else 0.9
    for lib in (oracle, reference):
        g, rep, code, msg = lib.run(p, raise_on_error=False)
        assert code == 1 and "gamma must lie in (0,1]" in msg
