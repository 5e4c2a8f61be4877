"""Seeded synthetic workloads of BASELINE.json's five configs.

No public benchmark or dataset is involved: every model parameter, curve and
instrument is drawn from the reference's splitmix64 (`mix_seed`,
montecarlo.cpp:12-17) with root = 0x11081688 ^ config_id and stream =
problem_index*64 + draw_index, draw order kappa, theta_v, eps, rho, sigma0,
a, b, c, kind, T, K. Builder decisions recorded in DESIGN.md: gamma = 0.9,
v(0) = 1, lambda = sigma0 / a^gamma; uniform axes r~ in [0,25], v in [0,1.5],
y~ in [0,250], r0 = 0.01; time levels t_s = T - s*dt; config 2
prices caplets only (floorlets are not in the reference).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List

from . import _abi as A
from .problem import AxisSpec, ProblemSpec, SolverConfig, curve_nodes, uniform_draw

R_MAX, V_MAX, Y_MAX, R0, GAMMA = 25.0, 1.5, 250.0, 0.01, 0.9


@dataclass(frozen=True)
class ConfigShape:
    config_id: int
    nr: int
    nv: int
    ny: int
    steps: int
    problems: int
    description: str


CONFIGS = {
    0: ConfigShape(0, 64, 32, 32, 200, 1, "ZCB T=5, 64x32x32, 200 steps"),
    1: ConfigShape(1, 256, 128, 128, 1000, 1, "ZCB T=5, 256x128x128, 1000 steps"),
    2: ConfigShape(2, 128, 64, 64, 500, 64, "64 caplets T~U[1,10], 128x64x64, 500 steps"),
    3: ConfigShape(3, 512, 256, 256, 2000, 1, "ZCB T=10 rho=-0.9, 512x256x256, 2000 steps"),
    4: ConfigShape(4, 64, 32, 32, 200, 1024, "1024 ZCB/caplet mix T~U[1,10], 64x32x32, 200 steps"),
}


def _u(root: int, p: int, d: int, lo: float, hi: float) -> float:
    return lo + (hi - lo) * uniform_draw(root, p * 64 + d)


def make_problem(config_id: int, index: int, nr: int | None = None, nv: int | None = None,
                 ny: int | None = None, steps: int | None = None) -> ProblemSpec:
    """Problem `index` of config `config_id`; dims/steps may be overridden for
    reduced-size parity cases (same draws, smaller grid)."""
    cs = CONFIGS[config_id]
    nr, nv, ny = nr or cs.nr, nv or cs.nv, ny or cs.ny
    steps = steps or cs.steps
    root = 0x11081688 ^ config_id
    kappa = _u(root, index, 0, 0.01, 0.2)
    theta_v = _u(root, index, 1, 0.5, 3.0)
    eps = _u(root, index, 2, 0.1, 0.6)
    rho = _u(root, index, 3, -0.7, 0.7)
    sigma0 = _u(root, index, 4, 0.005, 0.02)
    a = _u(root, index, 5, 0.01, 0.03)
    b = _u(root, index, 6, 0.0, 0.03)
    c = _u(root, index, 7, 0.1, 1.0)
    if config_id == 3:
        rho = -0.9
    lam = sigma0 / math.pow(a, GAMMA)
    mats, disc = curve_nodes(a, b, c)
    instrument, T, payment, strike = A.INSTRUMENT_ZCB, 5.0, 0.0, 0.0
    if config_id == 3:
        T = 10.0
    if config_id in (2, 4):
        kind_u = uniform_draw(root, index * 64 + 8)
        T = _u(root, index, 9, 1.0, 10.0)
        strike = _u(root, index, 10, 0.01, 0.06)
        if config_id == 2 or kind_u >= 0.5:
            instrument, payment = A.INSTRUMENT_CAPLET, T + 0.25
    return ProblemSpec(
        r=AxisSpec.uniform(0.0, R_MAX, nr), v=AxisSpec.uniform(0.0, V_MAX, nv),
        y=AxisSpec.uniform(0.0, Y_MAX, ny), kappa=kappa, lam=lam, gamma=GAMMA, eps=eps,
        theta=theta_v, rho=rho, maturity=T, r0=R0, curve_maturities=mats, curve_discounts=disc,
        instrument=instrument, payment=payment, strike=strike, n_steps=steps,
        time_levels=A.TIME_INDEXED)


def make_config(config_id: int, count: int | None = None, **overrides) -> List[ProblemSpec]:
    cs = CONFIGS[config_id]
    n = cs.problems if count is None else count
    return [make_problem(config_id, q, **overrides) for q in range(n)]


def solver_config() -> SolverConfig:
    """SolverConfig defaults (solver.hpp:10-20): theta 0.5, orders 2, smoothing m=3, bound 1e6."""
    return SolverConfig()


def with_model_functions(p: ProblemSpec, amp: float = 0.3) -> ProblemSpec:
    """The same problem with deterministic time-dependent model functions in
    place of the constants (ModelParams::lambda_fn / gamma_fn / eps_fn,
    model.hpp:22-24): a periodic volatility level, a drifting elasticity and a
    decaying vol-of-variance around the drawn values. Not a BASELINE config —
    the parity case for prepare(t)'s per-step evaluation (discretization.cpp:40-54)."""
    lam0, gam0, eps0 = p.lam, p.gamma, p.eps
    p.lambda_fn = lambda t: lam0 * (1.0 + amp * math.sin(2.0 * t))
    p.gamma_fn = lambda t: gam0 - 0.05 * (1.0 - math.cos(t))
    p.eps_fn = lambda t: eps0 * math.exp(-0.1 * t)
    return p
