"""Callers of the hot path on the batch engine.

    caplet_ladder(base, strikes)      instruments.cpp:238-266  one caplet per strike
    convergence(make, ...)            job.cpp:381-472          cmd_convergence's table
    reference_caplet(payment, expiry) job.cpp:148-193          the job defaults' caplet
    reference_zcb(maturity)           instruments.cpp:173-208  price_zcb's default (collapsed v)
    bench(cases)                      job.cpp:540-567          cmd_bench's timing table

The reference fans caplet_ladder's strikes over std::threads (each a full
price_caplet); here the strikes share mesh, model, curve and maturity, so they
are one batched solve per GPU (hjmsv_batch_run), returned in input order.
cmd_convergence refines one dimension at a time, so its runs have different
grid shapes; each is its own device solve, in the reference's row order.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from .api import _BY_CODE, HjmsvError, _check, batch_run, price
from .problem import AxisSpec, ProblemSpec, SolverConfig, _ptr

__all__ = ["caplet_ladder", "convergence", "reference_caplet", "reference_zcb", "bench", "PAPER_BENCH_SECONDS"]

# The paper's timing table: caplet, default 100x50x50 mesh,
# 12 steps per year, wall seconds on a Pentium IV 3.2 GHz, keyed by (T_M, T).
PAPER_BENCH_SECONDS = {(2.0, 1.0): 0.9, (11.0, 10.0): 7.3, (20.0, 19.0): 14.0}


def caplet_ladder(base: ProblemSpec, strikes: Sequence[float], config: Optional[SolverConfig] = None,
                  devices: Sequence[int] = (0,), mode: str = "fast") -> List[Tuple[float, float]]:
    """(strike, price) per strike of the caplet `base` (instruments.cpp:238-266).

    A failing strike raises like the reference's worker would (the first failure in
    input order, with its status)."""
    if base.instrument != A.INSTRUMENT_CAPLET:
        raise ValueError("caplet_ladder needs a caplet problem")
    if len(strikes) == 0:
        return []
    probs = [dataclasses.replace(base, strike=float(k)) for k in strikes]
    prices, reps, _ = batch_run(probs, config, devices=devices, mode=mode)
    for k, r in zip(strikes, reps):
        if r["status"] != A.OK:
            raise _BY_CODE.get(r["status"], HjmsvError)(
                f"caplet_ladder: strike {k}: status {A.STATUS_NAMES[r['status']]} at step {r['failed_step']}")
    return [(float(k), float(p)) for k, p in zip(strikes, prices)]


def _zcb_reference(p: ProblemSpec) -> float:
    """price_zcb's reference: zcb_closed_form at the natural spot (x = 0, y = 0) at t = 0,
    i.e. p(0, T) / p(0, 0) (instruments.cpp:180-205, model.cpp:48-54)."""
    cp = p.to_c()  # holds the curve arrays alive for the call
    t, out = np.array([p.maturity]), np.empty(1)
    _check(A.load().hjmsv_curve_eval(ctypes.byref(cp.curve), 0, 1, _ptr(t), _ptr(out)))
    return float(out[0])


def convergence(make: Callable[[int, int, int], ProblemSpec], nr_list: Sequence[int],
                ny_list: Sequence[int], nt_list: Sequence[int], nv_list: Sequence[int] = (),
                base: Tuple[int, int, int] = (0, 0, 0), config: Optional[SolverConfig] = None,
                device: int = 0, mode: str = "fast") -> List[dict]:
    """cmd_convergence's rows (job.cpp:381-472): sweep, nr, nv, ny, steps_per_year,
    value, error_or_delta, plus the 'order' rows from the ZCB mesh errors.

    make(nr, nv, ny) builds the problem on a mesh (its n_steps is ignored: the step
    count is lround(steps_per_year * T), solver.cpp:234-236). `base` is the base
    mesh; the ZCB sweep pairs nr_list with ny_list, caplets refine nr, nv, ny in turn.
    """
    cfg0 = config or SolverConfig()
    rows: List[dict] = []

    def run_one(nr: int, nv: int, ny: int, spy: int):
        p = dataclasses.replace(make(nr, nv, ny), n_steps=0)
        cfg = dataclasses.replace(cfg0, steps_per_year=int(spy))
        value = price(p, cfg, device=device, mode=mode)
        err = abs(value - _zcb_reference(p)) if p.instrument == A.INSTRUMENT_ZCB else 0.0
        return p, value, err

    def emit(sweep, nr, nv, ny, spy, value, err):
        rows.append({"sweep": sweep, "nr": nr, "nv": nv, "ny": ny, "steps_per_year": spy,
                     "value": value, "error_or_delta": err})

    bnr, bnv, bny = base
    spy0 = cfg0.steps_per_year
    is_zcb = make(bnr, bnv, bny).instrument == A.INSTRUMENT_ZCB
    mesh_errors = []
    if is_zcb:  # paired (nr, ny) refinement
        for nr, ny in zip(nr_list, ny_list):
            _, value, err = run_one(nr, bnv, ny, spy0)
            emit("mesh", nr, bnv, ny, spy0, value, err)
            mesh_errors.append(err)
    else:
        def sweep_dim(name, values, mesh_of):
            prev = None
            for n in values:
                nr, nv, ny = mesh_of(int(n))
                _, value, _ = run_one(nr, nv, ny, spy0)
                emit(name, nr, nv, ny, spy0, value, abs(value - prev) if prev is not None else 0.0)
                prev = value
        sweep_dim("nr", nr_list, lambda n: (n, bnv, bny))
        if len(nv_list):
            sweep_dim("nv", nv_list, lambda n: (bnr, n, bny))
        sweep_dim("ny", ny_list, lambda n: (bnr, bnv, n))
    prev = None
    for nt in nt_list:  # time-step sweep on the base mesh
        _, value, err = run_one(bnr, bnv, bny, int(nt))
        emit("nt", bnr, bnv, bny, int(nt), value,
             err if is_zcb else (abs(value - prev) if prev is not None else 0.0))
        prev = value
    for q in range(1, len(mesh_errors)):  # observed spatial order (bond sweeps halve dx)
        ratio = mesh_errors[q - 1] / max(mesh_errors[q], 1e-300)
        rows.append({"sweep": "order", "error_or_delta": math.log2(ratio)})
    return rows


def _discount(p: ProblemSpec, t: float) -> float:
    cp = p.to_c()
    tt, out = np.array([t]), np.empty(1)
    _check(A.load().hjmsv_curve_eval(ctypes.byref(cp.curve), 0, 1, _ptr(tt), _ptr(out)))
    return float(out[0])


def reference_caplet(payment: float, expiry: float, strike: Optional[float] = None) -> ProblemSpec:
    """The caplet an empty job file prices (JobConfig defaults, job.hpp:43-85):
    flat curve 1.04 (curve.cpp:11-20), ModelParams::market_2007 (model.cpp:8-10:
    kappa 0.001, lambda 0.15, gamma 0.9, eps 1.5, theta 0.25, rho -0.75), strike =
    the period forward rate (job.cpp:154-166), mesh MeshSpec::caplet_default
    (instruments.cpp:11-22: 100 x 50 x 50 sinh axes from default_axes, mesh.cpp:94-102,
    r0 = 0.01), and run()'s own step count lround(steps_per_year * T) and time levels
    (solver.cpp:213-258), as price_caplet builds it (instruments.cpp:210-236)."""
    r0 = 0.01
    base = ProblemSpec(r=AxisSpec.uniform(0, 1, 3), v=AxisSpec.uniform(0, 1, 3), y=AxisSpec.uniform(0, 1, 3),
                       kappa=0.001, lam=0.15, gamma=0.9, eps=1.5, theta=0.25, rho=-0.75, maturity=expiry,
                       r0=r0, flat_base=1.04)
    if strike is None:  # period_forward_rate (job.cpp:154-157)
        strike = (_discount(base, expiry) / _discount(base, payment) - 1.0) / (payment - expiry)
    k = strike / r0
    return dataclasses.replace(
        base, r=AxisSpec.sinh(k, 0.05, 0.0, 250.0, 100), v=AxisSpec.sinh(0.5, 0.5, 0.0, 30.0, 50),
        y=AxisSpec.sinh(0.0, 0.05, 0.0, 250.0, 50), instrument=A.INSTRUMENT_CAPLET, payment=payment,
        strike=strike, n_steps=0, time_levels=A.TIME_REFERENCE)


def reference_zcb(maturity: float) -> ProblemSpec:
    """The bond an empty job file prices with instrument = zcb: flat curve 1.04,
    ModelParams::market_2007, MeshSpec::zcb_default(f(0,0), r0 = 0.01)
    (instruments.cpp:24-35: 100 sinh r nodes centred on the spot rate, 40 sinh y
    nodes) and price_zcb's collapsed v axis (the singleton v = 0 plane,
    instruments.cpp:140-143) — a 100 x 1 x 40 grid, run()'s own step count and
    time levels."""
    r0 = 0.01
    base = ProblemSpec(r=AxisSpec.uniform(0, 1, 3), v=AxisSpec.singleton(0.0), y=AxisSpec.uniform(0, 1, 3),
                       kappa=0.001, lam=0.15, gamma=0.9, eps=1.5, theta=0.25, rho=-0.75, maturity=maturity,
                       r0=r0, flat_base=1.04)
    cp = base.to_c()
    t, f0 = np.array([0.0]), np.empty(1)
    _check(A.load().hjmsv_curve_eval(ctypes.byref(cp.curve), 1, 1, _ptr(t), _ptr(f0)))  # forward(0)
    return dataclasses.replace(base, r=AxisSpec.sinh(float(f0[0]) / r0, 0.05, 0.0, 25.0, 100),
                               y=AxisSpec.sinh(0.0, 0.5, 0.0, 250.0, 40), n_steps=0,
                               time_levels=A.TIME_REFERENCE)


def bench(cases: Sequence[Tuple[float, float]] = ((2.0, 1.0), (11.0, 10.0), (20.0, 19.0)),
          config: Optional[SolverConfig] = None, device: int = 0, mode: str = "fast",
          warmup: bool = True) -> List[dict]:
    """cmd_bench's rows (job.cpp:540-567): for each (payment, expiry) case the job
    defaults' caplet priced end to end — lowering, terminal level + smoothing,
    the march, the spot readout — with its wall time, beside the paper's figure.
    warmup: one untimed solve first, so the device context and memory pool are
    not charged to the first case."""
    import time
    from .api import Solver
    if warmup:
        with Solver([reference_caplet(*cases[0])], config, device, mode) as s:
            s.step(1)
    rows = []
    for payment, expiry in cases:
        p = reference_caplet(payment, expiry)
        t0 = time.perf_counter()
        with Solver([p], config, device, mode) as s:
            s.run()
            value = float(s.spot_prices()[0])
            n_steps = s.n_steps
        wall = time.perf_counter() - t0
        rows.append({"payment_years": payment, "expiry_years": expiry, "n_steps": n_steps,
                     "wall_seconds": wall, "price": value,
                     "paper_seconds": PAPER_BENCH_SECONDS.get((float(payment), float(expiry)))})
    return rows
