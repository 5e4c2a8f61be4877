"""Callers of the hot path on the batch engine.

    caplet_ladder(base, strikes)      instruments.cpp:238-266  one caplet per strike
    convergence(make, ...)            job.cpp:381-472          cmd_convergence's table

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
from .problem import ProblemSpec, SolverConfig, _ptr

__all__ = ["caplet_ladder", "convergence"]


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
