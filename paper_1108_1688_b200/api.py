"""Python surface of the C-ABI: the reference's solver entry points on B200.

    run(problem, config)            -> (grid, report)   solver.cpp:213-258
    douglas_step(problem, ...)      -> (grid, max_dU)   solver.cpp:81-178
    apply_operator(problem, t, u)   -> F(u)             discretization.cpp:302-364
    thomas_batch(lower, diag, ...)  -> x                solver.cpp:22-57
    batch_run(problems, devices)    -> prices, reports  instruments.cpp:238-266 on GPUs
    Solver                          handle: step/run/reset/grid/spot prices

Errors are raised as the Python analogues of the reference's exceptions with
the reference's messages.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from .problem import ProblemSpec, SolverConfig, problems_to_c, _ptr


class HjmsvError(Exception):
    code = -1


class InvalidArgument(HjmsvError, ValueError):      # std::invalid_argument
    code = A.INVALID_ARGUMENT


class DomainError(HjmsvError, ArithmeticError):     # std::domain_error
    code = A.DOMAIN


class LogicError(HjmsvError):                        # std::logic_error
    code = A.LOGIC


class SolverRuntimeError(HjmsvError, RuntimeError):  # std::runtime_error
    code = -2


class SingularPivot(SolverRuntimeError):
    code = A.SINGULAR_PIVOT


class NonFinite(SolverRuntimeError):
    code = A.NONFINITE


class Diverged(SolverRuntimeError):
    code = A.DIVERGED


class Unsupported(HjmsvError):
    code = A.UNSUPPORTED


class CudaError(HjmsvError, RuntimeError):
    code = A.CUDA_ERROR


_BY_CODE = {c.code: c for c in (InvalidArgument, DomainError, LogicError, SingularPivot, NonFinite,
                                 Diverged, Unsupported, CudaError)}


def _check(code: int):
    if code != A.OK:
        msg = A.load().hjmsv_last_error().decode()
        raise _BY_CODE.get(code, HjmsvError)(msg)


MODES = {"strict": A.MODE_STRICT, "fast": A.MODE_FAST}


def _mode(mode) -> int:
    return MODES[mode] if isinstance(mode, str) else int(mode)


def _cfg(config: Optional[SolverConfig]):
    return (config or SolverConfig()).to_c()


class Solver:
    """A batch of problems (equal dims/steps) resident on one GPU."""

    def __init__(self, problems: Sequence[ProblemSpec] | ProblemSpec,
                 config: Optional[SolverConfig] = None, device: int = 0, mode="fast"):
        if isinstance(problems, ProblemSpec):
            problems = [problems]
        self.lib = A.load()
        self.problems = list(problems)
        self._c = problems_to_c(self.problems)
        self._cfg = _cfg(config)
        h = ctypes.c_void_p()
        _check(self.lib.hjmsv_solver_create(self._c, len(self.problems), ctypes.byref(self._cfg),
                                            device, _mode(mode), ctypes.byref(h)))
        self.h = h
        d = [ctypes.c_int32() for _ in range(5)]
        _check(self.lib.hjmsv_solver_dims(self.h, *[ctypes.byref(x) for x in d]))
        self.nr, self.nv, self.ny, self.count, self.n_steps = (x.value for x in d)

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.hjmsv_solver_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- stepping
    def reset(self):
        _check(self.lib.hjmsv_solver_reset(self.h))

    def step_async(self, steps: int):
        _check(self.lib.hjmsv_solver_step_async(self.h, steps))

    def synchronize(self):
        _check(self.lib.hjmsv_solver_synchronize(self.h))

    def step(self, steps: int = 1):
        _check(self.lib.hjmsv_solver_step(self.h, steps))

    def run(self):
        _check(self.lib.hjmsv_solver_run(self.h))

    # -- readouts
    def report(self, problem: int = 0) -> dict:
        r = A.CReport()
        _check(self.lib.hjmsv_solver_report(self.h, problem, ctypes.byref(r)))
        return r.as_dict()

    def grid(self, problem: int = 0) -> np.ndarray:
        out = np.empty(self.nr * self.nv * self.ny)
        _check(self.lib.hjmsv_solver_get_grid(self.h, problem, _ptr(out)))
        return out.reshape(self.nr, self.nv, self.ny)

    def grids(self) -> np.ndarray:
        """All problems' levels in one device-to-host copy, shape (P, nr, nv, ny)."""
        out = np.empty(self.count * self.nr * self.nv * self.ny)
        _check(self.lib.hjmsv_solver_get_grids(self.h, _ptr(out)))
        return out.reshape(self.count, self.nr, self.nv, self.ny)

    def set_grid(self, problem: int, grid: np.ndarray, step_index: int):
        g = np.ascontiguousarray(grid, dtype=np.float64).reshape(-1)
        _check(self.lib.hjmsv_solver_set_grid(self.h, problem, _ptr(g), step_index))

    def price(self, problem: int, zr: float, zv: float, zy: float) -> float:
        out = ctypes.c_double()
        _check(self.lib.hjmsv_solver_price(self.h, problem, zr, zv, zy, ctypes.byref(out)))
        return out.value

    def spot_prices(self) -> np.ndarray:
        out = np.empty(self.count)
        _check(self.lib.hjmsv_solver_spot_prices(self.h, _ptr(out)))
        return out

    def greeks(self, problem: int = 0, scale_rate: bool = True):
        """extract_greeks (instruments.cpp:90-132) of the current level, on the device;
        scale_rate applies finish()'s rho /= r0 (instruments.cpp:150-152). -> (rho, vega)"""
        rho, vega = np.empty(self.nr * self.nv * self.ny), np.empty(self.nr * self.nv * self.ny)
        _check(self.lib.hjmsv_solver_greeks(self.h, problem, int(scale_rate), _ptr(rho), _ptr(vega)))
        shape = (self.nr, self.nv, self.ny)
        return rho.reshape(shape), vega.reshape(shape)

    def surface(self, problem: int = 0, k: int = 0) -> np.ndarray:
        """write_surface_csv's rows (job.cpp:300-310) at y-slice k: columns r_rate,
        v_variance, price, rho_dprice_dr, vega_dprice_dv; shape (nr*nv, 5)."""
        out = np.empty(self.nr * self.nv * 5)
        _check(self.lib.hjmsv_solver_surface(self.h, problem, k, _ptr(out)))
        return out.reshape(self.nr * self.nv, 5)

    def device_ptr(self, problem: int = 0) -> int:
        p = A.PD()
        _check(self.lib.hjmsv_solver_device_grid(self.h, problem, ctypes.byref(p)))
        return ctypes.cast(p, ctypes.c_void_p).value

    def last_device_ms(self) -> float:
        ms = ctypes.c_double()
        _check(self.lib.hjmsv_solver_last_device_ms(self.h, ctypes.byref(ms)))
        return ms.value

    def kernel_profile(self, steps: int, with_total: bool = False):
        """Per-kernel average ms (device timeline, launched as a first march) and
        algorithmic bytes per launch over `steps` steps; with_total also returns
        the event-timed ms of the whole profiled sequence."""
        K, L = 16, 64
        ms, by = np.zeros(K), np.zeros(K)
        n, nk = ctypes.c_int64(), ctypes.c_int32()
        total = ctypes.c_double()
        names = ctypes.create_string_buffer(K * L)
        _check(self.lib.hjmsv_solver_kernel_timeline(self.h, steps, K, _ptr(ms), _ptr(by),
                                                     ctypes.byref(n), ctypes.byref(nk), names, L,
                                                     ctypes.byref(total)))
        out = []
        for q in range(nk.value):
            nm = names.raw[q * L:(q + 1) * L].split(b"\0", 1)[0].decode()
            if not nm:  # index slot unused by this step variant
                continue
            out.append({"name": nm, "avg_ms": float(ms[q]), "alg_bytes": float(by[q])})
        if with_total:
            return out, n.value, total.value
        return out, n.value

    def last_launches(self) -> int:
        n = ctypes.c_int64()
        _check(self.lib.hjmsv_solver_last_launches(self.h, ctypes.byref(n)))
        return n.value


def run(problem: ProblemSpec, config: Optional[SolverConfig] = None, device: int = 0,
        mode="fast"):
    """run() (solver.cpp:213-258): the t = 0 level and its SolveReport."""
    with Solver([problem], config, device, mode) as s:
        s.run()
        return s.grid(0), s.report(0)


def price(problem: ProblemSpec, config: Optional[SolverConfig] = None, device: int = 0,
          mode="fast") -> float:
    """Spot price after the march (finish(), instruments.cpp:145-149)."""
    with Solver([problem], config, device, mode) as s:
        s.run()
        return float(s.spot_prices()[0])


def apply_operator(problem: ProblemSpec, t: float, u: np.ndarray,
                   config: Optional[SolverConfig] = None, mode="strict") -> np.ndarray:
    lib = A.load()
    p = problem.to_c()
    c = _cfg(config)
    uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    out = np.empty_like(uu)
    _check(lib.hjmsv_apply_operator(ctypes.byref(p), ctypes.byref(c), t, _ptr(uu), _ptr(out),
                                    _mode(mode)))
    return out.reshape(problem.shape)


def douglas_step(problem: ProblemSpec, u: np.ndarray, t_from: float, dt: float,
                 config: Optional[SolverConfig] = None, mode="strict"):
    lib = A.load()
    p = problem.to_c()
    c = _cfg(config)
    uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    out = np.empty_like(uu)
    md = ctypes.c_double()
    _check(lib.hjmsv_douglas_step(ctypes.byref(p), ctypes.byref(c), _ptr(uu), t_from, dt,
                                  _ptr(out), ctypes.byref(md), _mode(mode)))
    return out.reshape(problem.shape), md.value


def thomas_batch(lower, diag, upper, super2, rhs, mode="strict") -> np.ndarray:
    """Batched thomas_solve_inplace (solver.cpp:22-57). mode "strict": the
    reference's Thomas; "fast": pass A's partition solver; "fast_twisted": pass
    B's twisted segment solver (both n <= 512)."""
    lib = A.load()
    if mode == "fast_twisted":
        mode = 2
    lower, diag, upper, rhs = (np.ascontiguousarray(x, dtype=np.float64) for x in (lower, diag, upper, rhs))
    count, n = rhs.shape
    s2 = np.ascontiguousarray(super2, dtype=np.float64).reshape(count)
    x = rhs.copy()
    _check(lib.hjmsv_thomas_batch(n, count, _ptr(lower), _ptr(diag), _ptr(upper), _ptr(s2),
                                  _ptr(x), _mode(mode)))
    return x


def batch_run(problems: Sequence[ProblemSpec], config: Optional[SolverConfig] = None,
              devices: Sequence[int] = (0,), mode="fast", grids: bool = False):
    """caplet_ladder-style fan-out over GPUs: contiguous shards, no inter-GPU traffic."""
    lib = A.load()
    arr = problems_to_c(problems)
    c = _cfg(config)
    devs = (ctypes.c_int32 * len(devices))(*devices)
    prices = np.empty(len(problems))
    reports = (A.CReport * len(problems))()
    g = np.empty(sum(p.size for p in problems)) if grids else None
    code = lib.hjmsv_batch_run(arr, len(problems), ctypes.byref(c), devs, len(devices),
                               _mode(mode), _ptr(prices), reports, _ptr(g))
    reps: List[dict] = [r.as_dict() for r in reports]
    if code != A.OK and code not in (A.SINGULAR_PIVOT, A.NONFINITE, A.DIVERGED):
        _check(code)
    return prices, reps, g


def mc_price(problem: ProblemSpec, n_paths: int = 200000, steps_per_year: int = 96,
             seed: int = 20070423, full_truncation: bool = True, device: int = 0):
    """Monte Carlo validator on the device (simulate_zcb / simulate_caplet,
    montecarlo.cpp:142-160) -> (mean, std_error, n_paths). Counter-based normals:
    a different sample from the reference's mt19937_64 stream (compare within
    standard errors)."""
    lib = A.load()
    cp = problem.to_c()
    cfg = A.CMcConfig(n_paths, steps_per_year, seed, int(full_truncation))
    mean, se, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    _check(lib.hjmsv_mc_price(ctypes.byref(cp), ctypes.byref(cfg), device, ctypes.byref(mean),
                              ctypes.byref(se), ctypes.byref(n)))
    return mean.value, se.value, n.value


def device_count() -> int:
    return int(A.load().hjmsv_device_count())
