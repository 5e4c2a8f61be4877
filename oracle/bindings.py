"""ctypes access to the parity checkers — TEST INFRASTRUCTURE ONLY.

    restatement()  oracle/lib/liboracle.so   plain-C restatement (hjmsv_oracle.c)
    reference()    oracle/_ref/libhjmsv_ref.so  the unmodified reference sources +
                   ref_driver.cpp, built here by oracle/Makefile (None if absent)

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
arm import this module. Both libraries take the framework's plain-data problem
(include/hjmsv_b200.h), so the checker and the checked see identical inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_uint64
from typing import Optional

import numpy as np

from paper_1108_1688_b200 import _abi as A
from paper_1108_1688_b200.problem import ProblemSpec, SolverConfig, problems_to_c, _ptr

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhjmsv_ref.so")
PD = A.PD


def build(reference: bool = True) -> None:
    """Build the checkers (reference only where /root/reference exists)."""
    target = "all"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


class Checker:
    """One checker library (prefix 'oracle_' or 'ref_')."""

    def __init__(self, path: str, prefix: str):
        self.path, self.prefix = path, prefix
        self.lib = ctypes.CDLL(path)
        P, C, R = POINTER(A.CProblem), POINTER(A.CSolverConfig), POINTER(A.CReport)
        sig = {
            "last_error": (ctypes.c_char_p, []),
            "uniform_axis": (c_int, [c_double, c_double, c_int, PD, PD, PD]),
            "sinh_axis": (c_int, [c_double, c_double, c_double, c_double, c_int, PD, PD, PD, PD]),
            "curve_eval": (c_int, [POINTER(A.CCurve), c_int, c_int, PD, PD]),
            "zcb_closed_form": (c_int, [POINTER(A.CCurve), c_double, c_double, c_double, c_double, c_double, PD]),
            "initial_level": (c_int, [P, C, PD]),
            "run": (c_int, [P, C, c_int, PD, R]),
            "douglas_step": (c_int, [P, C, PD, c_double, c_double, PD, PD, PD]),
            "apply_operator": (c_int, [P, C, c_double, PD, PD]),
            "assemble_line": (c_int, [P, C, c_int, c_int, c_int, c_double, c_double, PD, PD, PD, PD]),
            "thomas": (c_int, [c_int, c_int, PD, PD, PD, PD, PD]),
            "interpolate": (c_int, [P, PD, c_double, c_double, c_double, PD]),
            "spot_price": (c_int, [P, PD, PD]),
            "batch_run": (c_int, [P, c_int, C, c_int, PD, R]),
            "extract_greeks": (c_int, [P, PD, c_int, PD, PD]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype, fn.argtypes = res, args
        if prefix == "ref_":
            self.lib.ref_session_create.restype = ctypes.c_void_p
            self.lib.ref_session_create.argtypes = [P, C]
            self.lib.ref_session_steps.restype = c_int
            self.lib.ref_session_steps.argtypes = [ctypes.c_void_p, c_int, PD]
            self.lib.ref_session_destroy.restype = None
            self.lib.ref_session_destroy.argtypes = [ctypes.c_void_p]
            self.lib.ref_mix_seed.restype = c_uint64
            self.lib.ref_mix_seed.argtypes = [c_uint64, c_uint64]
            self.lib.ref_mc_price.restype = c_int
            self.lib.ref_mc_price.argtypes = [P, POINTER(A.CMcConfig), c_int, PD, PD,
                                              POINTER(ctypes.c_longlong)]
            self.lib.ref_g_factor.restype = c_int
            self.lib.ref_g_factor.argtypes = [c_double, c_double, PD]

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def error(self) -> str:
        return self._f("last_error")().decode()

    def _chk(self, code: int):
        if code:
            raise RuntimeError(f"[{A.STATUS_NAMES[code]}] {self.error()}")

    def run(self, p: ProblemSpec, cfg: Optional[SolverConfig] = None, steps: int = -1,
            raise_on_error: bool = True):
        cp, cc = p.to_c(), (cfg or SolverConfig()).to_c()
        g = np.empty(p.size)
        rep = A.CReport()
        code = self._f("run")(ctypes.byref(cp), ctypes.byref(cc), steps, _ptr(g), ctypes.byref(rep))
        if raise_on_error:
            self._chk(code)
        return g.reshape(p.shape), rep.as_dict(), code, (self.error() if code else "")

    def session(self, p: ProblemSpec, cfg: Optional[SolverConfig] = None) -> "RefSession":
        """Resumable reference march (setup once, then timed douglas_step loops)."""
        return RefSession(self, p, cfg)

    def initial_level(self, p: ProblemSpec, cfg: Optional[SolverConfig] = None):
        cp, cc = p.to_c(), (cfg or SolverConfig()).to_c()
        g = np.empty(p.size)
        self._chk(self._f("initial_level")(ctypes.byref(cp), ctypes.byref(cc), _ptr(g)))
        return g.reshape(p.shape)

    def douglas_step(self, p: ProblemSpec, u, t_from, dt, cfg: Optional[SolverConfig] = None):
        cp, cc = p.to_c(), (cfg or SolverConfig()).to_c()
        uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        out = np.empty_like(uu)
        md, tn = c_double(), c_double()
        code = self._f("douglas_step")(ctypes.byref(cp), ctypes.byref(cc), _ptr(uu), t_from, dt,
                                       _ptr(out), ctypes.byref(md), ctypes.byref(tn))
        return out.reshape(p.shape), md.value, code, (self.error() if code else "")

    def apply_operator(self, p: ProblemSpec, t, u, cfg: Optional[SolverConfig] = None):
        cp, cc = p.to_c(), (cfg or SolverConfig()).to_c()
        uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        out = np.empty_like(uu)
        self._chk(self._f("apply_operator")(ctypes.byref(cp), ctypes.byref(cc), t, _ptr(uu), _ptr(out)))
        return out.reshape(p.shape)

    def assemble_line(self, p: ProblemSpec, axis, a, b, t, theta_dt, cfg=None):
        cp, cc = p.to_c(), (cfg or SolverConfig()).to_c()
        n = p.shape[axis]
        lo, di, up, s2 = np.empty(n), np.empty(n), np.empty(n), c_double()
        self._chk(self._f("assemble_line")(ctypes.byref(cp), ctypes.byref(cc), axis, a, b, t,
                                           theta_dt, _ptr(lo), _ptr(di), _ptr(up), ctypes.byref(s2)))
        return lo, di, up, s2.value

    def thomas(self, lower, diag, upper, super2, rhs):
        lower, diag, upper = (np.ascontiguousarray(x, dtype=np.float64) for x in (lower, diag, upper))
        x = np.ascontiguousarray(rhs, dtype=np.float64).copy()
        count, n = x.shape
        s2 = np.ascontiguousarray(super2, dtype=np.float64).reshape(count)
        code = self._f("thomas")(n, count, _ptr(lower), _ptr(diag), _ptr(upper), _ptr(s2), _ptr(x))
        return x, code, (self.error() if code else "")

    def spot_price(self, p: ProblemSpec, grid) -> float:
        cp = p.to_c()
        g = np.ascontiguousarray(grid, dtype=np.float64).reshape(-1)
        out = c_double()
        self._chk(self._f("spot_price")(ctypes.byref(cp), _ptr(g), ctypes.byref(out)))
        return out.value

    def interpolate(self, p: ProblemSpec, grid, zr, zv, zy) -> float:
        cp = p.to_c()
        g = np.ascontiguousarray(grid, dtype=np.float64).reshape(-1)
        out = c_double()
        self._chk(self._f("interpolate")(ctypes.byref(cp), _ptr(g), zr, zv, zy, ctypes.byref(out)))
        return out.value

    def greeks(self, p: ProblemSpec, grid, scale_rate: bool = True):
        """extract_greeks (instruments.cpp:90-132) [+ finish()'s rho /= r0] -> (rho, vega)."""
        cp = p.to_c()
        g = np.ascontiguousarray(grid, dtype=np.float64).reshape(-1)
        rho, vega = np.empty_like(g), np.empty_like(g)
        self._chk(self._f("extract_greeks")(ctypes.byref(cp), _ptr(g), int(scale_rate), _ptr(rho), _ptr(vega)))
        return rho.reshape(p.shape), vega.reshape(p.shape)

    def mc_price(self, p: ProblemSpec, n_paths: int = 200000, steps_per_year: int = 96,
                 seed: int = 20070423, full_truncation: bool = True, threads: int = 0):
        """The reference's simulate_zcb / simulate_caplet (reference checker only)."""
        cp = p.to_c()
        cfg = A.CMcConfig(n_paths, steps_per_year, seed, int(full_truncation))
        mean, se, n = c_double(), c_double(), ctypes.c_longlong()
        self._chk(self.lib.ref_mc_price(ctypes.byref(cp), ctypes.byref(cfg), threads, ctypes.byref(mean),
                                        ctypes.byref(se), ctypes.byref(n)))
        return mean.value, se.value, n.value

    def curve_eval(self, p: ProblemSpec, what: int, t) -> np.ndarray:
        c = p.to_c().curve
        tt = np.ascontiguousarray(t, dtype=np.float64)
        out = np.empty_like(tt)
        self._chk(self._f("curve_eval")(ctypes.byref(c), what, tt.shape[0], _ptr(tt), _ptr(out)))
        return out

    def uniform_axis(self, z0, z_inf, n):
        z, j1, j2 = np.empty(n), np.empty(n), np.empty(n)
        self._chk(self._f("uniform_axis")(z0, z_inf, n, _ptr(z), _ptr(j1), _ptr(j2)))
        return z, j1, j2

    def sinh_axis(self, center, alpha, z0, z_inf, n):
        z, j1, j2, cc = np.empty(n), np.empty(n), np.empty(n), np.empty(2)
        self._chk(self._f("sinh_axis")(center, alpha, z0, z_inf, n, _ptr(z), _ptr(j1), _ptr(j2), _ptr(cc)))
        return z, j1, j2, cc

    def batch_run(self, problems, cfg: Optional[SolverConfig] = None, threads: int = 1):
        arr = problems_to_c(problems)
        cc = (cfg or SolverConfig()).to_c()
        prices = np.empty(len(problems))
        reps = (A.CReport * len(problems))()
        code = self._f("batch_run")(arr, len(problems), ctypes.byref(cc), threads, _ptr(prices), reps)
        return prices, [r.as_dict() for r in reps], code


class RefSession:
    """ref_session_*: run()'s setup once, then `steps(n)` advances the march with
    the reference's douglas_step and returns the stepping loop's own seconds."""

    def __init__(self, chk: Checker, p: ProblemSpec, cfg: Optional[SolverConfig] = None):
        self.chk = chk
        self._keep = (p.to_c(), (cfg or SolverConfig()).to_c())
        self.h = chk.lib.ref_session_create(ctypes.byref(self._keep[0]), ctypes.byref(self._keep[1]))
        if not self.h:
            raise RuntimeError(chk.error())

    def steps(self, n: int) -> float:
        secs = c_double()
        code = self.chk.lib.ref_session_steps(self.h, n, ctypes.byref(secs))
        if code:
            raise RuntimeError(f"[{A.STATUS_NAMES[code]}] {self.chk.error()}")
        return secs.value

    def close(self):
        if self.h:
            self.chk.lib.ref_session_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


_cache = {}


def restatement() -> Checker:
    if "o" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build()
        _cache["o"] = Checker(ORACLE_SO, "oracle_")
    return _cache["o"]


def reference() -> Optional[Checker]:
    if "r" not in _cache:
        _cache["r"] = Checker(REF_SO, "ref_") if os.path.exists(REF_SO) else None
    return _cache["r"]


def normwise_rel(a, b) -> float:
    """max|a-b| / max|b| — the SURVEY §8d grid parity measure."""
    a, b = np.asarray(a), np.asarray(b)
    den = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / den) if den > 0 else float(np.max(np.abs(a - b)))
