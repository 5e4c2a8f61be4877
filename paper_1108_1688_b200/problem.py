"""Plain-data pricing problems: the Python face of ``hjmsv_problem``.

Mirrors the reference's PdeProblem (proj/core/include/hjmsv/solver.hpp:59-72)
plus the explicit instrument descriptor of SURVEY.md §8b. Arrays are numpy
float64 and are kept alive by the spec while a C struct points at them.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi as A


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.cast(None, A.PD)
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(A.PD)


@dataclass
class AxisSpec:
    """One direction (reference Axis, mesh.hpp:25-40)."""
    z: np.ndarray
    j1: np.ndarray
    j2: np.ndarray
    map: int = A.MAP_LINEAR
    center: float = 0.0
    alpha: float = 1.0
    z0: float = 0.0
    z_inf: float = 1.0
    c1: float = 0.0
    c2: float = 0.0

    @property
    def n(self) -> int:
        return int(self.z.shape[0])

    @staticmethod
    def uniform(z0: float, z_inf: float, n: int) -> "AxisSpec":
        """uniform_axis (mesh.cpp:46-62), same IEEE operations."""
        z0, z_inf = float(z0), float(z_inf)
        if not z0 < z_inf:
            raise ValueError("axis requires z0 < z_inf")
        if n < 3:
            raise ValueError("axis needs at least 3 nodes")
        x = np.arange(n, dtype=np.float64) / float(n - 1)
        z = z0 + (z_inf - z0) * x
        return AxisSpec(z=np.ascontiguousarray(z), j1=np.full(n, z_inf - z0), j2=np.zeros(n),
                        map=A.MAP_LINEAR, center=z0, alpha=1.0, z0=z0, z_inf=z_inf)

    @staticmethod
    def sinh(center: float, alpha: float, z0: float, z_inf: float, n: int) -> "AxisSpec":
        """build_axis (mesh.cpp:16-44) via the framework's host restatement."""
        lib = A.load()
        z, j1, j2, cc = np.empty(n), np.empty(n), np.empty(n), np.empty(2)
        code = lib.hjmsv_sinh_axis(center, alpha, z0, z_inf, n, _ptr(z), _ptr(j1), _ptr(j2), _ptr(cc))
        if code:
            raise ValueError(lib.hjmsv_last_error().decode())
        return AxisSpec(z=z, j1=j1, j2=j2, map=A.MAP_SINH, center=center, alpha=alpha, z0=z0,
                        z_inf=z_inf, c1=float(cc[0]), c2=float(cc[1]))

    @staticmethod
    def singleton(value: float) -> "AxisSpec":
        """singleton_axis (mesh.cpp:64-73)."""
        return AxisSpec(z=np.array([value]), j1=np.ones(1), j2=np.zeros(1), map=A.MAP_SINGLETON,
                        center=value, z0=value, z_inf=value)

    def to_c(self) -> A.CAxis:
        return A.CAxis(self.n, self.map, _ptr(self.z), _ptr(self.j1), _ptr(self.j2), self.center,
                       self.alpha, self.z0, self.z_inf, self.c1, self.c2)


@dataclass
class ProblemSpec:
    """One pricing problem (PdeProblem + instrument + time-level policy)."""
    r: AxisSpec
    v: AxisSpec
    y: AxisSpec
    kappa: float
    lam: float
    gamma: float
    eps: float
    theta: float
    rho: float
    maturity: float
    r0: float = 0.01
    curve_maturities: Optional[np.ndarray] = None  # None -> flat curve
    curve_discounts: Optional[np.ndarray] = None
    flat_base: float = 1.04
    instrument: int = A.INSTRUMENT_ZCB
    payment: float = 0.0
    strike: float = 0.0
    n_steps: int = 0
    time_levels: int = A.TIME_INDEXED
    face_rule: Sequence[int] = (1, 0, 1, 0, 2, 0)
    face_value: Sequence[tuple] = ((0, 0, 0, 0, 0),) * 6   # (kind, a, t1, b, t2)
    initial_grid: Optional[np.ndarray] = None
    # time-dependent model functions lambda(t), gamma(t), eps(t) (ModelParams::
    # lambda_fn / gamma_fn / eps_fn, model.hpp:22-24); None -> the constant above
    lambda_fn: Optional[Callable[[float], float]] = None
    gamma_fn: Optional[Callable[[float], float]] = None
    eps_fn: Optional[Callable[[float], float]] = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def shape(self):
        return (self.r.n, self.v.n, self.y.n)

    @property
    def size(self) -> int:
        return self.r.n * self.v.n * self.y.n

    def to_c(self) -> A.CProblem:
        p = A.CProblem()
        p.r, p.v, p.y = self.r.to_c(), self.v.to_c(), self.y.to_c()
        p.model = A.CModel(self.kappa, self.lam, self.gamma, self.eps, self.theta, self.rho)
        fns = []
        for name in ("lambda_fn", "gamma_fn", "eps_fn"):
            f = getattr(self, name)
            if f is not None:
                # the C callback must outlive the C struct: kept with the spec
                cb = A.TIME_FN(lambda t, _u, f=f: float(f(t)))
                fns.append(cb)
                setattr(p.model, name, cb)
        self._fns = fns
        if self.curve_maturities is None:
            p.curve = A.CCurve(A.CURVE_FLAT, self.flat_base, 0, _ptr(None), _ptr(None))
        else:
            m = np.ascontiguousarray(self.curve_maturities, dtype=np.float64)
            d = np.ascontiguousarray(self.curve_discounts, dtype=np.float64)
            self._keep[:] = [m, d]
            p.curve = A.CCurve(A.CURVE_NODES, 0.0, int(m.shape[0]), _ptr(m), _ptr(d))
        p.r0, p.maturity, p.instrument = self.r0, self.maturity, self.instrument
        p.payment, p.strike = self.payment, self.strike
        for f in range(6):
            p.face_rule[f] = int(self.face_rule[f])
            k, a, t1, b, t2 = self.face_value[f]
            p.face_value[f] = A.CFaceValue(int(k), a, t1, b, t2)
        p.n_steps, p.time_levels = int(self.n_steps), int(self.time_levels)
        if self.initial_grid is not None:
            g = np.ascontiguousarray(self.initial_grid, dtype=np.float64).reshape(-1)
            self._keep.append(g)
            p.initial_grid = _ptr(g)
        else:
            p.initial_grid = _ptr(None)
        return p

    def curve_c(self) -> A.CCurve:
        return self.to_c().curve


def problems_to_c(specs: Sequence[ProblemSpec]):
    arr = (A.CProblem * len(specs))()
    for q, s in enumerate(specs):
        arr[q] = s.to_c()
    return arr


@dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:10-20)."""
    theta_cn: float = 0.5
    steps_per_year: int = 12
    y_boundary_order: int = 2
    r_boundary_order: int = 2
    smoothing: bool = True
    smoothing_subsamples: int = 3
    divergence_bound: float = 1e6

    def to_c(self) -> A.CSolverConfig:
        return A.CSolverConfig(self.theta_cn, self.steps_per_year, self.y_boundary_order,
                               self.r_boundary_order, int(bool(self.smoothing)),
                               self.smoothing_subsamples, self.divergence_bound)


def mix_seed(root: int, stream: int) -> int:
    """splitmix64 step of the reference (montecarlo.cpp:12-17), 64-bit wrap."""
    M = (1 << 64) - 1
    z = (root + 0x9E3779B97F4A7C15 * (stream + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def uniform_draw(root: int, stream: int) -> float:
    """u = (mix_seed(root, stream) >> 11) * 2^-53."""
    return (mix_seed(root, stream) >> 11) * (2.0 ** -53)


def curve_nodes(a: float, b: float, c: float, t_max: float = 30.0, step: float = 0.25):
    """Quarterly discount quotes of f(0,T) = a + b(1 - e^{-cT})."""
    n = int(round(t_max / step))
    mats = np.array([step * (q + 1) for q in range(n)], dtype=np.float64)
    disc = np.array([math.exp(-a * T - b * (T - (1.0 - math.exp(-c * T)) / c)) for T in mats])
    return mats, disc
