"""ctypes mirror of include/hjmsv_b200.h (the framework's C-ABI).

The structs here are byte-for-byte the C structs; `load()` opens the in-tree
``lib/libhjmsv_b200.so`` and fails loudly when it has not been built — there is
no CPU fallback for the solver.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# HJMSV_LIB: another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("HJMSV_LIB") or os.path.join(HERE, "lib", "libhjmsv_b200.so")

# hjmsv_status
OK, INVALID_ARGUMENT, SINGULAR_PIVOT, NONFINITE, DIVERGED, DOMAIN, UNSUPPORTED, CUDA_ERROR, LOGIC = range(9)
STATUS_NAMES = ["OK", "INVALID_ARGUMENT", "SINGULAR_PIVOT", "NONFINITE", "DIVERGED", "DOMAIN",
                "UNSUPPORTED", "CUDA_ERROR", "LOGIC"]
MAP_SINH, MAP_LINEAR, MAP_SINGLETON = 0, 1, 2
CURVE_FLAT, CURVE_NODES = 0, 1
FACE_DIRICHLET, FACE_DEGENERATE, FACE_ONE_SIDED = 0, 1, 2
VALUE_ZERO, VALUE_ZCB, VALUE_ZCB_DIFF = 0, 1, 2
INSTRUMENT_ZCB, INSTRUMENT_CAPLET, INSTRUMENT_CUSTOM = 0, 1, 2
TIME_REFERENCE, TIME_INDEXED = 0, 1
MODE_STRICT, MODE_FAST = 0, 1

PD = POINTER(c_double)


class CAxis(ctypes.Structure):
    _fields_ = [("n", c_int32), ("map", c_int32), ("z", PD), ("j1", PD), ("j2", PD),
                ("center", c_double), ("alpha", c_double), ("z0", c_double), ("z_inf", c_double),
                ("c1", c_double), ("c2", c_double)]


# hjmsv_time_fn: double (*)(double t, void* user) — TimeFn (model.hpp:10)
TIME_FN = ctypes.CFUNCTYPE(c_double, c_double, ctypes.c_void_p)


class CModel(ctypes.Structure):
    _fields_ = [("kappa", c_double), ("lam", c_double), ("gamma", c_double), ("eps", c_double),
                ("theta", c_double), ("rho", c_double), ("lambda_fn", TIME_FN), ("gamma_fn", TIME_FN),
                ("eps_fn", TIME_FN), ("fn_user", ctypes.c_void_p)]


class CCurve(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("flat_base", c_double), ("n_nodes", c_int32),
                ("maturities", PD), ("discounts", PD)]


class CFaceValue(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("a", c_double), ("t1", c_double), ("b", c_double), ("t2", c_double)]


class CProblem(ctypes.Structure):
    _fields_ = [("r", CAxis), ("v", CAxis), ("y", CAxis), ("model", CModel), ("curve", CCurve),
                ("r0", c_double), ("maturity", c_double), ("instrument", c_int32),
                ("payment", c_double), ("strike", c_double), ("face_rule", c_int32 * 6),
                ("face_value", CFaceValue * 6), ("n_steps", c_int32), ("time_levels", c_int32),
                ("initial_grid", PD)]


class CSolverConfig(ctypes.Structure):
    _fields_ = [("theta_cn", c_double), ("steps_per_year", c_int32), ("y_boundary_order", c_int32),
                ("r_boundary_order", c_int32), ("smoothing", c_int32),
                ("smoothing_subsamples", c_int32), ("divergence_bound", c_double)]


class CMcConfig(ctypes.Structure):
    _fields_ = [("n_paths", ctypes.c_int64), ("steps_per_year", c_int32), ("seed", ctypes.c_uint64),
                ("full_truncation", c_int32)]


class CReport(ctypes.Structure):
    _fields_ = [("wall_seconds", c_double), ("n_steps", c_int32), ("steps_done", c_int32),
                ("last_max_delta", c_double), ("nan_guard_ok", c_int32), ("status", c_int32),
                ("failed_step", c_int32), ("failed_row", c_int32), ("time", c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


# Every symbol the header declares, with its ctypes signature.
I32, HP = c_int32, c_void_p
SIGNATURES = {
    "hjmsv_default_solver_config": (None, [POINTER(CSolverConfig)]),
    "hjmsv_default_mc_config": (None, [POINTER(CMcConfig)]),
    "hjmsv_mc_price": (I32, [POINTER(CProblem), POINTER(CMcConfig), I32, PD, PD,
                             POINTER(ctypes.c_int64)]),
    "hjmsv_last_error": (ctypes.c_char_p, []),
    "hjmsv_abi_version": (I32, []),
    "hjmsv_device_count": (I32, []),
    "hjmsv_uniform_axis": (I32, [c_double, c_double, I32, PD, PD, PD]),
    "hjmsv_sinh_axis": (I32, [c_double, c_double, c_double, c_double, I32, PD, PD, PD, PD]),
    "hjmsv_curve_eval": (I32, [POINTER(CCurve), I32, I32, PD, PD]),
    "hjmsv_zcb_closed_form": (I32, [POINTER(CCurve), c_double, c_double, c_double, c_double, c_double, PD]),
    "hjmsv_solver_create": (I32, [POINTER(CProblem), I32, POINTER(CSolverConfig), I32, I32, POINTER(HP)]),
    "hjmsv_solver_destroy": (None, [HP]),
    "hjmsv_solver_reset": (I32, [HP]),
    "hjmsv_solver_step_async": (I32, [HP, I32]),
    "hjmsv_solver_synchronize": (I32, [HP]),
    "hjmsv_solver_step": (I32, [HP, I32]),
    "hjmsv_solver_run": (I32, [HP]),
    "hjmsv_solver_report": (I32, [HP, I32, POINTER(CReport)]),
    "hjmsv_solver_dims": (I32, [HP, POINTER(I32), POINTER(I32), POINTER(I32), POINTER(I32), POINTER(I32)]),
    "hjmsv_solver_get_grid": (I32, [HP, I32, PD]),
    "hjmsv_solver_get_grids": (I32, [HP, PD]),
    "hjmsv_solver_set_grid": (I32, [HP, I32, PD, I32]),
    "hjmsv_solver_price": (I32, [HP, I32, c_double, c_double, c_double, PD]),
    "hjmsv_solver_spot_prices": (I32, [HP, PD]),
    "hjmsv_solver_greeks": (I32, [HP, I32, I32, PD, PD]),
    "hjmsv_solver_surface": (I32, [HP, I32, I32, PD]),
    "hjmsv_solver_device_grid": (I32, [HP, I32, POINTER(PD)]),
    "hjmsv_solver_last_device_ms": (I32, [HP, PD]),
    "hjmsv_solver_last_launches": (I32, [HP, POINTER(c_int64)]),
    "hjmsv_solver_kernel_profile": (I32, [HP, I32, I32, PD, PD, POINTER(c_int64), POINTER(I32),
                                          ctypes.c_char_p, I32]),
    "hjmsv_solver_kernel_timeline": (I32, [HP, I32, I32, PD, PD, POINTER(c_int64), POINTER(I32),
                                           ctypes.c_char_p, I32, PD]),
    "hjmsv_apply_operator": (I32, [POINTER(CProblem), POINTER(CSolverConfig), c_double, PD, PD, I32]),
    "hjmsv_douglas_step": (I32, [POINTER(CProblem), POINTER(CSolverConfig), PD, c_double, c_double, PD, PD, I32]),
    "hjmsv_thomas_batch": (I32, [I32, I32, PD, PD, PD, PD, PD, I32]),
    "hjmsv_batch_run": (I32, [POINTER(CProblem), I32, POINTER(CSolverConfig), POINTER(I32), I32, I32,
                              PD, POINTER(CReport), PD]),
}

_LIB = None


def load(path: str | None = None):
    """Open the C-ABI library; raise if it is missing (no fallback path exists)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the solver has no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib
