"""The C-ABI boundary on CPU: the library loads, exports every symbol the header
declares, and its host-side logic (validation, lowering helpers) matches the
reference without any device call."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import _abi as A
from paper_1108_1688_b200 import workloads as W
from paper_1108_1688_b200.problem import AxisSpec, SolverConfig, _ptr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hjmsv_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hjmsv_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("hjmsv_solver_create", "hjmsv_solver_run", "hjmsv_solver_get_grid",
                 "hjmsv_douglas_step", "hjmsv_apply_operator", "hjmsv_thomas_batch",
                 "hjmsv_batch_run", "hjmsv_solver_spot_prices"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = A.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) == set(A.SIGNATURES), "ctypes table out of sync with header"
    assert lib.hjmsv_abi_version() == 2  # hjmsv_model gained the model functions of t


def test_library_is_sm100a_native():
    """The shared library embeds sm_100a SASS (cuobjdump lists the cubin arch)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([tool, "--list-elf", A.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config_matches_reference_defaults():
    c = A.CSolverConfig()
    A.load().hjmsv_default_solver_config(ctypes.byref(c))
    assert (c.theta_cn, c.steps_per_year, c.y_boundary_order, c.r_boundary_order, c.smoothing,
            c.smoothing_subsamples, c.divergence_bound) == (0.5, 12, 2, 2, 1, 3, 1e6)


@pytest.mark.parametrize("cfg,msg", [
    (SolverConfig(theta_cn=1.5), "theta_cn must lie in [0,1]"),
    (SolverConfig(steps_per_year=0), "steps_per_year must be >= 1"),
    (SolverConfig(y_boundary_order=3), "y_boundary_order must be 1 or 2"),
    (SolverConfig(smoothing_subsamples=0), "smoothing_subsamples must be >= 1"),
    (SolverConfig(divergence_bound=0.0), "divergence_bound must be positive"),
    (SolverConfig(r_boundary_order=5), "r boundary order must be 1 or 2"),
])
def test_validation_messages_match_reference(cfg, msg):
    p = W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=4)
    with pytest.raises(hj.InvalidArgument, match=re.escape(msg)):
        hj.Solver([p], config=cfg, mode="strict")


def test_model_and_instrument_validation():
    p = W.make_problem(2, 0, nr=8, nv=4, ny=4, steps=4)
    p.payment = p.maturity
    with pytest.raises(hj.InvalidArgument, match="caplet payment date must exceed expiry"):
        hj.Solver([p])
    p = W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=4)
    p.rho = -1.5
    with pytest.raises(hj.InvalidArgument, match=re.escape("rho must lie in [-1,1]")):
        hj.Solver([p])
    p = W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=4)
    p.gamma = 1.2
    with pytest.raises(hj.InvalidArgument, match=re.escape("gamma must lie in (0,1]")):
        hj.Solver([p])
    p = W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=4)
    p.face_rule = (1, 1, 1, 0, 2, 0)
    p.instrument = A.INSTRUMENT_CUSTOM
    p.initial_grid = np.ones(p.size)
    with pytest.raises(hj.InvalidArgument, match="upper faces must carry Dirichlet rules"):
        hj.Solver([p])


def test_time_bug_surfaces_as_domain_error_before_device_work():
    p = W.make_problem(3, 0, nr=4, nv=3, ny=3, steps=2000)
    p.time_levels = A.TIME_REFERENCE
    with pytest.raises(hj.DomainError, match="discount: negative maturity"):
        hj.Solver([p])


def test_host_axis_helpers_match_oracle(oracle):
    lib = A.load()
    n = 37
    z, j1, j2, cc = np.empty(n), np.empty(n), np.empty(n), np.empty(2)
    assert lib.hjmsv_sinh_axis(2.5, 0.05, 0.0, 250.0, n, _ptr(z), _ptr(j1), _ptr(j2), _ptr(cc)) == 0
    oz, oj1, oj2, occ = oracle.sinh_axis(2.5, 0.05, 0.0, 250.0, n)
    assert np.array_equal(z, oz) and np.array_equal(j1, oj1) and np.array_equal(j2, oj2)
    assert np.array_equal(cc, occ)
    assert lib.hjmsv_uniform_axis(0.0, 25.0, n, _ptr(z), _ptr(j1), _ptr(j2)) == 0
    u = AxisSpec.uniform(0.0, 25.0, n)
    assert np.array_equal(z, u.z) and np.array_equal(z, oracle.uniform_axis(0.0, 25.0, n)[0])


def test_host_curve_matches_oracle(oracle):
    lib = A.load()
    p = W.make_problem(4, 17)
    t = np.linspace(0.0, 40.0, 401)
    c = p.to_c().curve
    for what in (0, 1, 2):
        out = np.empty_like(t)
        assert lib.hjmsv_curve_eval(ctypes.byref(c), what, t.shape[0], _ptr(t), _ptr(out)) == 0
        assert np.array_equal(out, oracle.curve_eval(p, what, t))
    out = np.empty(1)
    assert lib.hjmsv_curve_eval(ctypes.byref(c), 0, 1, _ptr(np.array([-1e-13])), _ptr(out)) == A.DOMAIN
    assert lib.hjmsv_last_error() == b"discount: negative maturity"


def test_solver_requires_a_device_here():
    """No CPU fallback: without a GPU the handle cannot be created."""
    if hj.device_count() > 0:
        pytest.skip("a device is visible")
    p = W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=4)
    with pytest.raises(hj.CudaError):
        hj.Solver([p])


def test_fast_lines_are_bounded_and_modes_validated():
    """hjmsv_thomas_batch: FAST lines hold at most 32 segments of 16 rows (n <= 512);
    an unknown mode is an invalid argument. Both are decided before any device work."""
    import numpy as np
    import paper_1108_1688_b200 as hj
    n, c = 600, 2
    z = np.zeros((c, n))
    d = np.ones((c, n))
    with pytest.raises(hj.Unsupported):
        hj.thomas_batch(z, d, z, np.zeros(c), d, mode="fast")
    with pytest.raises(hj.Unsupported):
        hj.thomas_batch(z, d, z, np.zeros(c), d, mode="fast_twisted")
    with pytest.raises(hj.InvalidArgument):
        hj.thomas_batch(z[:, :8], d[:, :8], z[:, :8], np.zeros(c), d[:, :8], mode=7)


@pytest.mark.gpu
def test_kernel_timeline_shares(gpu):
    """hjmsv_solver_kernel_timeline: per-kernel durations from the device clock of
    every block in a march launched like the timed one; the per-step kernels'
    durations add up to at most the march (no overlap is counted twice)."""
    import paper_1108_1688_b200 as hj
    from paper_1108_1688_b200 import workloads as W
    p = W.make_problem(1, 0, steps=40)
    with hj.Solver([p], mode="fast") as s:
        # the first profiled sequence of a fresh process also pays module loading
        # and first-touch costs inside its event-timed total: warm up once
        s.kernel_profile(40)
        s.reset()
        prof, launches, total_ms = s.kernel_profile(40, with_total=True)
        names = [k["name"] for k in prof]
        assert "fx_explicit_sweep_r" in names and "fx_plane_vy_update" in names
        per_step = sum(k["avg_ms"] for k in prof if k["name"] != "fx_faces") * 40
        assert 0.5 * total_ms < per_step <= 1.0 * total_ms
        assert launches >= 80
        alg = {k["name"]: k["alg_bytes"] for k in prof}
        assert alg["fx_explicit_sweep_r"] == 16.0 * p.size and alg["fx_plane_vy_update"] == 24.0 * p.size
        with pytest.raises(hj.InvalidArgument):
            s.kernel_profile(1)  # the march is over: reset first
        s.reset()
        s.kernel_profile(2)
