"""GPU parity: the sm_100a path through the C-ABI vs the oracle restatement.

Bar (BASELINE north_star): |p_gpu - p_ref| <= 1e-10 |p_ref| and
max|U_gpu - U_ref| <= 1e-10 max|U_ref|, per problem, FP64. STRICT mode keeps
the reference's operation order, so it is held to a tighter 1e-13 on grids.
"""
import dataclasses

import numpy as np
import pytest

import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import workloads as W
from paper_1108_1688_b200.problem import AxisSpec
from paper_1108_1688_b200 import _abi as A
from oracle import bindings as B

pytestmark = pytest.mark.gpu

TOL = 1e-10          # north_star parity tolerance (relative, FP64)
STRICT_TOL = 1e-13   # strict mode: reference operation order, only libm exp ulps differ
MODES = ["strict", "fast"]


def tol_for(mode):
    return STRICT_TOL if mode == "strict" else TOL


def solve(problems, mode, steps=None):
    with hj.Solver(problems, mode=mode) as s:
        if steps is None:
            s.run()
        else:
            s.step(steps)
        grids = [s.grid(q) for q in range(len(problems))]
        prices = s.spot_prices()
        reps = [s.report(q) for q in range(len(problems))]
        launches = s.last_launches()
    return grids, prices, reps, launches


def assert_parity(p, g, price, oracle, mode, steps=-1):
    g_ref, rep_ref, _, _ = oracle.run(p, steps=steps)
    err = B.normwise_rel(g, g_ref)
    assert err <= tol_for(mode), f"grid normwise rel err {err:.3e}"
    if steps < 0:
        p_ref = oracle.spot_price(p, g_ref)
        perr = abs(price - p_ref) / abs(p_ref)
        assert perr <= TOL, f"price rel err {perr:.3e} ({price} vs {p_ref})"
    return g_ref, rep_ref


@pytest.mark.parametrize("mode", MODES)
def test_config0_full_march(gpu, oracle, mode):
    p = W.make_problem(0, 0)
    grids, prices, reps, launches = solve([p], mode)
    _, rep_ref = assert_parity(p, grids[0], prices[0], oracle, mode)
    assert reps[0]["status"] == 0 and reps[0]["steps_done"] == 200
    assert abs(reps[0]["last_max_delta"] - rep_ref["last_max_delta"]) <= 1e-10 * rep_ref["last_max_delta"]
    assert launches > 0


@pytest.mark.parametrize("mode", MODES)
def test_config2_reduced_caplet(gpu, oracle, mode):
    p = W.make_problem(2, 3, nr=48, nv=24, ny=24, steps=60)
    grids, prices, _, _ = solve([p], mode)
    assert_parity(p, grids[0], prices[0], oracle, mode)


@pytest.mark.parametrize("mode", MODES)
def test_config4_batch(gpu, oracle, mode):
    probs = W.make_config(4, count=12)
    kinds = {p.instrument for p in probs}
    assert kinds == {0, 1}, "the batch must mix ZCBs and caplets"
    grids, prices, reps, _ = solve(probs, mode)
    for q, p in enumerate(probs):
        assert reps[q]["status"] == 0
        assert_parity(p, grids[q], prices[q], oracle, mode)


@pytest.mark.parametrize("mode", MODES)
def test_sinh_mesh_caplet(gpu, oracle, mode):
    """Non-uniform j1/j2: the reference's caplet_default metric (instruments.cpp:11-22)."""
    p = W.make_problem(2, 1, nr=40, nv=20, ny=20, steps=30)
    k_scaled = p.strike / p.r0
    p.r = AxisSpec.sinh(k_scaled, 0.05, 0.0, 250.0, 40)
    p.v = AxisSpec.sinh(0.5, 0.5, 0.0, 30.0, 20)
    p.y = AxisSpec.sinh(0.0, 0.05, 0.0, 250.0, 20)
    grids, prices, _, _ = solve([p], mode)
    assert_parity(p, grids[0], prices[0], oracle, mode)


@pytest.mark.parametrize("mode", MODES)
def test_config1_prefix_full_size(gpu, oracle, mode):
    p = W.make_problem(1, 0)
    grids, _, reps, _ = solve([p], mode, steps=4)
    assert reps[0]["steps_done"] == 4
    assert_parity(p, grids[0], None, oracle, mode, steps=4)


@pytest.mark.parametrize("mode", MODES)
def test_config3_prefix_full_size(gpu, oracle, mode):
    p = W.make_problem(3, 0)
    grids, _, _, _ = solve([p], mode, steps=1)
    assert_parity(p, grids[0], None, oracle, mode, steps=1)


@pytest.mark.parametrize("mode", MODES)
def test_step_by_step_matches_full_march(gpu, mode):
    p = W.make_problem(0, 1, nr=32, nv=16, ny=16, steps=30)
    with hj.Solver([p], mode=mode) as s:
        for _ in range(30):
            s.step(1)
        g1 = s.grid(0)
        s.reset()
        s.run()      # first full march of the handle: direct launches
        g2 = s.grid(0)
        s.reset()
        s.run()      # repeated full march: the captured graph
        g3 = s.grid(0)
    assert np.array_equal(g1, g2)
    assert np.array_equal(g2, g3)


def test_repeated_full_march_two_pass(gpu):
    """The two-pass FAST schedule gives the same level from direct launches (a
    handle's first march) and from its captured graph (later marches)."""
    p = W.make_problem(1, 0, nr=64, nv=128, ny=128, steps=12)
    with hj.Solver([p], mode="fast") as s:
        s.run()
        g1 = s.grid(0)
        s.reset()
        s.run()
        g2 = s.grid(0)
    assert np.array_equal(g1, g2)


@pytest.mark.parametrize("mode", MODES)
def test_apply_operator_stage(gpu, oracle, mode):
    p = W.make_problem(2, 2, nr=24, nv=12, ny=16, steps=10)
    rng = np.random.default_rng(7)
    u = oracle.initial_level(p) + 1e-3 * rng.standard_normal(p.shape)
    for t in (p.maturity, 0.5 * p.maturity, 0.0):
        f_ref = oracle.apply_operator(p, t, u)
        f = hj.apply_operator(p, t, u, mode=mode)
        assert B.normwise_rel(f, f_ref) <= tol_for(mode) * 10


@pytest.mark.parametrize("mode", MODES)
def test_douglas_step_stage(gpu, oracle, mode):
    p = W.make_problem(4, 5, steps=200)
    rng = np.random.default_rng(11)
    u = oracle.initial_level(p) * (1 + 1e-4 * rng.standard_normal(p.shape))
    dt = p.maturity / 200
    ref, md_ref, code, _ = oracle.douglas_step(p, u, p.maturity, dt)
    assert code == 0
    out, md = hj.douglas_step(p, u, p.maturity, dt, mode=mode)
    assert B.normwise_rel(out, ref) <= tol_for(mode)
    assert abs(md - md_ref) <= 1e-10 * md_ref


def test_thomas_batch_matches_reference_solver(gpu, oracle):
    rng = np.random.default_rng(3)
    count, n = 64, 50
    lower = rng.uniform(-1, 1, (count, n))
    upper = rng.uniform(-1, 1, (count, n))
    diag = 3.0 + rng.uniform(0, 1, (count, n))
    lower[:, 0] = 0.0
    upper[:, -1] = 0.0
    s2 = rng.uniform(-0.5, 0.5, count)
    s2[::4] = 0.0
    rhs = rng.standard_normal((count, n))
    x_ref, code, _ = oracle.thomas(lower, diag, upper, s2, rhs)
    assert code == 0
    x = hj.thomas_batch(lower, diag, upper, s2, rhs, mode="strict")
    assert np.array_equal(x, x_ref)


def test_thomas_singular_pivot_message(gpu):
    n = 5
    lower, diag, upper = np.zeros((1, n)), np.ones((1, n)), np.zeros((1, n))
    diag[0, 2] = 0.0
    with pytest.raises(hj.SingularPivot, match="thomas_solve: singular pivot at row 2"):
        hj.thomas_batch(lower, diag, upper, np.zeros(1), np.ones((1, n)))


@pytest.mark.parametrize("mode", MODES)
def test_divergence_parity(gpu, oracle, mode):
    """Wide variance domain v in [0,30] diverges; the GPU must flag it."""
    p = W.make_problem(0, 0)
    p.v = AxisSpec.uniform(0.0, 30.0, 32)
    _, rep_ref, code_ref, msg_ref = oracle.run(p, raise_on_error=False)
    assert code_ref == 4 and rep_ref["failed_step"] > 0
    with hj.Solver([p], mode=mode) as s:
        with pytest.raises(hj.Diverged) as ei:
            s.run()
        rep = s.report(0)
    assert rep["status"] == 4
    if mode == "strict":
        assert rep["failed_step"] == rep_ref["failed_step"]
        assert str(ei.value) == msg_ref
    else:
        assert abs(rep["failed_step"] - rep_ref["failed_step"]) <= 1


def test_reference_time_levels_domain_error(gpu):
    """run()'s repeated-subtraction time levels reach t < 0 at T=10, N=2000."""
    p = W.make_problem(3, 0, nr=4, nv=3, ny=3, steps=2000)
    p.time_levels = 0
    with pytest.raises(hj.DomainError, match="discount: negative maturity"):
        hj.Solver([p], mode="strict")


def test_batch_run_driver(gpu, oracle):
    probs = W.make_config(4, count=6, nr=24, nv=12, ny=12, steps=40)
    prices, reps, grids = hj.batch_run(probs, devices=list(range(hj.device_count())),
                                       mode="strict", grids=True)
    off = 0
    for q, p in enumerate(probs):
        g_ref, _, _, _ = oracle.run(p)
        g = grids[off:off + p.size].reshape(p.shape)
        off += p.size
        assert B.normwise_rel(g, g_ref) <= STRICT_TOL
        assert abs(prices[q] - oracle.spot_price(p, g_ref)) <= TOL * abs(prices[q])
        assert reps[q]["status"] == 0


@pytest.mark.parametrize("smoothing", [True, False])
def test_device_terminal_matches_host(gpu, oracle, smoothing):
    """FAST builds the terminal level on the device (smooth_terminal,
    solver.cpp:180-211, caplet_payoff model.cpp:105-112); it must match the host
    restatement up to libm-vs-device exp ulps, for caplets on uniform and sinh meshes."""
    cfg = hj.SolverConfig(smoothing=smoothing)
    probs = W.make_config(2, count=3, nr=32, nv=16, ny=16, steps=10)
    sinh = W.make_problem(2, 5, nr=24, nv=12, ny=20, steps=10)
    sinh.r = AxisSpec.sinh(sinh.strike / sinh.r0, 0.05, 0.0, 250.0, 24)
    sinh.v = AxisSpec.sinh(0.5, 0.5, 0.0, 30.0, 12)
    sinh.y = AxisSpec.sinh(0.0, 0.05, 0.0, 250.0, 20)
    zcb = W.make_problem(0, 0, nr=16, nv=8, ny=8, steps=10)
    for batch in (probs, [sinh], [zcb]):
        with hj.Solver(batch, mode="fast", config=cfg) as s:
            for q, p in enumerate(batch):
                ref = oracle.initial_level(p, cfg)
                g = s.grid(q)
                err = np.max(np.abs(g - ref)) / max(np.max(np.abs(ref)), 1e-300)
                assert err <= 1e-14, f"terminal max rel err {err:.3e}"


@pytest.mark.parametrize("mode", MODES)
def test_device_greeks_and_surface(gpu, oracle, mode):
    """extract_greeks + finish()'s rho scaling + write_surface_csv's slice on the device
     vs the reference's loops on the same level: same operation order."""
    p = W.make_problem(2, 3, nr=32, nv=16, ny=16, steps=20)
    with hj.Solver([p], mode=mode) as s:
        s.run()
        g = s.grid(0)
        rho, vega = s.greeks(0)
        rho_u, _ = s.greeks(0, scale_rate=False)
        surf = s.surface(0, k=0)
    rho_ref, vega_ref = oracle.greeks(p, g)
    rho_uref, _ = oracle.greeks(p, g, scale_rate=False)
    for a, b in ((rho, rho_ref), (vega, vega_ref), (rho_u, rho_uref)):
        assert np.max(np.abs(a - b)) <= 1e-15 * max(np.max(np.abs(b)), 1e-300)
    rz = np.asarray(p.r.z)
    vz = np.asarray(p.v.z)
    ref = np.stack([np.repeat(p.r0 * rz, p.v.n), np.tile(vz, p.r.n), g[:, :, 0].ravel(),
                    rho_ref[:, :, 0].ravel(), vega_ref[:, :, 0].ravel()], axis=1)
    assert np.array_equal(surf, ref)


@pytest.mark.parametrize("mode", MODES)
def test_config2_full_shape_prefix(gpu, oracle, mode):
    """The config-2 grid (128x64x64) through the two-pass FAST kernels (pass A
    k_pa<64,64>, pass B k_plane<64,64>), 30 of its 500 steps."""
    p = W.make_problem(2, 5)
    grids, _, _, _ = solve([p], mode, steps=30)
    assert_parity(p, grids[0], None, oracle, mode, steps=30)


@pytest.mark.parametrize("mode", MODES)
def test_sinh_mesh_two_pass_shape(gpu, oracle, mode):
    """Non-uniform Jacobians on a shape served by the two-pass kernels (64x32x32)."""
    p = W.make_problem(2, 6, nr=64, nv=32, ny=32, steps=50)
    p.r = AxisSpec.sinh(p.strike / p.r0, 0.05, 0.0, 250.0, 64)
    p.v = AxisSpec.sinh(0.5, 0.5, 0.0, 30.0, 32)
    p.y = AxisSpec.sinh(0.0, 0.05, 0.0, 250.0, 32)
    grids, prices, _, _ = solve([p], mode)
    assert_parity(p, grids[0], prices[0], oracle, mode)


FACE_CASES = {
    "all_dirichlet": ((0, 0, 0, 0, 0, 0), 2, 2),
    "rmin_dirichlet": ((0, 0, 1, 0, 2, 0), 2, 2),
    "vmin_dirichlet": ((1, 0, 0, 0, 2, 0), 2, 2),
    "ymin_dirichlet": ((1, 0, 1, 0, 0, 0), 2, 2),
    "first_order_rows": ((1, 0, 1, 0, 2, 0), 1, 1),
}


@pytest.mark.parametrize("case", sorted(FACE_CASES))
@pytest.mark.parametrize("mode", MODES)
def test_custom_face_rules_two_pass(gpu, oracle, mode, case):
    """BoundarySpec face rules beyond the instruments' (discretization.cpp:153-192,
    precedence r_max > y_max > v_max > r_min > y_min > v_min) and first-order
    boundary rows, on the two-pass shape 32^3."""
    rules, y_order, r_order = FACE_CASES[case]
    p = W.make_problem(0, 3, nr=32, nv=32, ny=32, steps=40)
    p.instrument = A.INSTRUMENT_CUSTOM
    p.face_rule = rules
    # every face: P(t, T) (ZCB closed form); the v_max face: P(t,T) - 0.5 P(t, 1.5 T)
    zcb = (1, 1.0, p.maturity, 0.0, 0.0)
    p.face_value = (zcb, zcb, zcb, (2, 1.0, p.maturity, 0.5, 1.5 * p.maturity), zcb, zcb)
    rng = np.random.default_rng(7)
    p.initial_grid = 1.0 + 0.01 * rng.standard_normal(p.shape)
    cfg = hj.SolverConfig(y_boundary_order=y_order, r_boundary_order=r_order)
    with hj.Solver([p], mode=mode, config=cfg) as s:
        s.run()
        g = s.grid(0)
    g_ref, _, _, _ = oracle.run(p, cfg)
    err = B.normwise_rel(g, g_ref)
    assert err <= tol_for(mode), f"{case}: grid normwise rel err {err:.3e}"


def test_get_grids_matches_get_grid(gpu):
    probs = W.make_config(4, count=5, nr=16, nv=8, ny=8, steps=10)
    with hj.Solver(probs, mode="fast") as s:
        s.run()
        allg = s.grids()
        for q in range(len(probs)):
            assert np.array_equal(allg[q], s.grid(q))


def test_collapsed_v_axis_zcb(gpu, oracle):
    """price_zcb's collapsed mesh (singleton v axis, instruments.cpp:134-143): the
    SPEC.md acceptance case (flat 4%, T=20, 100x40, 12 steps/yr) on the device.
    STRICT and FAST (four-kernel schedule without the v sweep) both serve it;
    other collapsed axes are STRICT-only and FAST reports UNSUPPORTED."""
    import math
    spot = math.log(1.04)
    rax = AxisSpec.sinh(spot / 0.01, 0.05, 0.0, 25.0, 100)
    yax = AxisSpec.sinh(0.0, 0.5, 0.0, 250.0, 40)
    p = hj.ProblemSpec(r=rax, v=AxisSpec.singleton(0.0), y=yax, kappa=0.001, lam=0.15, gamma=0.9,
                       eps=1.5, theta=0.25, rho=-0.75, maturity=20.0, flat_base=1.04, n_steps=0,
                       time_levels=A.TIME_REFERENCE)
    with hj.Solver([p], mode="strict") as s:
        s.run()
        g = s.grid(0)
        price = s.price(0, spot / 0.01, 0.0, 0.0)  # interpolate_at on the device
    g_ref, rep_ref, _, _ = oracle.run(p)
    assert B.normwise_rel(g, g_ref) <= STRICT_TOL
    assert rep_ref["n_steps"] == 240
    assert abs(price - oracle.interpolate(p, g_ref, spot / 0.01, 0.0, 0.0)) <= 1e-12
    assert abs(price - 1.04 ** -20) < 1e-5  # SPEC.md:525 acceptance
    with hj.Solver([p], mode="fast") as s:
        s.run()
        assert B.normwise_rel(s.grid(0), g_ref) <= TOL
        assert abs(s.price(0, spot / 0.01, 0.0, 0.0) - price) <= 1e-10 * price
    py = dataclasses.replace(p, v=AxisSpec.sinh(0.5, 0.5, 0.0, 30.0, 8), y=AxisSpec.singleton(0.0))
    with pytest.raises(hj.Unsupported):
        hj.Solver([py], mode="fast")


@pytest.mark.parametrize("mode", MODES)
def test_random_shapes(gpu, oracle, mode):
    """Seeded random grids (any nr, nv != ny, odd sizes) exercise the generic
    FAST kernels and every STRICT path against the oracle."""
    rng = np.random.default_rng(20261020)
    for case in range(6):
        nr, nv, ny = (int(rng.integers(3, 41)), int(rng.integers(3, 25)), int(rng.integers(3, 25)))
        steps = int(rng.integers(5, 30))
        cfg_id = int(rng.choice([0, 2, 4]))
        p = W.make_problem(cfg_id, int(rng.integers(0, 50)), nr=nr, nv=nv, ny=ny, steps=steps)
        grids, prices, reps, _ = solve([p], mode)
        g_ref, rep_ref, code, _ = oracle.run(p, raise_on_error=False)
        if code:  # the reference's scheme itself left the bound: divergence parity
            assert reps[0]["status"] == code
            continue
        err = B.normwise_rel(grids[0], g_ref)
        assert err <= tol_for(mode), f"case {case} {nr}x{nv}x{ny}: {err:.3e}"
        p_ref = oracle.spot_price(p, g_ref)
        assert abs(prices[0] - p_ref) <= TOL * abs(p_ref)


@pytest.mark.parametrize("nr", [16, 48, 80, 208, 512])
def test_pass_a_segment_counts(gpu, oracle, nr):
    """Pass A with 1, 3, 5 and 13 r-segments (warp 0's two-ended recurrence on
    the [column][field][segment] rows) and 32 segments (the lane scan over a
    512-thread block), full marches against the oracle."""
    p = W.make_problem(0, 3, nr=nr, nv=32, ny=32, steps=30)
    grids, prices, _, _ = solve([p], "fast")
    assert_parity(p, grids[0], prices[0], oracle, "fast")


_SCHEDULE_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import workloads as W
from oracle import bindings as B
o = B.restatement()
worst = 0.0
for (nr, n, steps) in [(32, 128, 6), (32, 256, 3), (48, 64, 10)]:
    p = W.make_problem(2, 5, nr=nr, nv=n, ny=n, steps=steps)
    with hj.Solver([p], mode="fast") as s:
        s.run()
        g = s.grid(0)
    g_ref, _, _, _ = o.run(p)
    worst = max(worst, B.normwise_rel(g, g_ref))
print("WORST", worst)
"""


@pytest.mark.parametrize("env", [{"HJMSV_PLANE": "0"}, {"HJMSV_PLANE": "0", "HJMSV_PA": "0"},
                                 {"HJMSV_PLANE": "3"}, {"HJMSV_PLANE": "2"}, {"HJMSV_DBG": "2"},
                                 {"HJMSV_PA_TM": "0", "HJMSV_PA_SEG": "16"},
                                 {"HJMSV_YLU": "0"}, {"HJMSV_PF_AHEAD": "0", "HJMSV_PF_AHEAD_A": "0"},
                                 {"HJMSV_PF_AHEAD": "3", "HJMSV_PF_AHEAD_A": "5"}])
def test_diagnostic_schedules(gpu, env):
    """The schedules behind the diagnostic switches (split v + y kernels with the
    lane-scan k_y3, the four-kernel schedule, the 2-CTA cluster plane, pass A's
    two-ended recurrence at 16+ segments, pass B's partition-method y-lines instead
    of the pivot table, the next-wave prefetches off or at odd distances) stay at parity. The switches are read
    once per process, so each runs in its own interpreter."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _SCHEDULE_SCRIPT.format(root=root)],
                         env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.split("WORST")[-1])
    assert worst <= TOL, (env, worst)


# ---- time-dependent model functions lambda(t), gamma(t), eps(t) (model.hpp:22-24):
# per-step coefficient tables from prepare(t_mid) (discretization.cpp:40-54)
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", [(32, 32, 32), (24, 12, 16), (64, 32, 32)])
def test_model_functions_march(gpu, oracle, mode, shape):
    nr, nv, ny = shape
    for cfg, idx in ((0, 4), (2, 6)):
        p = W.with_model_functions(W.make_problem(cfg, idx, nr=nr, nv=nv, ny=ny, steps=40))
        grids, prices, reps, _ = solve([p], mode)
        g_ref, rep_ref = assert_parity(p, grids[0], prices[0], oracle, mode)
        assert abs(reps[0]["last_max_delta"] - rep_ref["last_max_delta"]) <= 1e-10 * rep_ref["last_max_delta"]
        # the functions matter: the constant model is measurably different
        q = W.make_problem(cfg, idx, nr=nr, nv=nv, ny=ny, steps=40)
        assert B.normwise_rel(oracle.run(q)[0], g_ref) > 1e-6


@pytest.mark.parametrize("mode", MODES)
def test_model_functions_mixed_batch(gpu, oracle, mode):
    """A batch mixing constant and time-dependent models (every problem then
    carries per-step tables)."""
    probs = [W.make_problem(4, q, steps=50) for q in range(4)]
    probs[1] = W.with_model_functions(probs[1])
    probs[3] = W.with_model_functions(probs[3], amp=-0.2)
    grids, prices, reps, _ = solve(probs, mode)
    for q, p in enumerate(probs):
        assert_parity(p, grids[q], prices[q], oracle, mode)


@pytest.mark.parametrize("mode", MODES)
def test_model_functions_stages(gpu, oracle, mode):
    p = W.with_model_functions(W.make_problem(2, 2, nr=24, nv=12, ny=16, steps=10))
    rng = np.random.default_rng(5)
    u = oracle.initial_level(p) * (1 + 1e-4 * rng.standard_normal(p.shape))
    for t in (p.maturity, 0.37 * p.maturity):
        f_ref = oracle.apply_operator(p, t, u)
        assert B.normwise_rel(hj.apply_operator(p, t, u, mode=mode), f_ref) <= tol_for(mode) * 10
    dt = p.maturity / 10
    ref, md_ref, code, _ = oracle.douglas_step(p, u, 0.6 * p.maturity, dt)
    out, md = hj.douglas_step(p, u, 0.6 * p.maturity, dt, mode=mode)
    assert code == 0 and B.normwise_rel(out, ref) <= tol_for(mode)
    assert abs(md - md_ref) <= 1e-10 * md_ref


def test_model_functions_vs_compiled_reference(gpu, reference):
    """FAST two-pass march with model functions against the compiled reference's run()."""
    p = W.with_model_functions(W.make_problem(2, 9, nr=64, nv=32, ny=32, steps=60))
    grids, prices, reps, _ = solve([p], "fast")
    g_ref, rep_ref, code, _ = reference.run(p)
    assert code == 0
    assert B.normwise_rel(grids[0], g_ref) <= TOL
    p_ref = reference.spot_price(p, g_ref)
    assert abs(prices[0] - p_ref) <= TOL * abs(p_ref)


@pytest.mark.parametrize("shape", [(100, 50, 50), (72, 40, 90), (130, 33, 64), (40, 24, 200), (20, 130, 17),
                                   (33, 100, 120), (17, 5, 3), (64, 64, 100)])
def test_padded_pass_a_shapes(gpu, oracle, shape):
    """Shapes outside the exact instantiations run the fused pass A padded (ny up
    to 32/64/128/256 and nr up to a multiple of 16 with inert lanes and rows),
    e.g. the reference's own 100x50x50 caplet mesh (instruments.cpp:11-22)."""
    nr, nv, ny = shape
    p = W.make_problem(2, 11, nr=nr, nv=nv, ny=ny, steps=40)
    with hj.Solver([p], mode="fast") as s:
        prof, _ = s.kernel_profile(2)
        names = [k["name"] for k in prof]
        assert "fx_explicit_sweep_r" in names
        if max(nv, ny) <= 128:  # and pass B on a padded plane: two kernels per step
            assert "fx_plane_vy_update" in names and "fx_sweep_v" not in names
        s.reset()
        s.run()
        g, price = s.grid(0), float(s.spot_prices()[0])
    assert_parity(p, g, price, oracle, "fast")


def test_pass_a_32_row_segments(gpu, oracle):
    """512-row lines run pass A with 32-row segments whose c' and alpha rows live
    in tensor memory (16 segments, lane-scan reduced systems); on a 128-wide plane
    too, against the oracle."""
    p = W.make_problem(2, 8, nr=512, nv=128, ny=128, steps=6)
    with hj.Solver([p], mode="fast") as s:
        s.step(6)
        g = s.grid(0)
    g_ref = oracle.run(p, steps=6)[0]
    assert B.normwise_rel(g, g_ref) <= TOL


def test_concurrent_handles_tensor_memory_and_model_functions(gpu, oracle):
    """Two handles at once on one device (hjmsv_batch_run over devices [0, 0]): their
    pass-A CTAs share the SMs' tensor memory (the lane-scan variants allocate TMEM
    columns per CTA), half the problems carry model functions of t; every grid
    against the oracle."""
    probs = [W.make_problem(1, q, steps=6) for q in range(4)]
    probs[1] = W.with_model_functions(probs[1])
    probs[2] = W.with_model_functions(probs[2], amp=-0.25)
    prices, reps, grids = hj.batch_run(probs, devices=[0, 0], mode="fast", grids=True)
    off = 0
    for q, p in enumerate(probs):
        assert reps[q]["status"] == 0 and reps[q]["steps_done"] == 6
        g = grids[off:off + p.size].reshape(p.shape)
        off += p.size
        g_ref = oracle.run(p)[0]
        assert B.normwise_rel(g, g_ref) <= TOL, q
