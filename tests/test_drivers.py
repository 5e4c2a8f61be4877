"""Callers on the batch engine: caplet_ladder
(instruments.cpp:238-266) and cmd_convergence's table (job.cpp:381-472)."""
import dataclasses

import numpy as np
import pytest

import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import drivers
from paper_1108_1688_b200 import workloads as W
from paper_1108_1688_b200 import _abi as A


def test_caplet_ladder_rejects_non_caplet():
    with pytest.raises(ValueError):
        drivers.caplet_ladder(W.make_problem(0, 0, nr=8, nv=4, ny=4, steps=2), [0.01])


@pytest.mark.gpu
def test_caplet_ladder_matches_per_strike_oracle(gpu, oracle):
    base = W.make_problem(2, 4, nr=24, nv=12, ny=12, steps=30)
    strikes = [0.01, 0.02, 0.035, 0.05]
    out = drivers.caplet_ladder(base, strikes)
    assert [k for k, _ in out] == strikes
    prev = None
    for k, price in out:
        p = dataclasses.replace(base, strike=k)
        g_ref, _, _, _ = oracle.run(p)
        p_ref = oracle.spot_price(p, g_ref)
        assert abs(price - p_ref) <= 1e-10 * abs(p_ref)
        if prev is not None:  # caplet value falls with the strike
            assert price <= prev + 1e-12
        prev = price


@pytest.mark.gpu
def test_convergence_table_rows(gpu, oracle):
    def make(nr, nv, ny):
        return W.make_problem(0, 1, nr=nr, nv=nv, ny=ny, steps=1)

    rows = drivers.convergence(make, nr_list=[16, 32], ny_list=[8, 16], nt_list=[20, 40],
                               base=(16, 8, 8), config=hj.SolverConfig(steps_per_year=20))
    sweeps = [r["sweep"] for r in rows]
    assert sweeps == ["mesh", "mesh", "nt", "nt", "order"]
    # each value is the device price of that mesh / step count; the error column is
    # |price - p(0,T)| (price_zcb's closed-form reference)
    for r in rows[:4]:
        p = dataclasses.replace(make(r["nr"], r["nv"], r["ny"]), n_steps=0)
        cfg = hj.SolverConfig(steps_per_year=r["steps_per_year"])
        g_ref, _, _, _ = oracle.run(p, cfg)
        p_ref = oracle.spot_price(p, g_ref)
        assert abs(r["value"] - p_ref) <= 1e-10 * abs(p_ref)
        disc = oracle.curve_eval(p, 0, np.array([p.maturity]))[0]
        assert abs(r["error_or_delta"] - abs(r["value"] - disc)) <= 1e-12
    assert np.isfinite(rows[-1]["error_or_delta"])


def test_reference_caplet_is_the_job_default(reference):
    """reference_caplet rebuilds price_caplet's problem for the job defaults: the
    strike is the period forward rate, the axes are MeshSpec::caplet_default's."""
    p = drivers.reference_caplet(11.0, 10.0)
    assert p.shape == (100, 50, 50) and p.instrument == A.INSTRUMENT_CAPLET
    assert p.n_steps == 0 and p.time_levels == A.TIME_REFERENCE  # run()'s own steps and levels
    d = reference.curve_eval(p, 0, np.array([10.0, 11.0]))
    assert p.strike == (d[0] / d[1] - 1.0) / 1.0
    for ax, (c, a, n) in ((p.r, (p.strike / 0.01, 0.05, 100)), (p.v, (0.5, 0.5, 50)), (p.y, (0.0, 0.05, 50))):
        z, j1, j2, _ = reference.sinh_axis(c, a, 0.0, 30.0 if n == 50 and c == 0.5 else 250.0, n)
        assert np.array_equal(ax.z, z) and np.array_equal(ax.j1, j1) and np.array_equal(ax.j2, j2)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fast", "strict"])
def test_bench_rows_match_reference_price_caplet(gpu, reference, mode):
    """cmd_bench's three cases (job.cpp:540-567, paper table) on the
    reference's own 100 x 50 x 50 sinh mesh, against the reference's run() itself."""
    rows = drivers.bench(mode=mode)
    assert [(r["payment_years"], r["expiry_years"]) for r in rows] == [(2.0, 1.0), (11.0, 10.0), (20.0, 19.0)]
    assert [r["n_steps"] for r in rows] == [12, 120, 228]
    for r in rows:
        p = drivers.reference_caplet(r["payment_years"], r["expiry_years"])
        g_ref, rep, _, _ = reference.run(p)  # the unmodified run() (instruments.cpp:234)
        p_ref = reference.spot_price(p, g_ref)
        assert rep["n_steps"] == r["n_steps"]
        assert abs(r["price"] - p_ref) <= 1e-10 * abs(p_ref), (r, p_ref)
        assert r["paper_seconds"] is not None and r["wall_seconds"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("maturity", [1.0, 10.0, 20.0])
def test_collapsed_v_axis_runs_fast_and_matches_reference(gpu, reference, maturity):
    """price_zcb's default mesh (100 x 1 x 40, collapsed v axis; instruments.cpp:140-143,
    173-208) on the FAST four-kernel schedule without its v sweep (solver.cpp:136),
    against the reference's run() on the same problem, and the SPEC acceptance bound
    against the closed form (< 1e-5)."""
    p = drivers.reference_zcb(maturity)
    assert p.shape == (100, 1, 40)
    with hj.Solver([p], mode="fast") as s:
        s.run()
        price = float(s.spot_prices()[0])
        g = s.grid(0)
        assert s.last_launches() >= 3 * s.n_steps  # explicit, r-lines, y-lines: no v sweep
    g_ref, rep, _, _ = reference.run(p)
    p_ref = reference.spot_price(p, g_ref)
    assert abs(price - p_ref) <= 1e-10 * abs(p_ref), (price, p_ref)
    assert np.max(np.abs(g - g_ref)) <= 1e-10 * np.max(np.abs(g_ref))
    disc = reference.curve_eval(p, 0, np.array([maturity]))[0]
    assert abs(price - disc) < 1e-5
