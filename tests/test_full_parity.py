"""Full-length parity of every BASELINE config against the COMPILED REFERENCE.

The fixtures tests/golden/full_config{1,2,3,4}.npz were produced by
tests/golden/make_full_golden.py: the unmodified reference (oracle/_ref) marched
each problem of the config for its FULL step count (run(), solver.cpp:213-258,
with the indexed time levels of SURVEY §8c). A 268 MB config-3 grid cannot be
committed, so a fixture holds per problem the spot price (interpolate_at,
instruments.cpp:71-88), status and failed step, last_max_delta, whole-grid
checksums, per-r-plane sums and the values at a fixed seeded set of grid
indices. The device grid is compared at those indices normwise against the
reference's max|U|, and through its plane sums and checksums (size-independent
properties of the whole grid).

Bar (BASELINE north_star), per problem, FP64:
  |p_gpu - p_ref| <= 1e-10 |p_ref|,   max_q |U_gpu,q - U_ref,q| <= 1e-10 max|U_ref|.
Problems whose reference march trips guard_finite must be flagged with the same
status at the same step (divergence parity).
"""
import json
import os

import numpy as np
import pytest

import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import _abi as A
from paper_1108_1688_b200 import workloads as W

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10           # north_star parity tolerance (relative, FP64)
STRICT_TOL = 1e-13    # STRICT keeps the reference's operation order


def golden(config):
    path = os.path.join(HERE, f"full_config{config}.npz")
    if not os.path.exists(path):
        pytest.skip(f"missing fixture {path} (tests/golden/make_full_golden.py {config})")
    with open(os.path.join(HERE, f"full_config{config}.json")) as f:
        meta = json.load(f)
    return dict(np.load(path)), meta


def march(probs, mode):
    """Full march of one handle; returns (grids, prices, reports) — grids as (P, N)."""
    with hj.Solver(probs, mode=mode) as s:
        s.step_async(s.n_steps)
        code = s.lib.hjmsv_solver_synchronize(s.h)
        assert code in (A.OK, A.DIVERGED, A.NONFINITE, A.SINGULAR_PIVOT), code
        reps = [s.report(q) for q in range(len(probs))]
        grids = s.grids().reshape(len(probs), -1)
        prices = s.spot_prices()
    return grids, prices, reps


def check(config, probs, grids, prices, reps, gold, tol):
    worst_grid = worst_price = 0.0
    failed = 0
    for q, (p, rep) in enumerate(zip(probs, reps)):
        code = int(gold["codes"][q])
        if code != 0:  # divergence parity: same status at the same step
            failed += 1
            assert rep["status"] == code, (q, rep["status"], code)
            assert rep["failed_step"] == int(gold["failed_step"][q]), (q, rep["failed_step"])
            continue
        assert rep["status"] == 0 and rep["steps_done"] == p.n_steps, (q, rep)
        g = grids[q]
        maxabs = float(gold["checksum"][q][4])
        samp = g[gold["indices"]]
        err = float(np.max(np.abs(samp - gold["sample"][q]))) / maxabs
        assert err <= tol, f"problem {q}: sampled grid normwise rel err {err:.3e}"
        # whole-grid properties: every value enters these
        planes = g.reshape(p.shape[0], -1).sum(axis=1)
        perr = float(np.max(np.abs(planes - gold["plane_sums"][q]))) / (maxabs * p.shape[1] * p.shape[2])
        assert perr <= tol, f"problem {q}: plane sums rel err {perr:.3e}"
        cs = np.array([g.sum(), float(np.max(np.abs(g)))])
        cerr = float(np.max(np.abs(cs - gold["checksum"][q][[0, 4]]) / np.array([maxabs * g.size, maxabs])))
        assert cerr <= tol, f"problem {q}: checksum rel err {cerr:.3e}"
        pr = float(gold["prices"][q])
        prel = abs(prices[q] - pr) / abs(pr)
        assert prel <= TOL, f"problem {q}: price rel err {prel:.3e} ({prices[q]} vs {pr})"
        md = float(gold["max_delta"][q])
        assert abs(rep["last_max_delta"] - md) <= 1e-8 * md + 1e-300, (q, rep["last_max_delta"], md)
        worst_grid, worst_price = max(worst_grid, err, perr), max(worst_price, prel)
    print(f"config {config}: {len(probs)} problems ({failed} diverged in both), "
          f"worst grid rel {worst_grid:.2e}, worst price rel {worst_price:.2e}")


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_full_march_fast(gpu, config):
    gold, meta = golden(config)
    probs = W.make_config(config)
    assert len(probs) == meta["problems"] and probs[0].n_steps == meta["steps"]
    grids, prices, reps = march(probs, "fast")
    check(config, probs, grids, prices, reps, gold, TOL)


@pytest.mark.gpu
def test_full_march_strict_config1(gpu):
    gold, _ = golden(1)
    probs = W.make_config(1)
    grids, prices, reps = march(probs, "strict")
    check(1, probs, grids, prices, reps, gold, STRICT_TOL)


@pytest.mark.gpu
def test_batch_run_two_handles_one_device(gpu):
    """hjmsv_batch_run over devices [0, 0]: two concurrent handles (one host
    thread each, caplet_ladder's fan-out, instruments.cpp:238-266) on config 2's
    64 caplets, every price and status against the reference."""
    gold, _ = golden(2)
    probs = W.make_config(2)
    prices, reps, grids = hj.batch_run(probs, devices=[0, 0], mode="fast", grids=True)
    g = grids.reshape(len(probs), -1)
    check(2, probs, g, prices, reps, gold, TOL)


def test_golden_fingerprints():
    """The fixtures were made from the inputs the workload generator makes today."""
    import sys
    sys.path.insert(0, HERE)
    from make_golden import fingerprint
    for config in (1, 2, 3, 4):
        path = os.path.join(HERE, f"full_config{config}.json")
        if not os.path.exists(path):
            continue  # not generated yet (config 3 takes hours on one core)
        with open(path) as f:
            meta = json.load(f)
        probs = W.make_config(config)
        fps = [fingerprint(p) for p in probs]
        assert fps == meta["fingerprints"], f"config {config}: generator changed since the golden run"
