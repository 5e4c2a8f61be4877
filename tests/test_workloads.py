"""Seeded workload generator and the bench sharding logic."""
import numpy as np
import pytest

from paper_1108_1688_b200 import _abi as A
from paper_1108_1688_b200 import workloads as W
from paper_1108_1688_b200.problem import mix_seed


def test_mix_seed_matches_reference(reference):
    for s in (0, 1, 63, 64, 65535, 2**40 + 3):
        assert mix_seed(0x11081688 ^ 2, s) == reference.lib.ref_mix_seed(0x11081688 ^ 2, s)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_config_shapes_and_ranges(cfg):
    cs = W.CONFIGS[cfg]
    probs = W.make_config(cfg, count=min(cs.problems, 64))
    for p in probs:
        assert p.shape == (cs.nr, cs.nv, cs.ny) and p.n_steps == cs.steps
        assert 0.01 <= p.kappa <= 0.2 and 0.5 <= p.theta <= 3.0 and 0.1 <= p.eps <= 0.6
        assert (p.rho == -0.9) if cfg == 3 else (-0.7 <= p.rho <= 0.7)
        assert p.gamma == 0.9 and p.r0 == 0.01 and p.time_levels == A.TIME_INDEXED
        assert np.all(np.diff(p.curve_discounts) < 0) and p.curve_maturities[-1] == 30.0
        if cfg in (0, 1):
            assert p.maturity == 5.0 and p.instrument == A.INSTRUMENT_ZCB
        if cfg == 3:
            assert p.maturity == 10.0
        if cfg in (2, 4):
            assert 1.0 <= p.maturity <= 10.0
            if p.instrument == A.INSTRUMENT_CAPLET:
                assert p.payment == p.maturity + 0.25 and 0.01 <= p.strike <= 0.06
    if cfg == 2:
        assert all(p.instrument == A.INSTRUMENT_CAPLET for p in probs)


def test_config4_mixes_instruments():
    kinds = [p.instrument for p in W.make_config(4)]
    assert 300 < sum(kinds) < 724  # ~Bernoulli(1/2) over 1024


def test_generator_is_deterministic():
    a, b = W.make_problem(4, 77), W.make_problem(4, 77)
    assert (a.kappa, a.lam, a.maturity, a.strike) == (b.kappa, b.lam, b.maturity, b.strike)
    assert np.array_equal(a.curve_discounts, b.curve_discounts)


def test_shard_partition():
    import bench
    for count in (1, 7, 64, 1024):
        for world in (1, 2, 3, 4, 8):
            spans = [bench.shard(count, r, world) for r in range(world)]
            covered = [q for lo, hi in spans for q in range(lo, hi)]
            assert covered == list(range(count))
