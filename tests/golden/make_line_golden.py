"""Worst-conditioned tridiagonal lines + the reference's Thomas solutions.

TEST INFRASTRUCTURE ONLY. Run where oracle/_ref exists (make -C oracle):
    python tests/golden/make_line_golden.py
writes tests/golden/lines.npz, consumed by tests/test_lines.py.

Lines are assembled by the reference's own SpatialOperator::assemble_line_r/v/y
(discretization.cpp:194-300) at the first step's t_mid and theta*dt, and solved
by its thomas_solve_inplace (solver.cpp:22-57):
  * config 4: of the five problems with the largest dt * lambda^2 (SURVEY §7
    hard part 3 — the least diagonally dominant lines of any config), the one
    with the worst y-line; every line of every axis of it scanned, the 48 lines
    with the largest interior (|l|+|u|)/|d| kept per axis (r: 64 rows = 4
    segments; v, y: 32 rows = 2 segments). Worst ratios r / v / y: 0.995 /
    0.787 / 3.94 (problem 301, dt 0.0473);
  * config 3 (rho = -0.9): 32 r-lines of 512 rows (32 segments: the lane scan
    at full width) and 32 y-lines of 256 rows (16 segments);
  * the super2 fold's lag branch (|upper[1]| <= 1e-300, solver.cpp:36-39): the
    worst y-line with upper[1] set to 0.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings as B  # noqa: E402
from paper_1108_1688_b200 import workloads as W  # noqa: E402


def ratio(lo, di, up):
    r = (np.abs(lo[1:-1]) + np.abs(up[1:-1])) / np.abs(di[1:-1])
    return float(r.max()) if r.size else 0.0


def lines_of(ref, p, axis, pairs, t, th):
    out = []
    for a, b in pairs:
        lo, di, up, s2 = ref.assemble_line(p, axis, a, b, t, th)
        out.append((lo, di, up, s2, ratio(lo, di, up)))
    return out


def pack(lines, rng):
    lo = np.stack([x[0] for x in lines])
    di = np.stack([x[1] for x in lines])
    up = np.stack([x[2] for x in lines])
    s2 = np.array([x[3] for x in lines])
    rhs = rng.standard_normal(lo.shape)
    return lo, di, up, s2, rhs, np.array([x[4] for x in lines])


def main():
    ref = B.reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(1108_1688)
    out = {}

    probs = W.make_config(4)
    # the y-line ratio grows with theta*dt*g6 ~ dt * lambda^2 (g6 = (2 a_i v - 2 kappa y)/J_y,
    # a_i ~ lambda^2): scan the five problems with the largest dt * lambda^2, keep the worst
    cand = np.argsort([-(p.maturity / p.n_steps) * p.lam ** 2 for p in probs])[:5]
    best = None
    for q in cand:
        p = probs[int(q)]
        dt = p.maturity / p.n_steps
        nr, nv, ny = p.shape
        ys = lines_of(ref, p, 2, [(i, j) for i in range(nr) for j in range(nv)], p.maturity - 0.5 * dt, 0.5 * dt)
        w = max(x[4] for x in ys)
        if best is None or w > best[0]:
            best = (w, int(q))
    q = best[1]
    p = probs[q]
    dt = p.maturity / p.n_steps
    t, th = p.maturity - 0.5 * dt, 0.5 * dt
    nr, nv, ny = p.shape
    grids = {0: [(j, k) for j in range(nv) for k in range(ny)],
             1: [(i, k) for i in range(nr) for k in range(ny)],
             2: [(i, j) for i in range(nr) for j in range(nv)]}
    worst_y = None
    for axis, name in ((0, "r"), (1, "v"), (2, "y")):
        ls = lines_of(ref, p, axis, grids[axis], t, th)
        ls.sort(key=lambda x: -x[4])
        keep = ls[:48]
        if axis == 2:
            worst_y = keep[0]
        lo, di, up, s2, rhs, rt = pack(keep, rng)
        x, code, _ = ref.thomas(lo, di, up, s2, rhs)
        assert code == 0
        out.update({f"c4{name}_lower": lo, f"c4{name}_diag": di, f"c4{name}_upper": up,
                    f"c4{name}_s2": s2, f"c4{name}_rhs": rhs, f"c4{name}_x": x, f"c4{name}_ratio": rt})
        print(f"config 4 problem {q} (dt {dt:.4f}) {name}-lines: worst ratio {rt.max():.3f}, "
              f"super2 != 0 on {(s2 != 0).sum()}")

    # lag branch of the super2 fold
    lo, di, up, s2 = (np.array(v, dtype=float) for v in worst_y[:4])
    up = up.copy()
    up[1] = 0.0
    rhs = rng.standard_normal(lo.shape)
    x, code, _ = ref.thomas(lo[None], di[None], up[None], np.array([s2]), rhs[None])
    assert code == 0 and s2 != 0.0
    out.update(lag_lower=lo[None], lag_diag=di[None], lag_upper=up[None], lag_s2=np.array([s2]),
               lag_rhs=rhs[None], lag_x=x)

    # long lines of config 3
    p3 = W.make_problem(3, 0)
    dt3 = p3.maturity / p3.n_steps
    t3, th3 = p3.maturity - 0.5 * dt3, 0.5 * dt3
    nr3, nv3, ny3 = p3.shape
    pick = rng.choice(nv3 * ny3, 32, replace=False)
    ls = lines_of(ref, p3, 0, [(int(v) // ny3, int(v) % ny3) for v in pick], t3, th3)
    lo, di, up, s2, rhs, rt = pack(ls, rng)
    x, code, _ = ref.thomas(lo, di, up, s2, rhs)
    assert code == 0
    out.update(c3r_lower=lo, c3r_diag=di, c3r_upper=up, c3r_s2=s2, c3r_rhs=rhs, c3r_x=x, c3r_ratio=rt)
    pick = rng.choice(nr3 * nv3, 32, replace=False)
    ls = lines_of(ref, p3, 2, [(int(v) // nv3, int(v) % nv3) for v in pick], t3, th3)
    lo, di, up, s2, rhs, rt = pack(ls, rng)
    x, code, _ = ref.thomas(lo, di, up, s2, rhs)
    assert code == 0
    out.update(c3y_lower=lo, c3y_diag=di, c3y_upper=up, c3y_s2=s2, c3y_rhs=rhs, c3y_x=x, c3y_ratio=rt)
    print(f"config 3 r-lines {out['c3r_x'].shape}, y-lines {out['c3y_x'].shape}")
    np.savez_compressed(os.path.join(HERE, "lines.npz"), **out)


if __name__ == "__main__":
    main()
