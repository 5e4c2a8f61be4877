"""Per-kernel device times (device-clock timeline of a directly launched march) for each config.

    python tools/kprofile.py [--mode fast] [--configs 0,1,2,3,4] [--steps 20]
Prints one line per kernel: average us per launch and algorithmic GB/s."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_1688_b200 as hj  # noqa: E402
from paper_1108_1688_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast")
ap.add_argument("--configs", default="0,1,2,3,4")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--count", type=int, default=0, help="limit batch size")
ap.add_argument("--reference-meshes", action="store_true",
                help="also the reference's own meshes: cmd_bench's 100x50x50 caplet (T=19) and "
                     "price_zcb's 100x1x40 bond (T=20)")
a = ap.parse_args()
out = []
from paper_1108_1688_b200 import drivers as D  # noqa: E402
jobs = [(c, None) for c in [int(x) for x in a.configs.split(",") if x != ""]]
if a.reference_meshes:
    jobs += [("caplet_default", [D.reference_caplet(20.0, 19.0)]), ("zcb_default", [D.reference_zcb(20.0)])]
for c, given in jobs:
    if given is None:
        cs = W.CONFIGS[c]
        n = cs.problems if not a.count else min(a.count, cs.problems)
        probs = W.make_config(c, count=n)
    else:
        probs, n = given, len(given)
    t0 = time.time()
    s = hj.Solver(probs, mode=a.mode)
    t_create = time.time() - t0
    s.kernel_profile(2)  # warm
    s.reset()
    prof, launches, total_ms = s.kernel_profile(min(a.steps, s.n_steps - 2), with_total=True)
    step_us = 1e3 * total_ms / min(a.steps, s.n_steps - 2)
    pts = sum(p.size for p in probs)
    rec = {"config": c, "problems": n, "mode": a.mode, "step_us": step_us,
           "pt_steps_per_s": pts / (step_us * 1e-6), "create_s": t_create,
           "equiv_GBps_40B": pts * 40 / (step_us * 1e-6) / 1e9,
           "kernels": [(k["name"], round(k["avg_ms"] * 1e3, 2),
                        round(k["alg_bytes"] / (k["avg_ms"] * 1e-3) / 1e9, 1)) for k in prof]}
    out.append(rec)
    print(json.dumps(rec), flush=True)
    s.close()
