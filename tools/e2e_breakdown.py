"""Where does the end-to-end time of one C-ABI march go? (create, run, readouts, destroy)

    python tools/e2e_breakdown.py [config]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1108_1688_b200 as hj  # noqa: E402
from paper_1108_1688_b200 import _abi as A, workloads as W  # noqa: E402
from paper_1108_1688_b200.problem import problems_to_c, _ptr  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lib = A.load()
probs = W.make_config(cfg_id)
arr = problems_to_c(probs)
cfg = hj.SolverConfig().to_c()
grids = np.empty(sum(p.size for p in probs))
prices = np.empty(len(probs))
for it in range(3):
    t = [time.perf_counter()]
    h = ctypes.c_void_p()
    assert lib.hjmsv_solver_create(arr, len(probs), ctypes.byref(cfg), 0, A.MODE_FAST, ctypes.byref(h)) == 0
    t.append(time.perf_counter())
    lib.hjmsv_solver_step_async(h, probs[0].n_steps)
    t.append(time.perf_counter())
    lib.hjmsv_solver_synchronize(h)
    t.append(time.perf_counter())
    lib.hjmsv_solver_spot_prices(h, _ptr(prices))
    lib.hjmsv_solver_get_grids(h, _ptr(grids))  # every level, one call
    t.append(time.perf_counter())
    lib.hjmsv_solver_destroy(h)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"config {cfg_id} iter {it}: create {d[0]:.1f} ms, enqueue {d[1]:.1f} ms, wait {d[2]:.1f} ms, "
          f"readout {d[3]:.1f} ms, destroy {d[4]:.1f} ms")
