"""Full-length goldens for BASELINE configs 1-4, from the COMPILED REFERENCE.

TEST INFRASTRUCTURE ONLY. Run in the container where /root/reference exists
(oracle/_ref/libhjmsv_ref.so built by `make -C oracle`):

    python tests/golden/make_full_golden.py 1      # ~12 min, 1 core
    python tests/golden/make_full_golden.py 2      # 64 caplets, all cores
    python tests/golden/make_full_golden.py 3      # ~2.7 h, 1 core
    python tests/golden/make_full_golden.py 4      # 1024 problems, all cores

Each problem is marched through the reference's own douglas_step for the FULL
step count of BASELINE.json (the harness of SURVEY §8c: run() at
solver.cpp:213-258 with indexed time levels). A full config-3 grid is 268 MB,
so a fixture keeps, per problem: the spot price (interpolate_at,
instruments.cpp:71-88), status code, failed step, last_max_delta, whole-grid
checksums (sum, sum of squares, min, max, max|U|), per-r-plane sums, and the
values at a fixed seeded set of flat grid indices (stored with the indices).
The GPU tests (tests/test_full_parity.py) compare the device grid at those
indices normwise against max|U_ref| and the plane sums / checksums relatively.
"""
from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import bindings as B  # noqa: E402
from paper_1108_1688_b200 import workloads as W  # noqa: E402
from make_golden import fingerprint  # noqa: E402

# seeded sample sizes per problem (single grids get more points)
SAMPLE = {1: 65536, 2: 2048, 3: 65536, 4: 256}
SEED = 0x1108_1688_2


def sample_indices(config_id: int, size: int) -> np.ndarray:
    rng = np.random.default_rng(SEED + config_id)
    idx = rng.choice(size, size=min(SAMPLE[config_id], size), replace=False)
    return np.sort(idx).astype(np.int64)


def one(ref, p, idx):
    t0 = time.time()
    g, rep, code, msg = ref.run(p, raise_on_error=False)
    out = {"code": code, "failed_step": rep["failed_step"], "steps_done": rep["steps_done"],
           "max_delta": rep["last_max_delta"], "message": msg, "seconds": time.time() - t0}
    if code == 0:
        flat = g.reshape(-1)
        out["price"] = ref.spot_price(p, g)
        out["checksum"] = np.array([flat.sum(), (flat * flat).sum(), flat.min(), flat.max(),
                                    np.abs(flat).max()])
        out["plane_sums"] = g.reshape(p.shape[0], -1).sum(axis=1)
        out["sample"] = flat[idx].copy()
    else:
        out["price"] = np.nan
        out["checksum"] = np.full(5, np.nan)
        out["plane_sums"] = np.full(p.shape[0], np.nan)
        out["sample"] = np.full(idx.shape[0], np.nan)
    return out


def main(config_id: int, threads: int):
    ref = B.reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    probs = W.make_config(config_id)
    idx = sample_indices(config_id, probs[0].size)
    t0 = time.time()
    if threads <= 1 or len(probs) == 1:
        res = [one(ref, p, idx) for p in probs]
    else:
        # ctypes drops the GIL, so the reference marches run concurrently —
        # the caplet_ladder pattern (instruments.cpp:242-264)
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(lambda p: one(ref, p, idx), probs))
    out = {
        "indices": idx,
        "prices": np.array([r["price"] for r in res]),
        "codes": np.array([r["code"] for r in res], dtype=np.int32),
        "failed_step": np.array([r["failed_step"] for r in res], dtype=np.int32),
        "steps_done": np.array([r["steps_done"] for r in res], dtype=np.int32),
        "max_delta": np.array([r["max_delta"] for r in res]),
        "checksum": np.stack([r["checksum"] for r in res]),
        "plane_sums": np.stack([r["plane_sums"] for r in res]),
        "sample": np.stack([r["sample"] for r in res]),
    }
    path = os.path.join(HERE, f"full_config{config_id}.npz")
    np.savez_compressed(path, **out)
    meta = {"config": config_id, "problems": len(probs), "steps": probs[0].n_steps,
            "shape": list(probs[0].shape), "fingerprints": [fingerprint(p) for p in probs],
            "messages": {str(q): r["message"] for q, r in enumerate(res) if r["code"]},
            "wall_seconds": time.time() - t0, "threads": threads,
            "cpu_seconds_per_problem": [round(r["seconds"], 2) for r in res]}
    with open(os.path.join(HERE, f"full_config{config_id}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"config {config_id}: {len(probs)} problems in {time.time() - t0:.0f} s; "
          f"failed {[q for q, r in enumerate(res) if r['code']]}; prices {out['prices'][:4]}")


if __name__ == "__main__":
    cid = int(sys.argv[1])
    nthreads = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    main(cid, nthreads)
