#!/usr/bin/env python3
"""bench.py — Douglas-ADI march throughput (grid-point-steps/s) on B200.

Contract (one JSON line on rank 0):
  * a bench "step" = one full march of the configured workload (default
    BASELINE config 1: ZCB 256x128x128, 1000 ADI steps), inputs resident in HBM;
    W untimed warm-up marches, then K timed marches, each bracketed by CUDA
    events on the solver's stream; L2 is flushed (256 MiB write) between timed
    marches; timing is the max over ranks.
  * value  = all ranks' grid-point-steps / max-rank time (whole job).
  * e2e    = the same metric through the C-ABI with HOST buffers: descriptor ->
    hjmsv_solver_create (lowering, terminal level, H2D) -> run -> spot prices +
    final grid D2H -> destroy, wall-clock per call.
  * roofline: dominant kernel, algorithmic bytes per launch (SURVEY §8d
    accounting) / its CUDA-event duration measured live, vs MEASURED_PEAKS.json.
  * cpu_baseline: oracle/_ref (the compiled reference) on a bounded prefix of
    the same workload, 1 core (the reference has no intra-solve parallelism).
  * --impl reference: the reference CPU solver itself (oracle/_ref, else the
    oracle restatement), all host threads as independent replicas through the
    reference's caplet_ladder-style pool; rank 0 only.
Multi-GPU (torchrun): batched configs shard problems contiguously (no data-path
collective); single-grid configs run one replica per rank.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point-updates/sec (pts×ADI steps/s) per GPU & box; % of HBM roofline"
UNIT = "pt-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--mode", default="fast", choices=["fast", "strict"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="one warm march, for ncu")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(count: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of ceil(count/world) problems."""
    per = (count + world - 1) // world
    lo = min(count, rank * per)
    return lo, min(count, lo + per)


def workload(config: int, rank: int, world: int):
    from paper_1108_1688_b200 import workloads as W
    cs = W.CONFIGS[config]
    if cs.problems == 1:
        probs = [W.make_problem(config, 0)]       # replica per rank
        scaling = "weak"
    else:
        lo, hi = shard(cs.problems, rank, world)
        probs = [W.make_problem(config, q) for q in range(lo, hi)]
        scaling = "strong"
    return cs, probs, scaling


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: wait for its first sample so that
            # short timed regions (config 0) are sampled too
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for q, nm in enumerate(names):
                if len(r) > 5 + q and r[5 + q].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def l2_flusher():
    import torch
    buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    return lambda: buf.fill_(1.0)


def cpu_baseline_sample(config: int):
    """oracle/_ref (else the restatement) on a bounded prefix, 1 core."""
    from oracle import bindings as B
    from paper_1108_1688_b200 import workloads as W
    chk = B.reference()
    kind = "reference"
    if chk is None:
        chk, kind = B.restatement(), "port"
    p = W.make_problem(config, 0)
    pts = p.size
    steps = max(1, min(p.n_steps, int(round(6.0e7 / pts))))  # ~10 s of reference work
    t0 = time.perf_counter()
    _, rep, code, _ = chk.run(p, steps=steps, raise_on_error=False)
    dt = time.perf_counter() - t0
    return {"value": pts * steps / dt, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"config {config} ({p.shape[0]}x{p.shape[1]}x{p.shape[2]}), first {steps} of "
                      f"{p.n_steps} ADI steps incl. terminal setup, 1 core, {dt:.2f} s"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import bindings as B
    from paper_1108_1688_b200 import workloads as W
    chk = B.reference()
    kind = "reference"
    if chk is None:
        chk, kind = B.restatement(), "port"
    cs = W.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    base = [W.make_problem(args.config, q % cs.problems) for q in range(threads)]
    pts = base[0].size
    # bounded sample per step: each thread advances its own problem a prefix of
    # the march, sized so one step is ~5 s of one core's reference work
    prefix = max(1, min(base[0].n_steps, int(round(3.0e7 / pts))))
    probs = []
    for p in base:
        p.n_steps = p.n_steps  # keep the workload's dt; run only `prefix` steps
        probs.append(p)

    def one_step():
        import concurrent.futures as cf
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
            list(ex.map(lambda p: chk.run(p, steps=prefix, raise_on_error=False), probs))
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    times = [one_step() for _ in range(args.steps)]
    total = sum(times)
    work = threads * pts * prefix * args.steps
    value = work / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"config {args.config}: {cs.description}",
                       "sample": f"{threads} concurrent reference solves x {prefix} ADI steps each"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"{threads} threads, each {prefix} of {base[0].n_steps} ADI steps "
                                       f"of config {args.config} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/ncu_traffic.json), or None if that kernel was not captured."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(kernel)
        return float(ent["dram_bytes"]) if ent else None
    except (OSError, ValueError, KeyError):
        return None


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1108_1688_b200 as hj
    cs, probs, scaling = workload(args.config, rank, world)
    pts_per_march = sum(p.size * p.n_steps for p in probs)

    solver = hj.Solver(probs, device=local, mode=args.mode)
    flush = l2_flusher()

    from paper_1108_1688_b200 import _abi as A
    done_pts = [pts_per_march]
    diverged = [0]

    def march():
        solver.reset()
        solver.step_async(solver.n_steps)
        code = solver.lib.hjmsv_solver_synchronize(solver.h)
        if code not in (A.OK, A.DIVERGED, A.NONFINITE):
            hj.api._check(code)
        if code != A.OK:
            # a problem whose scheme leaves the divergence bound stops where the
            # reference's run() throws (guard_finite, solver.cpp:69-77; divergence
            # parity); only the steps it actually took are counted
            reps = [solver.report(q) for q in range(len(probs))]
            done_pts[0] = sum(p.size * r["steps_done"] for p, r in zip(probs, reps))
            diverged[0] = sum(1 for r in reps if r["status"] != A.OK)
        return solver.last_device_ms()

    if args.profile_only:
        march()
        march()
        return

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else args.warmup):
        march()
    launches = solver.last_launches()

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            torch.cuda.synchronize()
            times.append(march())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    my_ms = sum(times)
    pts_per_march = done_pts[0]
    t = torch.tensor([my_ms, float(pts_per_march)], dtype=torch.float64, device="cuda")
    if dist:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
        total_ms, total_pts = float(tmax[0]), float(tsum[1])
    else:
        total_ms, total_pts = my_ms, float(pts_per_march)
    value = total_pts * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # live per-kernel roofline: dominant kernel of one march
    solver.reset()
    prof, _ = solver.kernel_profile(solver.n_steps)
    march_ms = ms_per_step or 1.0  # the measured march (one bench step) on this rank
    # the dominant per-step kernel (fx_faces runs once per launched march)
    dom = max((k for k in prof if k["name"] != "fx_faces"), key=lambda k: k["avg_ms"])
    peak, peak_kind = measured_peak()
    achieved = dom["alg_bytes"] / (dom["avg_ms"] / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom["name"]), "kernel": dom["name"],
                "kernel_share_of_step": dom["avg_ms"] * solver.n_steps / march_ms,
                "peak_kind": peak_kind,
                "step_equiv_GBps": total_pts * args.steps * 40.0 / (total_ms / 1e3) / 1e9 / world,
                "step_equiv_frac": total_pts * args.steps * 40.0 / (total_ms / 1e3) / 1e9 / world / peak,
                "kernels": [{"name": k["name"], "avg_us": 1e3 * k["avg_ms"],
                             "alg_GBps": k["alg_bytes"] / (k["avg_ms"] / 1e3) / 1e9 if k["avg_ms"] else None}
                            for k in prof]}

    # end to end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        from paper_1108_1688_b200 import _abi as A
        import ctypes
        import numpy as np
        from paper_1108_1688_b200.problem import problems_to_c, _ptr
        lib = A.load()
        cfg = hj.SolverConfig().to_c()
        mode = hj.api._mode(args.mode)
        arr = problems_to_c(probs)
        grids = np.empty(sum(p.size for p in probs))
        prices = np.empty(len(probs))
        e2e_t = []
        reps = max(1, min(3, args.steps))
        for it in range(reps + 1):
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            h = ctypes.c_void_p()
            code = lib.hjmsv_solver_create(arr, len(probs), ctypes.byref(cfg), local, mode, ctypes.byref(h))
            assert code == 0, lib.hjmsv_last_error()
            rc = lib.hjmsv_solver_run(h)
            assert rc in (A.OK, A.DIVERGED, A.NONFINITE), lib.hjmsv_last_error()
            assert lib.hjmsv_solver_spot_prices(h, _ptr(prices)) == 0
            assert lib.hjmsv_solver_get_grids(h, _ptr(grids)) == 0  # every level, one copy
            lib.hjmsv_solver_destroy(h)
            el = time.perf_counter() - t0
            if it > 0:
                e2e_t.append(el)
        el = torch.tensor([sum(e2e_t)], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        # descriptor tables per problem: axes, per-step scalars, FAST factor tables,
        # constants, readout corners; the terminal level is built on the device in
        # FAST mode and uploaded only in STRICT mode
        def h2d_bytes(p):
            nr, nv, ny = p.r.n, p.v.n, p.y.n
            b = 8 * (5 * nr + 3 * nv + 3 * ny) + 8 * 32 * p.n_steps + 256 + 8 * 16 + 48
            b += 8 * (8 * nr + 10 * nv + 4 * ny) if args.mode == "fast" else 8 * p.size
            return b
        h2d = sum(h2d_bytes(p) for p in probs)
        d2h = sum(8 * p.size for p in probs) + 8 * len(probs)
        e2e = {"value": total_pts * reps / float(el[0]), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "note": "per step: create(lower + descriptor H2D + device terminal) -> run -> spot prices + grid D2H -> destroy"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(args.config)
        except Exception as exc:  # the checker is reported, never measured as product
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "unavailable", "sample": str(exc)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"config {args.config}: {cs.description}",
                           "problems_per_rank": len(probs), "mode": args.mode,
                           "diverged_problems": diverged[0],
                           "step": "one full march (all ADI steps) per bench step",
                           "l2": "256 MiB write between timed marches; a march's own state is "
                                 "carried step to step on device"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches * args.steps),
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    solver.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
