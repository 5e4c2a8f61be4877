#!/usr/bin/env python3
"""bench.py — Douglas-ADI march throughput (grid-point-steps/s) on B200.

Contract (one JSON line on rank 0):
  * a bench "step" = one full march of the configured workload (default
    BASELINE config 3: ZCB 512x256x256, rho = -0.9, 2000 ADI steps — the
    largest single-GPU config), inputs resident in HBM; W untimed warm-up
    marches, then K timed marches, each bracketed by CUDA events on the
    solver's stream; L2 is flushed (256 MiB write) between timed marches (the
    config-3 arrays are 268 MB each, larger than L2, anyway); timing is the max
    over ranks.
  * value  = all ranks' grid-point-steps / max-rank time (whole job).
  * e2e    = the same metric through the C-ABI with HOST buffers: descriptor ->
    hjmsv_solver_create (lowering, device terminal level, H2D) -> run -> spot
    prices + final grid D2H -> destroy, wall-clock per call.
  * roofline: dominant kernel, algorithmic bytes per launch (SURVEY §8d
    accounting) / its duration measured live on the device clock
    in a march launched like the timed one (hjmsv_solver_kernel_timeline), vs
    MEASURED_PEAKS.json; traffic = ncu dram bytes per launch of that kernel on
    this config (profiles/ncu_traffic.json), else null.
  * batched: BASELINE config 2 (64 caplets, 128x64x64, 500 steps) sharded
    contiguously over the ranks (strong scaling, no data-path collective),
    timed the same way in the same run.
  * cpu_baseline: oracle/_ref (the compiled reference) on 1 core, the
    stepping loop only (setup untimed), a few ADI steps of the same workload.
  * --impl reference: the reference CPU solver itself (oracle/_ref, else the
    oracle restatement) on all host threads as independent replicas (the
    caplet_ladder pool pattern); per bench step every thread advances its own
    replica one ADI step (stepping loop only); rank 0 only.
Multi-GPU: `--gpus N` re-executes itself under torch.distributed.run (one rank
per GPU) unless it already runs under it. Single-grid configs run one replica
per rank (weak scaling, "replicas only"); batched configs shard
problems contiguously (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point-updates/sec (pts×ADI steps/s) per GPU & box; % of HBM roofline"
UNIT = "pt-steps/s"
BYTES_PER_PT_STEP = 40.0  # SURVEY §8d two-pass algorithmic traffic


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--batched-config", type=int, default=2,
                    help="batched config timed beside the main line (-1: none)")
    ap.add_argument("--mode", default="fast", choices=["fast", "strict"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="two warm marches, for ncu")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def maybe_relaunch(args):
    """`--gpus N` outside torchrun: re-exec under torch.distributed.run."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


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


def host_cpu():
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


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
            # short timed regions are sampled too
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


def checker():
    """oracle/_ref (the compiled reference) if present, else the C restatement."""
    from oracle import bindings as B
    chk = B.reference()
    if chk is not None:
        return chk, "reference"
    return B.restatement(), "port"


def cpu_baseline_sample(config: int):
    """oracle/_ref on 1 core (the reference has no intra-solve parallelism):
    run()'s setup untimed, then a few douglas_step calls of the same workload,
    timed over the stepping loop only."""
    from paper_1108_1688_b200 import workloads as W
    chk, kind = checker()
    p = W.make_problem(config, 0)
    pts = p.size
    steps = max(1, min(p.n_steps, int(round(1.2e8 / pts))))  # ~15-20 s of reference work
    if kind == "reference":
        ses = chk.session(p)
        secs = ses.steps(steps)
        ses.close()
    else:  # the restatement has no session: a prefix march, setup included
        t0 = time.perf_counter()
        chk.run(p, steps=steps, raise_on_error=False)
        secs = time.perf_counter() - t0
    cpu = host_cpu()
    return {"value": pts * steps / secs, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"config {config} ({p.shape[0]}x{p.shape[1]}x{p.shape[2]}), {steps} of {p.n_steps} "
                      f"ADI steps, stepping loop only (setup untimed), 1 core, {secs:.2f} s",
            "cpu_model": cpu["model"], "nproc": cpu["nproc"]}


def run_reference_arm(args, rank, world):
    """The reference CPU solver on all host threads (rank 0 only)."""
    if rank != 0:
        return
    import concurrent.futures as cf
    from paper_1108_1688_b200 import workloads as W
    chk, kind = checker()
    cs = W.CONFIGS[args.config]
    cpu = host_cpu()
    p0 = W.make_problem(args.config, 0)
    pts = p0.size
    # one replica per host thread, bounded by host memory (~5 arrays per replica)
    threads = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
        threads = max(1, min(threads, int(0.7 * avail // (5 * 8 * pts))))
    except Exception:
        pass
    probs = [W.make_problem(args.config, q % cs.problems) for q in range(threads)]
    # each bench step advances every replica by `per` ADI steps, sized so one
    # bench step is a few seconds of one core's reference work
    per = max(1, min(p0.n_steps, int(round(2.0e7 / pts))))
    if kind == "reference":
        with cf.ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
            sessions = list(ex.map(lambda p: chk.session(p), probs))

        def one_step():
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda s: s.steps(per), sessions))
            return time.perf_counter() - t0
        sample = (f"{threads} concurrent reference replicas, each advancing {per} of {p0.n_steps} ADI steps "
                  f"per bench step (setup untimed, stepping loops only)")
    else:
        def one_step():
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda p: chk.run(p, steps=per, raise_on_error=False), probs))
            return time.perf_counter() - t0
        sample = f"{threads} concurrent restatement solves x {per} ADI steps each (setup included)"

    for _ in range(args.warmup):
        one_step()
    times = [one_step() for _ in range(args.steps)]
    total = sum(times)
    value = threads * pts * per * args.steps / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"config {args.config}: {cs.description}", "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                             "cpu_model": cpu["model"], "nproc": cpu["nproc"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def ncu_traffic(config: int, kernel: str):
    """DRAM bytes per launch of `kernel` on `config` from the committed ncu
    --set full captures (profiles/ncu_traffic.json), or None if not captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(f"config{config}", {}).get(kernel)
        return float(ent["dram_bytes"]) if ent else None
    except (OSError, ValueError, KeyError, AttributeError):
        return None


class Marcher:
    """One handle over this rank's problems; march() = reset + full march on the
    device (graph-replayed after the first), device ms from CUDA events."""

    def __init__(self, probs, device, mode):
        import paper_1108_1688_b200 as hj
        from paper_1108_1688_b200 import _abi as A
        self.hj, self.A = hj, A
        self.probs = probs
        self.solver = hj.Solver(probs, device=device, mode=mode)
        self.done_pts = sum(p.size * p.n_steps for p in probs)
        self.diverged = 0

    def march(self):
        s, A = self.solver, self.A
        s.reset()
        s.step_async(s.n_steps)
        code = s.lib.hjmsv_solver_synchronize(s.h)
        if code not in (A.OK, A.DIVERGED, A.NONFINITE):
            self.hj.api._check(code)
        if code != A.OK:
            # a problem whose scheme leaves the divergence bound stops where the
            # reference's run() throws (guard_finite, solver.cpp:69-77; divergence
            # parity); only the steps it actually took are counted
            reps = [s.report(q) for q in range(len(self.probs))]
            self.done_pts = sum(p.size * r["steps_done"] for p, r in zip(self.probs, reps))
            self.diverged = sum(1 for r in reps if r["status"] != A.OK)
        return s.last_device_ms()

    def close(self):
        self.solver.close()


def timed(marcher, steps, warmup, flush, dist, clk=None, red_dev="cuda"):
    """W warm-up marches, K timed marches (clock sampler `clk` running over the
    timed ones only); returns (max-rank ms, summed pts per march)."""
    import contextlib
    import torch
    for _ in range(warmup):
        marcher.march()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with (clk if clk is not None else contextlib.nullcontext()):
        for _ in range(steps):
            flush()
            torch.cuda.synchronize()
            times.append(marcher.march())
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = torch.tensor([sum(times), float(marcher.done_pts), float(marcher.diverged)], dtype=torch.float64,
                     device=red_dev)
    if dist:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
        marcher.diverged_all = int(tsum[2])
        return float(tmax[0]), float(tsum[1])
    marcher.diverged_all = marcher.diverged
    return float(t[0]), float(t[1])


def main():
    args = parse()
    maybe_relaunch(args)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    # one rank per GPU; with fewer GPUs than ranks (a test of the multi-rank path on
    # one device) ranks share devices round-robin and the host-side reductions go
    # over gloo, as NCCL refuses two ranks on one GPU
    ndev = max(1, torch.cuda.device_count())
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    red_dev = "cuda" if dist is None or dist.get_backend() == "nccl" else "cpu"

    import paper_1108_1688_b200 as hj
    cs, probs, scaling = workload(args.config, rank, world)
    m = Marcher(probs, local, args.mode)
    flush = l2_flusher()

    if args.profile_only:
        m.march()
        m.march()
        return

    warm = max(args.warmup, 3)
    clk = ClockSampler(local)
    total_ms, total_pts = timed(m, args.steps, warm, flush, dist, clk, red_dev)
    launches = m.solver.last_launches()
    value = total_pts * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # live per-kernel roofline: the device timeline of one march launched like
    # the first march of a handle (direct launches + programmatic dependent launch)
    peak, peak_kind = measured_peak()
    roofline = None
    if args.mode == "fast":
        m.solver.reset()
        prof, _, prof_ms = m.solver.kernel_profile(m.solver.n_steps, with_total=True)
        steps_per_march = m.solver.n_steps
        per_step = [k for k in prof if k["name"] != "fx_faces"]  # fx_faces: once per march
        dom = max(per_step, key=lambda k: k["avg_ms"])
        achieved = dom["alg_bytes"] / (dom["avg_ms"] / 1e3) / 1e9
        step_equiv = total_pts * args.steps * BYTES_PER_PT_STEP / (total_ms / 1e3) / 1e9 / world
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": ncu_traffic(args.config, dom["name"]),
                    "kernel": dom["name"], "peak_kind": peak_kind,
                    "alg_bytes_per_launch": dom["alg_bytes"],
                    "kernel_share_of_step": dom["avg_ms"] * steps_per_march / prof_ms,
                    "profiled_march_ms": prof_ms,
                    "step_equiv_GBps": step_equiv, "step_equiv_frac": step_equiv / peak,
                    "kernels": [{"name": k["name"], "avg_us": 1e3 * k["avg_ms"],
                                 "share_of_step": k["avg_ms"] * (1 if k["name"] == "fx_faces" else steps_per_march)
                                 / prof_ms,
                                 "alg_GBps": k["alg_bytes"] / (k["avg_ms"] / 1e3) / 1e9 if k["avg_ms"] else None,
                                 "frac": k["alg_bytes"] / (k["avg_ms"] / 1e3) / 1e9 / peak if k["avg_ms"] else None,
                                 "traffic": ncu_traffic(args.config, k["name"])}
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
        el = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=red_dev)
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
               "note": "per step: create(lower + descriptor H2D + device terminal) -> run -> "
                       "spot prices + grid D2H -> destroy"}
    launches_main = int(launches * args.steps)
    m.close()

    # batched config beside the main line, sharded over the ranks (strong scaling)
    batched = None
    if args.batched_config >= 0 and args.batched_config != args.config:
        bcs, bprobs, bscaling = workload(args.batched_config, rank, world)
        bm = Marcher(bprobs, local, args.mode)
        b_ms, b_pts = timed(bm, args.steps, warm, flush, dist, None, red_dev)
        bval = b_pts * args.steps / (b_ms / 1e3)
        batched = {"workload": f"config {args.batched_config}: {bcs.description}", "value": bval,
                   "unit": UNIT, "ms_per_step": b_ms / args.steps, "scaling": bscaling,
                   "problems_per_rank": len(bprobs), "problems_total": bcs.problems,
                   "diverged_problems": bm.diverged_all,
                   "step_equiv_frac": bval * BYTES_PER_PT_STEP / 1e9 / world / peak,
                   "gpu_launches": int(bm.solver.last_launches() * args.steps)}
        bm.close()

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
                           "diverged_problems": m.diverged_all,
                           "step": "one full march (all ADI steps) per bench step",
                           "l2": "256 MiB write between timed marches; a march's own state is "
                                 "carried step to step on device"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "batched": batched,
                "gpu_launches": launches_main,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
