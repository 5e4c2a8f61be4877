"""World-size-2 gloo run of the batch driver's host logic on CPU.

Each rank takes its contiguous shard (bench.shard), prices it with
the CPU checker (the device path needs a GPU; the sharding, gather and
max-over-ranks timing logic is what is under test), and the gathered prices
must equal a single-process run. No data-path collective exists; the only
exchange is the final gather.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import bindings as B
    from paper_1108_1688_b200 import workloads as W
    count = 6
    lo, hi = bench.shard(count, rank, world)
    probs = [W.make_problem(4, q, nr=12, nv=6, ny=6, steps=10) for q in range(lo, hi)]
    prices, _, code = B.restatement().batch_run(probs, threads=1)
    assert code == 0
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, prices.tolist()))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py's max-over-ranks timing
    if rank == 0:
        flat = [None] * count
        for a, b, pr in gathered:
            flat[a:b] = pr
        out.put((flat, float(t[0])))
    dist.destroy_process_group()


def test_gloo_world2_sharded_batch_matches_single_process(oracle):
    from paper_1108_1688_b200 import workloads as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    flat, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    probs = [W.make_problem(4, i, nr=12, nv=6, ny=6, steps=10) for i in range(6)]
    ref, _, code = oracle.batch_run(probs, threads=2)
    assert code == 0
    assert np.array_equal(np.array(flat), ref)
    assert tmax == 2.0


@pytest.mark.gpu
def test_bench_two_ranks_shard_the_batched_config(gpu):
    """bench.py --gpus 2 relaunches itself under torch.distributed.run; the two
    ranks (sharing the box's device when it has one) take contiguous halves of
    config 2's 64 caplets (strong scaling, no data-path collective) and rank 0
    prints the job's line: max-over-ranks time, the sum of both ranks' work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "2",
                          "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--batched-config", "-1"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["problems_per_rank"] == 32
    # all 64 caplets' steps counted (problem 41 diverges at step 372 in both solvers)
    assert line["value"] > 0 and line["gpu_launches"] > 0
