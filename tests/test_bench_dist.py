"""The N>1 host logic of bench.py on CPU: world_size 2 over gloo (127.0.0.1).

The path does not shard: each rank runs
its own replica, the job time is the max over ranks and the whole-job value is
world x units / that time.  The reference arm runs on rank 0 only."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, r, loc = bench.dist_env()
        ms = bench.max_over_ranks(10.0 + 5.0 * rank, w, "cpu")      # rank 1 is slower
        rate = bench.job_rate(w, 1000 * 7, ms * 1e-3)

        class A:
            config, ref_sample, steps, warmup, impl = "C1", 64, 1, 3, "reference"
        rc_ref = bench.run_reference(A) if rank == 1 else None       # non-zero ranks: no work
        dist.barrier()
        q.put((rank, w, r, loc, ms, rate, rc_ref))
    finally:
        dist.destroy_process_group()


def test_two_rank_aggregation_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, w, r, loc, ms, rate, _ in res:
        assert (w, r, loc) == (world, rank, rank)
        assert ms == pytest.approx(15.0)                           # max over ranks
        assert rate == pytest.approx(world * 7000 / 15e-3)         # whole-job value
    assert res[1][6] == 0                                           # reference arm: rank 1 exits 0


def test_single_rank_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(3.5, 1, "cpu") == 3.5
    assert bench.job_rate(1, 100, 2.0) == 50.0


def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (here the
    reference arm, which needs no GPU): exactly one JSON line, from rank 0, with
    n_gpus = 2."""
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "C1", "--steps", "1", "--warmup", "3", "--ref-sample", "64"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2, r.stdout
