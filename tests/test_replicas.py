"""Multi-process (replicas-only) plumbing of bench.py on CPU with gloo,
world_size 2 (the update chain does not shard; N GPUs run N
independent replicas and the job clock is the max over ranks)."""
import os
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r timed (dev, wall) = (1 + r, 10 - r) seconds
    dev, wall = bench.job_max([1.0 + rank, 10.0 - rank])
    out.put((rank, dev, wall, bench.replica_value(1000, world, dev)))
    dist.barrier()
    dist.destroy_process_group()


def test_job_clock_is_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, dev, wall, value in res:
        assert dev == 2.0 and wall == 10.0  # max over ranks, identical everywhere
        assert value == pytest.approx(1000 * 2 / 2.0)


def test_single_process_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.job_max([3.0, 4.0]) == [3.0, 4.0]
    assert bench.replica_value(500, 1, 2.0) == 250.0


def test_reference_arm_non_zero_rank_exits_silently():
    # under torchrun only rank 0 runs the CPU reference arm
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == ""
