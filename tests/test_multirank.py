"""N > 1 host logic of bench.py (replicas only) on
CPU with the gloo backend, world_size 2: the max-over-ranks timing and the
whole-job value."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = 1.0 + rank  # rank 1 is the slower one
    tmax = bench.reduce_max(t)
    bench.barrier()
    ws, r, lr = bench.dist_env()
    q.put((rank, tmax, bench.job_value(ws, 10, tmax), ws, r, lr))
    dist.destroy_process_group()


def test_two_rank_max_and_value():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tmax, value, ws, r, lr in out:
        assert tmax == 2.0  # max over ranks, not the local time
        assert value == pytest.approx(2 * 10 / 2.0)  # all solves of all ranks / max time
        assert (ws, r, lr) == (2, rank, rank)


def test_single_rank_identity():
    import bench

    assert bench.reduce_max(3.5) == 3.5
    assert bench.job_value(1, 10, 2.0) == 5.0
