"""The N > 1 path of bench.py (replicas, max-over-ranks timing) on CPU with
the gloo backend, world_size 2."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t_ms = 10.0 * (rank + 1)          # rank 1 is the slow one
    t_max, value = bench.aggregate(torch, dist, t_ms, 1 << 24, 5, world, "cpu")
    q.put((rank, t_max, value, bench.dist_env()))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t_max, value, env in res:
        assert t_max == pytest.approx(20.0)                   # max over ranks
        assert value == pytest.approx(2 * (1 << 24) * 5 / 0.020)
        assert env[0] == rank and env[1] == world


def test_single_rank_aggregate():
    sys.path.insert(0, ROOT)
    import bench
    t_max, value = bench.aggregate(torch, None, 8.0, 1000, 4, 1, "cpu")
    assert t_max == 8.0 and value == pytest.approx(1000 * 4 / 0.008)
