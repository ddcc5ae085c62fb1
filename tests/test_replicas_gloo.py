"""Multi-process (world_size 2, gloo, CPU) test of the replica aggregation bench.py uses
for --gpus N: max-over-ranks time, summed DOF updates."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms_local = 10.0 + 5.0 * rank           # rank 1 is slower
    dof_local = 1000 * (rank + 1)
    ms, value, w = bench.aggregate(ms_local, dof_local, dist)
    q.put((rank, ms, value, w))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get() for _ in range(2))
    for rank, ms, value, w in out:
        assert w == 2
        assert ms == 15.0                  # max over ranks
        assert abs(value - 3000 / 0.015) < 1e-6   # all ranks' DOF / max time


def test_single_process_aggregation():
    import bench
    ms, value, w = bench.aggregate(20.0, 4000, None)
    assert (ms, w) == (20.0, 1) and abs(value - 4000 / 0.02) < 1e-9
