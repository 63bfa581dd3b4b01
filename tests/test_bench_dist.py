"""bench.py's multi-process host logic on CPU (gloo, world_size 2): replicas
only — each rank times its own sort, the job time is the max
over ranks and the value is N * n / time."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = bench.dist_env()
    ms_total = 100.0 + 50.0 * rank          # rank 1 is the slow one
    mx = bench.reduce_max(ms_total, w)
    value, ms_step = bench.aggregate(1 << 20, mx, steps=10, world=w)
    q.put((r, w, lr, mx, value, ms_step))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_timing_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (rank, w, lr, mx, value, ms_step) in enumerate(res):
        assert (rank, w, lr) == (r, world, r)
        assert mx == pytest.approx(150.0)             # max over ranks
        assert ms_step == pytest.approx(15.0)
        assert value == pytest.approx(world * (1 << 20) / 15e-3 / 1e9)


def test_single_process_aggregate():
    assert bench.reduce_max(3.0, 1) == 3.0
    v, ms = bench.aggregate(1 << 28, 260.0, steps=10, world=1)
    assert ms == pytest.approx(26.0) and v == pytest.approx((1 << 28) / 26e-3 / 1e9)
