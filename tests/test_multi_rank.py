"""N > 1 path on CPU (gloo, world_size 2): batch sharding covers every unit exactly once,
per-unit scalars come back in global order on every rank, and the job time is the max over
ranks."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2105_01586_b200 import multi  # noqa: E402


def test_shard_partitions_the_batch():
    for n in (0, 1, 5, 32, 33):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in multi.shard(n, r, world)]
            assert got == list(range(n))
            sizes = [len(multi.shard(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        multi.shard(4, 2, 2)


def test_not_distributed_identity():
    assert multi.max_over_ranks(3.5) == 3.5
    np.testing.assert_array_equal(multi.gather_scalars(np.arange(4.0), 4), np.arange(4.0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = multi.shard(n, rank, world)
        # per-unit "MSE" computed by this rank for its shard only: a function of the unit index
        local = np.array([1.0 + 0.5 * i for i in mine])
        allv = multi.gather_scalars(local, n)
        t = multi.max_over_ranks(10.0 + rank)
        q.put((rank, list(mine), allv.tolist(), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [32, 7])
def test_gloo_world2_shard_and_gather(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    covered = sorted(i for _, mine, _, _ in res for i in mine)
    assert covered == list(range(n))
    expect = [1.0 + 0.5 * i for i in range(n)]
    for rank, mine, allv, t in res:
        assert allv == expect  # every rank sees the whole batch in global order
        assert t == 10.0 + (world - 1)  # max over ranks
