"""world_size-2 gloo check (CPU) of the multi-GPU replica plumbing: shards are
disjoint and covering, and the timing/count reduction is MAX/SUM."""

import os
import socket

import pytest
import torch.multiprocessing as tmp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2012_08238_b200.replicas import combine, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = list(shard(1000, rank, world))
    ms, cnt = combine(10.0 + 5.0 * rank, len(mine))
    out[rank] = (mine[0], mine[-1], ms, cnt)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_cover():
    from paper_2012_08238_b200.replicas import shard
    for total in (0, 1, 7, 1000):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in shard(total, r, world)]
            assert got == list(range(total))


def test_gloo_world2():
    mgr = tmp.Manager()
    out = mgr.dict()
    port = _free_port()
    tmp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][:2] == (0, 499) and out[1][:2] == (500, 999)
    for r in (0, 1):
        assert out[r][2] == 15.0 and out[r][3] == 1000
