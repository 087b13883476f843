"""Multi-rank host logic of the cross-section sharding on CPU (gloo,
world_size 2): every section owned exactly once, balanced, and the timing
reductions used by bench.py (max over ranks, sum of work)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_03812_b200.shard import max_over_ranks, section_shard, sum_over_ranks


@pytest.mark.parametrize("world", [1, 2, 4, 8, 3])
def test_shards_cover_all_sections_once(world):
    owned = [section_shard(256, r, world) for r in range(world)]
    flat = sorted(i for o in owned for i in o)
    assert flat == list(range(256))
    assert max(map(len, owned)) - min(map(len, owned)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = section_shard(256, rank, world)
    t = max_over_ranks(10.0 + rank, dist)
    units = sum_over_ranks(float(len(mine)), dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, t, units, gathered))


def test_gloo_world2_reductions():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, units, gathered in res:
        assert t == 11.0  # max over ranks
        assert units == 256.0
        flat = sorted(i for g in gathered for i in g)
        assert flat == list(range(256))
