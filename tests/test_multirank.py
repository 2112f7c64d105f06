"""N>1 plumbing of the decode bench on CPU (gloo, world size 2): request / KV-head sharding covers
every (request, KV head) exactly once, and timings reduce as the max over ranks."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import importlib.util
import pathlib
import sys

# host-only helper module of the package, loaded by path so that this test (and its spawned
# workers) runs without the CUDA library
_spec = importlib.util.spec_from_file_location(
    "mv_shard", pathlib.Path(__file__).resolve().parent.parent / "paper_2506_09991_b200" / "shard.py")
_shard = importlib.util.module_from_spec(_spec)
sys.modules["mv_shard"] = _shard  # dataclasses resolve annotations through sys.modules
_spec.loader.exec_module(_shard)
shard_requests, shard_heads, max_over_ranks = _shard.shard_requests, _shard.shard_heads, _shard.max_over_ranks


@pytest.mark.parametrize("total,heads,world", [(64, 8, 1), (64, 8, 2), (64, 8, 8), (63, 8, 4), (2, 8, 4), (1, 8, 8),
                                               (3, 8, 2)])
def test_shards_partition_requests_and_heads(total, heads, world):
    seen = {}
    for rank in range(world):
        s = shard_requests(total, heads, world, rank)
        for r in s.requests:
            for h in range(*s.kv_heads):
                assert (r, h) not in seen
                seen[(r, h)] = rank
    assert len(seen) == total * heads


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_head_groups_partition(world):
    seen = set()
    for rank in range(world):
        s = shard_heads(16, 8, world, rank)
        assert s.requests == tuple(range(16))
        for h in range(*s.kv_heads):
            assert h not in seen
            seen.add(h)
    assert seen == set(range(8))
    with pytest.raises(ValueError):
        shard_heads(16, 8, 3, 0)


def _gather_worker(rank, world, port, q):
    """The layer-level collective on CPU: head-sharded outputs all-gathered in rank order."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = shard_heads(3, 8, world, rank)
        hq_l = (s.kv_heads[1] - s.kv_heads[0]) * 5
        out = torch.full((6, hq_l, 4), float(rank))
        g = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(g, out)
        full = torch.cat(g, dim=1)  # [tokens, 40 heads, d]: head h from rank h // hq_l
        q.put((rank, full[:, :, 0].tolist()))
    finally:
        dist.destroy_process_group()


def test_head_sharded_allgather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, full in res:
        assert all(row == [0.0] * 20 + [1.0] * 20 for row in full)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = [1.0 + rank, 10.0 - rank]  # rank 1 is slower on value 0, rank 0 on value 1
        q.put((rank, max_over_ranks(mine), shard_requests(16, 8, world, rank).requests))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
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
    assert res[0][1] == res[1][1] == [2.0, 10.0]
    assert set(res[0][2]) | set(res[1][2]) == set(range(16)) and not set(res[0][2]) & set(res[1][2])
