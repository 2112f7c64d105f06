"""Multi-GPU partition of the decode hot path: requests are independent and so
are KV-head groups under GQA, so attention needs no collective.  Requests are sharded across
ranks first; when there are fewer requests than ranks, KV-head groups are split instead.  Timing
is taken on the device and reduced as the max over ranks (the slowest rank bounds the step)."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    requests: tuple[int, ...]   # global request ids this rank serves
    kv_heads: tuple[int, int]   # [first, last) KV heads this rank computes for those requests


def shard_requests(total_requests: int, kv_heads: int, world: int, rank: int) -> Shard:
    """Contiguous request blocks per rank (sizes differ by at most one); with fewer requests than
    ranks, ranks that share a request split its KV heads into equal groups."""
    if world < 1 or not 0 <= rank < world or total_requests < 1 or kv_heads < 1:
        raise ValueError("bad shard arguments")
    if total_requests >= world:
        lo = total_requests * rank // world
        hi = total_requests * (rank + 1) // world
        return Shard(tuple(range(lo, hi)), (0, kv_heads))
    per_req = world // total_requests  # ranks per request (the remainder ranks idle)
    req = rank // per_req
    if req >= total_requests:
        return Shard((), (0, 0))
    g = rank % per_req
    if kv_heads % per_req:
        raise ValueError(f"{kv_heads} KV heads do not split into {per_req} groups")
    step = kv_heads // per_req
    return Shard((req,), (g * step, (g + 1) * step))


def shard_heads(total_requests: int, kv_heads: int, world: int, rank: int) -> Shard:
    """Layer-level sharding: every rank serves all requests for one contiguous KV-head group (and
    its GQA query heads); the head-sharded outputs are all-gathered afterwards."""
    if world < 1 or not 0 <= rank < world or total_requests < 1 or kv_heads < 1:
        raise ValueError("bad shard arguments")
    if kv_heads % world:
        raise ValueError(f"{kv_heads} KV heads do not split into {world} groups")
    step = kv_heads // world
    return Shard(tuple(range(total_requests)), (rank * step, (rank + 1) * step))


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    vals = [float(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()
