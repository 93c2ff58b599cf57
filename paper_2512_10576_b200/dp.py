"""Data-parallel sharding of decode requests across the GPUs of one box.

Every (request, layer) pool is independent (
cache.py:176-177), so the path shards by request with no data-path collective:
each rank owns a disjoint request subset, its own slot pools and its own
(NUMA-local) host store.  The only cross-rank step is the throughput
aggregate — the reference's replica factor R (pipeline.py:330,
scenario.py:62) — done on the host side as SUM(tokens) / MAX(time).
"""

from __future__ import annotations

import heapq

import torch
import torch.distributed as dist


def shard_requests(num_requests: int, world: int, rank: int, lengths=None) -> list:
    """Request ids owned by ``rank``.  Equal-length batches go round-robin; mixed
    lengths (config C5) use longest-processing-time greedy on per-request work
    (indexer cost is linear in context)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if lengths is None:
        return list(range(rank, num_requests, world))
    heap = [(0, r) for r in range(world)]
    owner = [0] * num_requests
    for i in sorted(range(num_requests), key=lambda i: (-int(lengths[i]), i)):
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + int(lengths[i]), r))
    return [i for i in range(num_requests) if owner[i] == rank]


def aggregate(tokens: float, seconds: float, device=None):
    """(total tokens over ranks, max seconds over ranks); identity when not distributed."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(tokens), float(seconds)
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    t = torch.tensor([float(tokens)], dtype=torch.float64, device=dev)
    s = torch.tensor([float(seconds)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dist.all_reduce(s, op=dist.ReduceOp.MAX)
    return float(t.item()), float(s.item())
