"""Frequency / polarisation sharding across ranks.

Independent frequencies go to different GPUs with no data-path collective:
each rank builds its own Green's operator and solves both polarisations of its
frequencies as one nrhs = 2 batch (they share every operator read). The only
communication is host-side bookkeeping: gathering per-frequency results on
rank 0 and the max-over-ranks time of the benchmark. Backend-agnostic: works
with NCCL on the GPU box and with gloo in the CPU tests.
"""
from __future__ import annotations

from typing import Callable, List, Sequence


def shard_indices(n_items: int, world: int, rank: int, cost: Sequence[float] | None = None) -> List[int]:
    """Indices of the items rank `rank` owns. Without costs: round robin
    (frequency f_i -> rank i mod world). With per-item
    costs (e.g. measured iteration counts): greedy longest-processing-time
    assignment, deterministic on every rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_indices: bad world/rank")
    if cost is None:
        return list(range(rank, n_items, world))
    order = sorted(range(n_items), key=lambda i: (-cost[i], i))
    load = [0.0] * world
    owner = [0] * n_items
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += cost[i]
    return [i for i in range(n_items) if owner[i] == rank]


def run_sweep(items: Sequence, job: Callable, rank: int, world: int, dist=None):
    """Run job(item) for this rank's items; gather {index: result} on rank 0
    (returns the merged dict there, this rank's dict elsewhere)."""
    mine = {i: job(items[i]) for i in shard_indices(len(items), world, rank)}
    if dist is None or world == 1:
        return mine
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    if rank != 0:
        return mine
    merged = {}
    for part in gathered:
        merged.update(part)
    return merged


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Benchmark time reduction: the job takes as long as its slowest rank."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
