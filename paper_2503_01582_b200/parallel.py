"""Multi-GPU partitioning of the per-object train step.

Objects are independent (each owns its parameters, Adam state, grid and
random stream: mapper.cpp:130-197, run under parallel_for at
mapper.cpp:572-585), so they are sharded across ranks with no data-path
collective. Ranks are balanced with LPT (longest processing time first) on
a per-object cost model of one train step:

    cost = samples_per_step * bytes_per_sample(arch) + 32 * P(arch)

(hash-grid gathers + table-gradient read-modify-write per sample, plus
dense Adam's 32 B/param).
"""
from __future__ import annotations

import heapq
import os
from dataclasses import dataclass

from .trainer import FieldArch


def bytes_per_sample(arch: FieldArch) -> int:
    """Encode fwd gathers (8 L F 4) + bwd RMW (2 * 8 L F 4) = 96 L F bytes."""
    return 96 * arch.hash_levels * arch.features_per_level


def step_cost(arch: FieldArch, rays: int, samples: int) -> float:
    return float(rays * samples * bytes_per_sample(arch) + 32 * arch.param_count())


def shard_lpt(costs, world: int) -> list[list[int]]:
    """Assign item indices to `world` ranks, greedily giving the next most
    expensive item to the least loaded rank. Deterministic (ties by index)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    for lst in out:
        lst.sort()
    return out


def imbalance(costs, shards) -> float:
    """max rank load / mean rank load (1.0 = perfect)."""
    loads = [sum(costs[i] for i in s) for s in shards]
    mean = sum(loads) / max(len(loads), 1)
    return max(loads) / mean if mean > 0 else 1.0


@dataclass
class DistInfo:
    world: int = 1
    rank: int = 0
    local_rank: int = 0

    @classmethod
    def from_env(cls) -> "DistInfo":
        return cls(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                   int(os.environ.get("LOCAL_RANK", "0")))
