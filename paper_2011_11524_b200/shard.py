"""Multi-GPU partitioning of the decimal-multiplication workload.

Batches of independent products (config 2) shard with no data-path collective: the
4096-product batch is split evenly, rank r of a world of G owning products
[r * count, (r + 1) * count) with count = 4096 / G (strong scaling, as BASELINE config 2
states; pair k is seeded (2k, 2k + 1)). The only cross-rank traffic is the timing
reduction (max over ranks) done by the bench (bench.py uses batch_range).
"""
from __future__ import annotations


def batch_range(rank: int, world: int, count_per_rank: int) -> range:
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return range(rank * count_per_rank, (rank + 1) * count_per_rank)


def pair_seeds(k: int) -> tuple[int, int]:
    """Seeds of the global product k: x = 2k, y = 2k + 1."""
    return 2 * k, 2 * k + 1


def shard_seeds(rank: int, world: int, count_per_rank: int) -> list[tuple[int, int]]:
    return [pair_seeds(k) for k in batch_range(rank, world, count_per_rank)]


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Device-time reduction used by the bench: every rank contributes its elapsed time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
